set -x
mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Core"
./tools/build/mix > gpurun_out/r2n_mix.log 2>&1
timeout 600 python tools/km_bench.py --configs 3 --reps 6 --workers 2 3 4 5 6 8 10 --only-workers > gpurun_out/r2n_km_workers.log 2>&1
echo done
