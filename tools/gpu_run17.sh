set -x
mkdir -p gpurun_out
./tools/build/mix > gpurun_out/r2t_mix.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kmedoids.py tests/test_gpu_dropin.py -x -q -p no:cacheprovider > gpurun_out/r2t_km_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2t_km_tests.log
timeout 600 python tools/km_bench.py --configs 3 5 --reps 6 --workers 4 --only-workers > gpurun_out/r2t_km.log 2>&1
echo done
