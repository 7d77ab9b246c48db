set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fill.py tests/test_gpu_kmedoids.py -x -q -p no:cacheprovider > gpurun_out/r2m_fill.log 2>&1; echo "exit $?" >> gpurun_out/r2m_fill.log
timeout 600 python tools/km_bench.py --configs 3 5 --reps 3 > gpurun_out/r2m_km.log 2>&1
echo done
