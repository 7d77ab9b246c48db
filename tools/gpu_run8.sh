set -x
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_run.py > gpurun_out/r2k_memcheck.log 2>&1; echo "memcheck exit $?" >> gpurun_out/r2k_memcheck.log
timeout 600 python -m pytest tests/test_gpu_fill.py -x -q -p no:cacheprovider > gpurun_out/r2k_fill.log 2>&1; echo "exit $?" >> gpurun_out/r2k_fill.log
for c in 5 1; do timeout 300 python tools/prof_fill.py --config $c --reps 3; done > gpurun_out/r2k_plans.log 2>&1
echo done
