set -x
mkdir -p gpurun_out
for c in 5 2 1 3; do timeout 300 python tools/prof_fill.py --config $c --reps 3; done > gpurun_out/r2h_plans.log 2>&1
timeout 300 python tools/prof_fill.py --config 5 --reps 3 --prec 1 >> gpurun_out/r2h_plans.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fill.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "c5 or planner or config or full_size" > gpurun_out/r2h_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2h_tests.log
echo done
