set -x
mkdir -p gpurun_out
DTWGPU_VERBOSE=1 timeout 300 python tools/prof_fill.py --config 5 --reps 2 > gpurun_out/r2z_plan.log 2>&1
DTWGPU_VERBOSE=1 DTWGPU_PLAN_TABLE=0 timeout 300 python tools/prof_fill.py --config 5 --reps 2 >> gpurun_out/r2z_plan.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fill.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py -x -q -p no:cacheprovider -k "not c3_full_matrix and not c3_kmedoids" > gpurun_out/r2z_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2z_tests.log
echo done
