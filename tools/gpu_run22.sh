set -x
mkdir -p gpurun_out
DTWGPU_VERBOSE=1 timeout 300 python tools/prof_fill.py --config 5 --reps 2 > gpurun_out/r2y_plan.log 2>&1
echo done
