set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fill.py -x -q -p no:cacheprovider -k "instantiation or kill or tiny or planner" > gpurun_out/r2g_fill_tests.log 2>&1; echo "fill tests exit $?" >> gpurun_out/r2g_fill_tests.log
for f in "6,1,24" "6,1,20" "6,1,16"; do timeout 300 python tools/prof_fill.py --config 5 --reps 3 --force $f; done > gpurun_out/r2g_c5.log 2>&1
for f in "6,1,20" "6,1,16"; do timeout 300 python tools/prof_fill.py --config 4 --reps 3 --force $f; done > gpurun_out/r2g_c4.log 2>&1
echo done
