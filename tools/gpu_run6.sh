set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fill.py -x -q -p no:cacheprovider -k "shared_y" > gpurun_out/r2i_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2i_tests.log
for f in "7,1,32" "7,1,28" "7,1,24"; do timeout 300 python tools/prof_fill.py --config 4 --reps 3 --force $f; done > gpurun_out/r2i_c4.log 2>&1
for f in "7,1,28" "7,1,24" "6,1,24"; do timeout 300 python tools/prof_fill.py --config 5 --reps 3 --force $f; done > gpurun_out/r2i_c5.log 2>&1
echo done
