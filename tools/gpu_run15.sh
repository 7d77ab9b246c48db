set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fill.py -x -q -p no:cacheprovider -k "parallelogram" > gpurun_out/r2r_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2r_tests.log
for f in "" "7,1,32" "7,1,28" "7,1,24"; do
  if [ -z "$f" ]; then timeout 300 python tools/prof_fill.py --config 4 --reps 3; else timeout 300 python tools/prof_fill.py --config 4 --reps 3 --force $f; fi
done > gpurun_out/r2r_c4.log 2>&1
echo done
