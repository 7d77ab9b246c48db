set -x
mkdir -p gpurun_out
for f in "" "0,16,32" "0,32,16" "3,16,16"; do
  if [ -z "$f" ]; then timeout 300 python tools/prof_fill.py --config 1 --reps 5; else timeout 300 python tools/prof_fill.py --config 1 --reps 5 --force $f; fi
done > gpurun_out/r2p_c1.log 2>&1
timeout 300 python -m pytest tests/test_gpu_fill.py -x -q -p no:cacheprovider -k "every_instantiation" > gpurun_out/r2p_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2p_tests.log
echo done
