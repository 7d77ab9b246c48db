set -x
mkdir -p gpurun_out
for f in "" "3,1,46" "0,1,46"; do
  if [ -z "$f" ]; then timeout 300 python tools/prof_fill.py --config 3 --reps 3; else timeout 300 python tools/prof_fill.py --config 3 --reps 3 --force $f; fi
done > gpurun_out/r2aa_c3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fill.py -x -q -p no:cacheprovider -k "table_planner or one_lane or tiny" > gpurun_out/r2aa_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2aa_tests.log
echo done
