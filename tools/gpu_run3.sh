# one lane per pair with y in shared memory (3 CTAs/SM): parity + c4/c5 timings
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fill.py -x -q -p no:cacheprovider -k "instantiation or kill or tiny or planner" > gpurun_out/r2f_fill_tests.log 2>&1; echo "fill tests exit $?" >> gpurun_out/r2f_fill_tests.log
for f in "" "6,1,32" "6,1,28" "6,1,24" "3,1,32"; do
  if [ -z "$f" ]; then timeout 300 python tools/prof_fill.py --config 4 --reps 3; else timeout 300 python tools/prof_fill.py --config 4 --reps 3 --force $f; fi
done > gpurun_out/r2f_c4.log 2>&1
for f in "" "6,1,28" "3,1,28" "6,1,24" "3,1,24"; do
  if [ -z "$f" ]; then timeout 300 python tools/prof_fill.py --config 5 --reps 3; else timeout 300 python tools/prof_fill.py --config 5 --reps 3 --force $f; fi
done > gpurun_out/r2f_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dtw_full -c 1 -o gpurun_out/r2f_ncu_c4sub400_ysm python tools/prof_fill.py --config 4 --subset 400 --force 6,1,32 > gpurun_out/r2f_ncu.log 2>&1
echo done
