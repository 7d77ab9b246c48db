set -x
mkdir -p gpurun_out
for f in "" "34,8,26" "32,8,28" "13,8,26"; do
  if [ -z "$f" ]; then timeout 300 python tools/prof_fill.py --config 2 --reps 5; else timeout 300 python tools/prof_fill.py --config 2 --reps 5 --force $f; fi
done > gpurun_out/r2q_c2.log 2>&1
echo done
