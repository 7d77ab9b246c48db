# c4 kernel experiments: parity of the Full family, timings of forced configs, ncu of c4
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fill.py -x -q -p no:cacheprovider > gpurun_out/r2e_fill_tests.log 2>&1; echo "fill tests exit $?" >> gpurun_out/r2e_fill_tests.log
for f in "" "3,1,32" "3,8,30" "3,4,30" "3,2,30" "3,1,28"; do
  if [ -z "$f" ]; then timeout 300 python tools/prof_fill.py --config 4 --reps 3; else timeout 300 python tools/prof_fill.py --config 4 --reps 3 --force $f; fi
done > gpurun_out/r2e_c4_forced.log 2>&1
timeout 300 python tools/prof_fill.py --config 4 --reps 3 --prec 1 >> gpurun_out/r2e_c4_forced.log 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:dtw_full -c 1 python tools/prof_fill.py --config 4 > gpurun_out/r2e_ncu_c4_dram.log 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:dtw_full -c 1 python tools/prof_fill.py --config 4 --force 3,8,30 > gpurun_out/r2e_ncu_c4_dram_g8.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dtw_full -c 1 -o gpurun_out/r2e_ncu_c4sub400 python tools/prof_fill.py --config 4 --subset 400 > gpurun_out/r2e_ncu_c4sub400.log 2>&1
echo done
