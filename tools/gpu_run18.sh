set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:dtw_ --csv --log-file gpurun_out/r2u_c5_launches.csv python tools/prof_fill.py --config 5 > gpurun_out/r2u_c5.log 2>&1
timeout 300 python tools/prof_fill.py --config 5 --reps 3 >> gpurun_out/r2u_c5.log 2>&1
timeout 300 python tools/prof_fill.py --config 5 --reps 3 --prec 1 >> gpurun_out/r2u_c5.log 2>&1
echo done
