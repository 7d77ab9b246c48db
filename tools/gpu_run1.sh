set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo "bench exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dtw_ -c 1 -o gpurun_out/r2_ncu_c4_full python tools/prof_fill.py --config 4 > gpurun_out/r2_ncu_c4.log 2>&1; echo "ncu exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_default.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r2_ncu_launch.log 2>&1; echo "ncu2 exit $?"
