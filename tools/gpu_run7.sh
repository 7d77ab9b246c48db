set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2j_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2j_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2j_bench_default.json 2> gpurun_out/r2j_bench_default.err; echo "bench exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tree_sum|assign_slots|cluster_select|permute|expand" -c 12 -o gpurun_out/r2j_ncu_c3_kmedoids python tools/km_bench.py --configs 3 --reps 1 > gpurun_out/r2j_ncu_km.log 2>&1; echo "ncu exit $?"
echo done
