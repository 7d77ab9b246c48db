set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2s_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2s_bench_default.json 2> gpurun_out/r2s_bench_default.err; echo "bench exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2s_smoke.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2s_bench_ref.json 2>&1
echo done
