set -x
mkdir -p gpurun_out
DTWGPU_LIB=$PWD/exp/libdtwgpu_chk.so timeout 900 python tools/sanitize_run.py > gpurun_out/r2l_bounds.log 2>&1; echo "bounds exit $?" >> gpurun_out/r2l_bounds.log
timeout 600 python -m pytest tests/test_gpu_fill.py -x -q -p no:cacheprovider > gpurun_out/r2l_fill.log 2>&1; echo "exit $?" >> gpurun_out/r2l_fill.log
echo done
