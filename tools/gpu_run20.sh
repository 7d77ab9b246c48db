mkdir -p gpurun_out
./tools/build/block > gpurun_out/r2w_block.log 2>&1
