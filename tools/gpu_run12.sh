set -x
mkdir -p gpurun_out
for lib in paper_2307_04904_b200/libdtwgpu.so exp/libdtwgpu_u2.so; do
  for c in 4 5 1; do DTWGPU_LIB=$PWD/$lib timeout 300 python tools/prof_fill.py --config $c --reps 3; done
  DTWGPU_LIB=$PWD/$lib timeout 300 python tools/prof_fill.py --config 4 --reps 3 --prec 1
done > gpurun_out/r2o_unroll.log 2>&1
echo done
