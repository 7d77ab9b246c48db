#!/bin/bash
# Bounds-checked build of libdtwgpu.so (-DDTWG_CHECK_BOUNDS: every sample load of the
# Full/lane kernels inside the guarded series buffer, every boundary-column row inside its
# group's scratch column; a violation prints and traps) and the sanitizer smoke over it.
# compute-sanitizer is closed on this GPU pool, so this is the memcheck substitute
# (ragged long/short pairs with one lane per pair).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -s -j8 -C "$ROOT/paper_2307_04904_b200/csrc" OUT="$ROOT/exp/libdtwgpu_chk.so" \
  OBJ="$ROOT/exp/build_chk" EXTRA=-DDTWG_CHECK_BOUNDS
[ "$1" = "--build-only" ] && exit 0
DTWGPU_LIB="$ROOT/exp/libdtwgpu_chk.so" python "$ROOT/tools/sanitize_run.py"
