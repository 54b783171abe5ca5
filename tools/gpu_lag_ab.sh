#!/bin/bash
# release-form A/B on the streaming 2-D kernels: race hunt + bench for each library
for lib in "" expbuild/relb2/libstencil_b200.so expbuild/relb4/libstencil_b200.so expbuild/rel2/libstencil_b200.so; do
  echo "== lib [$lib]"
  export STB200_LIB=$lib
  H="timeout 1200 python tools/flake_hunt.py"
  $H --kind jacobi2d5 --n 32768 --iters 10 --reps 6 2>&1 | tail -1
  $H --kind jacobi2d9 --n 32768 --iters 9 --reps 4 2>&1 | tail -1
  bash tools/bench_all.sh gaussblur jacobi2d_paper gameoflife
done
