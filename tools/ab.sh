#!/bin/bash
# A/B of experiment builds in one GPU session:  tools/ab.sh "<workloads>" exp1 exp2 ...
# ("base" = the in-tree library)
W=$1; shift
for e in "$@"; do
  if [ "$e" = base ]; then unset STB200_LIB; else export STB200_LIB=$PWD/expbuild/$e/libstencil_b200.so; fi
  echo "== $e"; bash tools/bench_all.sh $W
done
