#!/bin/bash
# ncu --set full of the final jacobi2d5 32768^2 three-sweep launch (both variants)
mkdir -p gpurun_out/ncu
for v in shuffle plain; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k2d2' -s 1 -c 1 -f -o gpurun_out/ncu/prof_jacobi2d_paper_pair_$v python tools/prof_run.py --workload jacobi2d_paper --variant $v --run > /dev/null 2>&1 || echo "ncu failed $v"
  python tools/ncu_ops.py gpurun_out/ncu/prof_jacobi2d_paper_pair_$v.ncu-rep > gpurun_out/ncu/ops_jacobi2d_paper_pair_$v.txt 2>&1
done
