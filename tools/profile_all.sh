#!/bin/bash
# ncu --set full capture of one launch per workload x variant (run under gpurun, 1 GPU).
#   tools/profile_all.sh [workloads...]   -> gpurun_out/prof_<workload>_<variant>.ncu-rep
W=${@:-"gaussblur jacobi2d_paper gameoflife laplacian wave13pt jacobi3d divergence gradient tricubic"}
mkdir -p gpurun_out
for w in $W; do for v in shuffle plain; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k2d|k3d|ktricubic' -s 2 -c 1 \
     -f -o gpurun_out/prof_${w}_${v} python tools/prof_run.py --workload $w --variant $v --launches 3 > /dev/null 2>&1 \
     || echo "ncu failed: $w $v"
done; done
ls gpurun_out/*.ncu-rep | wc -l
