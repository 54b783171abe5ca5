#!/bin/bash
# ncu --set full capture of one launch per workload x variant (run under gpurun, 1 GPU),
# summarised on the box (the reports are too large to bring back together):
#   tools/profile_all.sh [workloads...]
#   -> gpurun_out/ncu/r01_ncu_summary.md, traffic.json, ops_<w>_<v>.txt (dynamic opcode mix)
#      and the .ncu-rep of KEEP (default: tricubic shuffle) for source-level reading
W=${@:-"gaussblur jacobi2d_paper gameoflife laplacian wave13pt jacobi3d divergence gradient tricubic"}
KEEP=${KEEP:-"prof_tricubic_shuffle"}
mkdir -p gpurun_out/ncu /tmp/ncu_reps
for w in $W; do for v in shuffle plain; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k2d|k3d|ktricubic|kgrad' -s 2 -c 1 \
     -f -o /tmp/ncu_reps/prof_${w}_${v} python tools/prof_run.py --workload $w --variant $v --launches 3 > /dev/null 2>&1 \
     || echo "ncu failed: $w $v"
  python tools/ncu_ops.py /tmp/ncu_reps/prof_${w}_${v}.ncu-rep > gpurun_out/ncu/ops_${w}_${v}.txt 2>&1
done; done
cp profiles/traffic.json gpurun_out/ncu/ 2>/dev/null
python tools/ncu_summary.py --round ${ROUND:-r01} --out gpurun_out/ncu /tmp/ncu_reps/prof_*.ncu-rep
for k in $KEEP; do cp /tmp/ncu_reps/$k.ncu-rep gpurun_out/ 2>/dev/null; done
ls gpurun_out/ncu | wc -l
