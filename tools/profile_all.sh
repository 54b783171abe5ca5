#!/bin/bash
# ncu --set full capture of one launch per workload x variant (run under gpurun, 1 GPU),
# summarised on the box (the reports are too large to bring back together):
#   ROUND=r02 tools/profile_all.sh [workloads...]
#   -> gpurun_out/ncu/${ROUND}_ncu_summary.md, traffic.json, ops_<w>_<v>.txt (dynamic opcode mix)
#      and the .ncu-rep of KEEP for source-level reading.  Workloads ending in
#      _pair profile one multi-sweep launch inside a stencil_run (k2d2 / k2dlife).
W=${@:-"gaussblur jacobi2d_paper gameoflife laplacian wave13pt jacobi3d divergence gradient tricubic uxx1 whispering lapgsrb tricubic2 jacobi2d_paper_pair gameoflife_pair gaussblur_pair"}
KEEP=${KEEP:-"prof_tricubic_shuffle prof_lapgsrb_shuffle"}
ROUND=${ROUND:-r02}
mkdir -p gpurun_out/ncu /tmp/ncu_reps
for w in $W; do for v in shuffle plain; do
  case $w in
    *_pair) base=${w%_pair}; args="--workload $base --variant $v --run"; kre='k2d2|k2dlife'; skip=1 ;;
    *) args="--workload $w --variant $v --launches 3"; kre='k2d|k3d|ktricubic|kgrad|kuxx1|kwhisper|klapgsrb'; skip=2 ;;
  esac
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 \
     -f -o /tmp/ncu_reps/prof_${w}_${v} python tools/prof_run.py $args > /dev/null 2>&1 \
     || echo "ncu failed: $w $v"
  python tools/ncu_ops.py /tmp/ncu_reps/prof_${w}_${v}.ncu-rep > gpurun_out/ncu/ops_${w}_${v}.txt 2>&1
done; done
cp profiles/traffic.json gpurun_out/ncu/ 2>/dev/null
python tools/ncu_summary.py --round $ROUND --out gpurun_out/ncu /tmp/ncu_reps/prof_*.ncu-rep
for k in $KEEP; do cp /tmp/ncu_reps/$k.ncu-rep gpurun_out/ 2>/dev/null; done
ls gpurun_out/ncu | wc -l
