mkdir -p gpurun_out/ncu /tmp/ncu_reps
# ncu --set full of one two-sweep (k2d2) launch inside a stencil_run, per workload x variant
for w in jacobi2d_paper gameoflife; do for v in shuffle plain; do
  n=${w%_paper}_pair
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k2d2' -s 1 -c 1 -f -o /tmp/ncu_reps/prof_${n}_${v} python tools/prof_run.py --workload $w --variant $v --run > /dev/null 2>&1 || echo "ncu failed $w $v"
  python tools/ncu_ops.py /tmp/ncu_reps/prof_${n}_${v}.ncu-rep > gpurun_out/ncu/ops_${n}_${v}.txt 2>&1
done; done
cp profiles/traffic.json gpurun_out/ncu/
python tools/ncu_summary.py --round r01 --out gpurun_out/ncu /tmp/ncu_reps/prof_*_pair_*.ncu-rep
