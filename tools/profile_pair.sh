mkdir -p gpurun_out/ncu /tmp/ncu_reps
for v in shuffle plain; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k2d2' -s 1 -c 1 -f -o /tmp/ncu_reps/prof_jacobi2d_pair_${v} python tools/prof_run.py --workload jacobi2d_paper --variant $v --run > /dev/null 2>&1 || echo "ncu failed $v"
  python tools/ncu_ops.py /tmp/ncu_reps/prof_jacobi2d_pair_${v}.ncu-rep > gpurun_out/ncu/ops_jacobi2d_pair_${v}.txt 2>&1
done
cp profiles/traffic.json gpurun_out/ncu/
python tools/ncu_summary.py --round r01 --out gpurun_out/ncu /tmp/ncu_reps/prof_jacobi2d_pair_*.ncu-rep
