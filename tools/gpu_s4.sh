#!/bin/bash
# final profiles of the headline kernel (compile-time ring slots) and the bench launch list
mkdir -p gpurun_out/ncu
for v in shuffle plain; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k2d2' -s 1 -c 1 -f -o gpurun_out/ncu/prof_gaussblur_pair_$v python tools/prof_run.py --workload gaussblur --variant $v --run > /dev/null 2>&1 || echo "ncu failed $v"
  python tools/ncu_ops.py gpurun_out/ncu/prof_gaussblur_pair_$v.ncu-rep > gpurun_out/ncu/ops_gaussblur_pair_$v.txt 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu/r02_launches_gaussblur.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu/r02_launch_bench.log 2>&1; echo launches $?
