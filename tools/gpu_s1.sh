#!/bin/bash
# session 1 (round 2, late): guard bands, config-0 timing floor, gaussblur separable pair profile
bash tools/gpu_guard.sh
timeout 300 python tools/small_run_timing.py > gpurun_out/small_run_timing.txt 2>&1; echo timing $?; cat gpurun_out/small_run_timing.txt
mkdir -p gpurun_out/ncu /tmp/ncu_reps
for v in shuffle plain; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k2d2' -s 1 -c 1 -f -o gpurun_out/ncu/prof_gaussblur_pair_$v python tools/prof_run.py --workload gaussblur --variant $v --run > /dev/null 2>&1 || echo "ncu failed $v"
  python tools/ncu_ops.py gpurun_out/ncu/prof_gaussblur_pair_$v.ncu-rep --hot 100000000 > gpurun_out/ncu/ops_gaussblur_pair_$v.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'ktb2r' -s 0 -c 1 -f -o gpurun_out/ncu/prof_jacobi2d_c0_shuffle python tools/prof_run.py --workload jacobi2d --variant shuffle --run > /dev/null 2>&1 || echo "ncu failed c0"
python tools/ncu_ops.py gpurun_out/ncu/prof_jacobi2d_c0_shuffle.ncu-rep > gpurun_out/ncu/ops_jacobi2d_c0_shuffle.txt 2>&1
