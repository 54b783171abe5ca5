#!/bin/bash
# Round-2 evidence: launch list of the default bench command, then every workload's ncu capture.
mkdir -p gpurun_out/ncu
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu/r02_launches_gaussblur.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu/r02_launch_bench.log 2>&1; echo launches $?
ROUND=r02 bash tools/profile_all.sh
