#!/bin/bash
# ncu --set full capture of klapgsrb2 (both variants)
for v in shuffle plain; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:klapgsrb2 \
      --launch-skip 2 --launch-count 1 -f -o gpurun_out/prof_lapgsrb_$v \
      python tools/prof_run.py --workload lapgsrb --variant $v --launches 4 > gpurun_out/lap_prof_$v.log 2>&1
  echo $v $?
done
