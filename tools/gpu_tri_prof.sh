#!/bin/bash
# ncu --set full (source-level) capture of the fp32 tricubic kernel, both variants.
#   gpurun -- 'bash tools/gpu_tri_prof.sh'   -> gpurun_out/tri_{plain,shuffle}.ncu-rep
set -x
for v in plain shuffle; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:ktricubic \
      --launch-skip 2 --launch-count 1 -f -o gpurun_out/tri_$v \
      python tools/prof_run.py --workload tricubic --variant $v --launches 4 > gpurun_out/tri_prof_$v.log 2>&1
done
python bench.py --workload tricubic --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/tri_bench.json 2>gpurun_out/tri_bench.err
