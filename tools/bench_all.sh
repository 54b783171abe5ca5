#!/bin/bash
# One bench line per workload x variant (summary form).  Usage: tools/bench_all.sh [workloads...]
W=${@:-"gaussblur jacobi2d jacobi2d_paper gameoflife laplacian wave13pt jacobi3d divergence gradient tricubic"}
for w in $W; do for v in shuffle plain; do
  timeout 300 python bench.py --workload $w --variant $v --steps 10 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
t=sys.stdin.read().strip()
if not t: print('$w $v FAILED'); sys.exit()
d=json.loads(t); r=d['roofline']
print('%-14s %-8s %8.1f Gpt/s frac %.3f kern_us %8.1f kfrac %.3f clk %s %s'%(d['config']['kind'], d['config']['variant'], d['value'], r['frac'], r['kernel_only_us'], r['kernel_only_frac'], d['clocks']['sm_mhz'], ','.join(d['clocks']['reasons'])))"
done; done
