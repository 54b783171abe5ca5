#!/bin/bash
# gameoflife packed kernel (klife.cuh): parity, then bench lines (packed 2 / 3 sweeps, int32 k2d2)
timeout 900 python -m pytest tests/test_parity_2d.py -q -x -k "life or gameoflife" -p no:cacheprovider 2>&1 | tail -3
for env in "X=0" "STB200_2D_NSW=3" "STB200_LIFE_INT=1"; do for v in shuffle plain; do
  env $env timeout 300 python bench.py --workload gameoflife --variant $v --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$env] $v', round(d['value'],1), 'Gpt/s frac', round(r['frac'],3), 'kfrac', round(r['kernel_only_frac'],3), d['config']['sweeps_per_launch'], d['clocks']['sm_mhz'])"
done; done
