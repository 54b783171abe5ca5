#!/bin/bash
# lapgsrb: parity (klapgsrb2), then bench lines (auto tile height, and the env overrides given as args)
timeout 900 python -m pytest tests/test_parity_f3.py -q -x -k lapgsrb -p no:cacheprovider 2>&1 | tail -4
for env in "X=0" "$@"; do for v in shuffle plain; do
  env $env timeout 300 python bench.py --workload lapgsrb --variant $v --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$env] $v', round(d['value'],1), 'Gpt/s frac', round(r['frac'],3), 'kfrac', round(r['kernel_only_frac'],3), d['clocks'])"
done; done
