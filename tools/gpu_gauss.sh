#!/bin/bash
# gaussblur separable (OpGauss5Sep): parity, then bench lines; args: extra "ENV=..." settings to compare
timeout 900 python -m pytest tests/test_parity_2d.py tests/test_coeffs_gpu.py tests/test_large_gpu.py -q -x -k "gauss" -p no:cacheprovider 2>&1 | tail -3
for env in "X=0" "$@"; do for fu in 1 2; do for v in shuffle plain; do
  env $env timeout 300 python bench.py --workload gaussblur --variant $v --fusion $fu --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$env fusion=$fu] $v', round(d['value'],1), 'Gpt/s frac', round(r['frac'],3), 'kfrac', round(r['kernel_only_frac'],3), d['config']['sweeps_per_launch'], d['clocks']['sm_mhz'])"
done; done; done
