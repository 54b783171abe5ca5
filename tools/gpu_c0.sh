#!/bin/bash
# config 0 (jacobi 512^2 x 10): parity of the fused paths, then bench lines
# for the register kernel (default) and the shared-memory tile kernel
python -m pytest tests/test_parity_2d.py tests/test_coeffs_gpu.py -q -x -k "fused or config0 or run_parity or closed" 2>&1 | tail -3
for env in "" "STB200_TB_SMEM=1"; do
  env $env python bench.py --workload jacobi2d --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$env]', d['variants'], 'ms/step', round(d['ms_per_step']*1e3,2), 'us')"
done
