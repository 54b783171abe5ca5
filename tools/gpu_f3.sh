#!/bin/bash
# f3 kinds: parity (fast then slow) and bench lines
python -m pytest tests/test_parity_f3.py -q -x -m "not slow" 2>&1 | tail -5
python -m pytest tests/test_parity_f3.py -q -x -m "slow" 2>&1 | tail -5
for w in uxx1 whispering lapgsrb tricubic2; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['variants'], round(d['roofline']['frac'],3), round(d['roofline']['kernel_only_frac'],3))"
done
