#!/bin/bash
# A/B of fp32 tricubic builds in one session: parity of the default build,
# then bench lines for the default and every expbuild/tri_* library.
python -m pytest tests/test_parity_3d.py -q -x -k "tricubic" 2>&1 | tail -2
run() {
  python bench.py --workload tricubic --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['variants'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
}
for rep in 1 2; do
  run default
  for lib in expbuild/tri_*/libstencil_b200.so; do STB200_LIB=$lib run $(basename $(dirname $lib)); done
done
