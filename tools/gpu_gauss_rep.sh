for i in 1 2; do for fu in 2 3; do for v in shuffle plain; do
  timeout 300 python bench.py --workload gaussblur --variant $v --fusion $fu --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$i fusion=$fu] $v', round(d['value'],1), 'kfrac', round(r['kernel_only_frac'],3), d['clocks']['sm_mhz'])"
done; done; done
