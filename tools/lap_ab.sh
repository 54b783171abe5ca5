for env in "STB200_LAP_PACE=0" "STB200_LAP_PACE=8" "STB200_LAP_PACE=4" "STB200_LAP_PACE=16"; do for v in shuffle plain; do
  env $env timeout 300 python bench.py --workload lapgsrb --variant $v --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$env $v]', round(d['value'],1), round(r['kernel_only_frac'],3))"
done; done
