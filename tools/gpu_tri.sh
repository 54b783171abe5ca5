timeout 900 python -m pytest tests -x -q -m gpu -k "tricubic" > gpurun_out/pytest_tri.log 2>&1; echo pytest $?; tail -3 gpurun_out/pytest_tri.log
for v in shuffle plain; do timeout 300 python bench.py --workload tricubic --variant $v --steps 10 --no-e2e --no-cpu-baseline; done > gpurun_out/tri_bench.txt 2>&1
STB200_TRI1=1 timeout 300 python bench.py --workload tricubic --variant shuffle --steps 10 --no-e2e --no-cpu-baseline >> gpurun_out/tri_bench.txt 2>&1
python - <<'P'
import json
for l in open('gpurun_out/tri_bench.txt'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config']['variant'], round(d['value'],1), round(d['roofline']['frac'],3), d['roofline']['kernel_only_us'])
P
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'ktricubic' -s 2 -c 1 -f -o gpurun_out/prof_tri2_shuffle python tools/prof_run.py --workload tricubic --variant shuffle --launches 3 > /dev/null 2>&1; echo ncu $?
