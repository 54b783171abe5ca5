"""Per-launch event times of back-to-back sweeps (power / clock ramp check)."""
import os, sys, json, subprocess, threading, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2301_11389_b200 import inputs
from paper_2301_11389_b200.binding import Stencil
import bench
wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "gaussblur"]
var = sys.argv[2] if len(sys.argv) > 2 else "shuffle"
st = Stencil(wl["kind"], wl["dims"], wl["dtype"], variant=var)
n_in, n_out, _ = st.arity()
ins = [inputs.generate_torch(tuple(wl["dims"][::-1]), wl["dtype"], 1, k) for k in range(n_in)]
outs = [torch.zeros_like(ins[0]) for _ in range(n_out)]
pingpong = n_in == 1 and n_out == 1
N = 400
ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
for _ in range(5): st.step(ins, outs)
torch.cuda.synchronize(); time.sleep(1.0)
with bench.ClockSampler(0) as clk:
    ev[0].record()
    for i in range(N):
        if pingpong and i % 2:
            st.step(outs, ins)
        else:
            st.step(ins, outs)
        ev[i + 1].record()
    torch.cuda.synchronize()
t = [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(N)]
print(json.dumps({"first10_us": [round(x, 1) for x in t[:10]], "median_us": sorted(t)[N // 2],
                  "last10_us": [round(x, 1) for x in t[-10:]], "clocks": clk.summary(),
                  "raw_clock_lines": clk.lines[:3] + clk.lines[-3:]}))
