"""Minimal driver for ncu: run `--launches` single sweeps of a bench workload.

    ncu ... python tools/prof_run.py --workload gaussblur --variant shuffle --launches 8
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2301_11389_b200 import inputs  # noqa: E402
from paper_2301_11389_b200.binding import Stencil  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="gaussblur")
ap.add_argument("--variant", default="shuffle")
ap.add_argument("--launches", type=int, default=8)
ap.add_argument("--run", action="store_true", help="one stencil_run (graph) instead of steps")
ap.add_argument("--fusion", type=int, default=None, help="stencil_set_fusion before the run")
a = ap.parse_args()
wl = bench.WORKLOADS[a.workload]
st = Stencil(wl["kind"], wl["dims"], wl["dtype"], variant=a.variant)
if a.fusion is not None:
    st.set_fusion(a.fusion)
n_in, n_out, n_bufs = st.arity()
shape = tuple(wl["dims"][::-1])
f = [inputs.generate_torch(shape, wl["dtype"], 1, k) for k in range(n_in)]
outs = [torch.zeros_like(f[0]) for _ in range(n_out)]
if a.run:
    bufs = f + outs if n_bufs != 2 else [f[0], outs[0]]
    st.run(bufs, wl["iters"])
else:
    for i in range(a.launches):
        st.step(f, outs)
torch.cuda.synchronize()
print("done", a.workload, a.variant)
