#!/usr/bin/env python
"""B200 analogue of the paper's Figure 3: time of
the paper-literal variants (1 output/thread, Listing 6 code shape) relative
to ORIGINAL, next to the register-cache kernels, on the paper's 2-D size
32768^2 fp32, 10 kernel runs ("running the kernel ten
times").  Prints one JSON object.

    python tools/paper_fig3.py [--n 32768] [--runs 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2301_11389_b200 import inputs  # noqa: E402
from paper_2301_11389_b200.binding import Stencil  # noqa: E402

VARIANTS = ["paper_original", "paper_ptxasw", "paper_noload", "paper_nocorner", "paper_uniform",
            "plain", "shuffle"]


def time_variant(kind, dtype, dims, runs, var, ins, outs):
    st = Stencil(kind, dims, dtype, variant=var)
    for _ in range(3):
        st.step(ins, outs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(runs):
        st.step(ins, outs)
    e1.record()
    torch.cuda.synchronize()
    st.close()
    return e0.elapsed_time(e1)


# 3-D suite members: (kind, inputs, outputs, lo, hi)
KINDS_3D = [("laplacian3d7", 1, 1, 1, 1), ("wave13pt", 2, 1, 2, 2), ("divergence", 3, 1, 1, 1),
            ("gradient", 1, 3, 1, 1), ("tricubic", 4, 1, 1, 2)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--runs", type=int, default=10)
    ap.add_argument("--dims3", default="512,1024,1024",
                    help="3-D grid nx,ny,nz (the paper's 512x1024x1024, PAPER.md:645)")
    ap.add_argument("--no-2d", action="store_true")
    args = ap.parse_args()
    d3 = tuple(int(x) for x in args.dims3.split(","))
    out = {"source": "tools/paper_fig3.py", "grid": [args.n, args.n], "grid3": list(d3), "runs": args.runs,
           "results": {}}
    for kind, nin, nout, lo, hi in KINDS_3D:
        shape = d3[::-1]
        ins = [inputs.generate_torch(shape, "f32", inputs.BASE_SEED + 31, a) for a in range(nin)]
        outs = [torch.zeros_like(ins[0]) for _ in range(nout)]
        ms = {v: time_variant(kind, "f32", d3, args.runs, v, ins, outs) for v in VARIANTS}
        pts = (d3[0] - lo - hi) * (d3[1] - lo - hi) * (d3[2] - lo - hi) * args.runs
        out["results"][kind] = {
            v: {"ms": ms[v], "gpts": pts / (ms[v] / 1e3) / 1e9,
                "speedup_vs_original": ms["paper_original"] / ms[v]} for v in VARIANTS}
        del ins, outs
        torch.cuda.empty_cache()
    for kind, dtype in (() if args.no_2d else (("jacobi2d9", "f32"), ("gaussblur5x5", "f32"),
                                                ("gameoflife", "i32"))):
        a = inputs.generate_torch((args.n, args.n), dtype, inputs.BASE_SEED + 30)
        b = torch.zeros_like(a)
        ms = {v: time_variant(kind, dtype, (args.n, args.n), args.runs, v, [a], [b]) for v in VARIANTS}
        pts = (args.n - 2 * (2 if kind == "gaussblur5x5" else 1)) ** 2 * args.runs
        out["results"][kind] = {
            v: {"ms": ms[v], "gpts": pts / (ms[v] / 1e3) / 1e9,
                "speedup_vs_original": ms["paper_original"] / ms[v]} for v in VARIANTS}
        del a, b
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
