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


def time_variant(kind, dtype, n, runs, var, a, b):
    st = Stencil(kind, (n, n), dtype, variant=var)
    for _ in range(3):
        st.step([a], [b])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(runs):
        st.step([a], [b])
    e1.record()
    torch.cuda.synchronize()
    st.close()
    return e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--runs", type=int, default=10)
    args = ap.parse_args()
    out = {"source": "tools/paper_fig3.py", "grid": [args.n, args.n], "runs": args.runs, "results": {}}
    for kind, dtype in (("jacobi2d9", "f32"), ("gaussblur5x5", "f32"), ("gameoflife", "i32")):
        a = inputs.generate_torch((args.n, args.n), dtype, inputs.BASE_SEED + 30)
        b = torch.zeros_like(a)
        ms = {v: time_variant(kind, dtype, args.n, args.runs, v, a, b) for v in VARIANTS}
        pts = (args.n - 2 * (2 if kind == "gaussblur5x5" else 1)) ** 2 * args.runs
        out["results"][kind] = {
            v: {"ms": ms[v], "gpts": pts / (ms[v] / 1e3) / 1e9,
                "speedup_vs_original": ms["paper_original"] / ms[v]} for v in VARIANTS}
        del a, b
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
