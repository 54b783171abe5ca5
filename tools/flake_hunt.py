#!/usr/bin/env python
"""Repeat a stencil_run many times on the same input and compare every
result bit for bit with the first (the kernels are deterministic, so any
difference is a race).  Between repeats other kinds run on other buffers to
vary the SM / L2 state.  Usage: python tools/flake_hunt.py [--reps N]"""
import argparse
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_11389_b200 import inputs  # noqa: E402
from paper_2301_11389_b200.binding import Stencil  # noqa: E402


def digest(t):
    return hashlib.sha1(t.cpu().numpy().tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=40)
    ap.add_argument("--kind", default="gaussblur5x5")
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--shape", default="", help="nz,ny,nx for 3-D kinds (numpy order)")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--variants", default="plain,shuffle")
    a = ap.parse_args()
    shape = tuple(int(v) for v in a.shape.split(",")) if a.shape else (a.n, a.n)
    dims = shape[::-1]
    probe = Stencil(a.kind, dims, a.dtype)
    n_in, n_out, n_bufs = probe.arity()
    probe.close()
    fields = [torch.from_numpy(inputs.generate_np(shape, a.dtype, inputs.BASE_SEED + 1, k)).cuda()
              for k in range(n_in)]
    other = torch.from_numpy(inputs.generate_np((130, 258, 256), "f32", 7)).cuda()
    oth = Stencil("laplacian3d7", (256, 258, 130), "f32")
    bad = 0
    for var in a.variants.split(","):
        ref = None
        for r in range(a.reps):
            st = Stencil(a.kind, dims, a.dtype, variant=var)
            bufs = [t.clone() for t in fields] + [torch.zeros_like(fields[0]) for _ in range(n_bufs - n_in)]
            idx = st.run(bufs, a.iters)
            torch.cuda.synchronize()
            allb = torch.cat([b.reshape(-1) for b in bufs])     # every buffer of the run
            d = digest(allb)
            st.close()
            if ref is None:
                ref = (d, allb.clone())
            elif d != ref[0]:
                bad += 1
                diff = (allb != ref[1]).nonzero()
                print(f"{var} rep {r}: MISMATCH {diff.shape[0]} points, first {diff[:4].tolist()}")
            if r % 3 == 0:                                  # perturb: another kernel family
                o2 = torch.zeros_like(other)
                oth.run([other.clone(), o2], 3)
        print(f"{a.kind} {var}: {a.reps} reps, ref {ref[0][:12]}")
    print("mismatches", bad)


if __name__ == "__main__":
    main()
