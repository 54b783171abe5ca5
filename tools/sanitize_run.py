"""Tiny-shape driver for compute-sanitizer: every kind, dtype and
variant through every kernel family on small ragged grids, as single steps
and short runs (ping-pong / three-level / re-apply), plus the fused 2-D
paths (ktb2r, ktb2d, k2d2 two / three sweeps) and the paper-literal family.

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool synccheck python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick

Every output is also checked against the CPU oracle (tests/parity.py), so a
run under a tool that perturbs timing still proves the results.

Guard bands (always on; the gpurun pool refuses compute-sanitizer, so this is
the bounds check that runs there): every device buffer is a 16-byte-aligned
slice in the middle of a larger allocation whose GUARD elements before and
after are poisoned (NaN for floating point, 0x7f7f7f7f for int32).  A kernel
that writes outside its buffer changes a guard (checked bit for bit after
every run); one that reads outside its buffer into a result turns that
result NaN / garbage (caught by the oracle comparison).

    python tools/sanitize_run.py           # no tool: guard bands + oracle parity
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import pyoracle  # noqa: E402
from paper_2301_11389_b200 import inputs  # noqa: E402
from paper_2301_11389_b200.binding import Stencil  # noqa: E402
from parity import assert_parity  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true", help="one shape per kind, SHUFFLE + PLAIN only")
ap.add_argument("--canary", action="store_true",
                help="a deliberately undersized output buffer: the guard check MUST fire "
                     "(proves the guards see this library's out-of-bounds writes)")
a = ap.parse_args()

KINDS2 = ["jacobi2d5", "jacobi2d9", "gaussblur5x5", "gameoflife", "whispering"]
KINDS3 = ["laplacian3d7", "jacobi3d7", "wave13pt", "divergence", "gradient", "tricubic", "tricubic2",
          "uxx1", "lapgsrb"]
SH2 = [(37, 260), (9, 132)] if not a.quick else [(37, 260)]
SH3 = [(9, 35, 132), (6, 7, 68)] if not a.quick else [(9, 35, 132)]
PAPER = ["paper_original", "paper_ptxasw", "paper_noload", "paper_nocorner", "paper_uniform"]
n_checked = 0
GUARD = 4096                      # elements on each side (16 / 32 KiB)
POISON = {"f32": float("nan"), "f64": float("nan"), "i32": 0x7f7f7f7f}


def guarded(host: np.ndarray):
    """Device copy of `host` inside a poisoned allocation: (view, whole)."""
    n = host.size
    whole = torch.empty(n + 2 * GUARD, dtype=torch.from_numpy(host[:0].reshape(-1)).dtype, device="cuda")
    whole.fill_(POISON["i32" if host.dtype == np.int32 else "f32"])
    view = whole[GUARD:GUARD + n].view(host.shape)
    view.copy_(torch.from_numpy(host))
    assert view.data_ptr() % 16 == 0
    return view, whole


def check_guards(wholes, what):
    for w in wholes:
        h = w.cpu().numpy()
        for part in (h[:GUARD], h[-GUARD:]):
            if part.dtype == np.int32:
                ok = np.all(part == 0x7f7f7f7f)
            else:
                ok = np.all(np.isnan(part)) and np.all(part.view(np.uint32 if part.dtype == np.float32
                                                                    else np.uint64) == part[:1].view(
                    np.uint32 if part.dtype == np.float32 else np.uint64))
            assert ok, f"{what}: a guard band was overwritten (out-of-bounds write)"


if a.canary:
    # a deliberately undersized output buffer: the guard check MUST fire
    # (proves the guards see this library's out-of-bounds writes)
    st = Stencil("jacobi2d5", (260, 37), "f32")
    src, _ = guarded(np.ones((37, 260), np.float32))
    dst, whole = guarded(np.zeros((30, 260), np.float32))  # 7 rows short: writes land in the guard
    st.step([src], [dst])
    torch.cuda.synchronize()
    try:
        check_guards([whole], "canary")
    except AssertionError as e:
        print("canary detected:", e)
        sys.exit(0)
    print("canary NOT detected")
    sys.exit(1)


def dtypes(kind):
    if kind == "gameoflife":
        return ["i32"]
    if kind in ("whispering",):
        return ["f32"]
    return ["f32", "f64"] if not a.quick else ["f32"]


def bufs_of(kind, dtype, shape, seed):
    ar = pyoracle.arity(kind)
    ins = [inputs.generate_np(shape, dtype, seed, k) for k in range(ar["n_in"])]
    if ar["n_bufs"] == 2:
        return ar, [ins[0], np.zeros_like(ins[0])]
    if ar["n_bufs"] == 3 and ar["n_in"] == 2:
        return ar, [ins[0], ins[1], np.zeros_like(ins[0])]
    return ar, ins + [np.zeros_like(ins[0]) for _ in range(ar["n_out"])]


def check_run(kind, dtype, shape, variant, n, fusion=None):
    global n_checked
    ar, bufs = bufs_of(kind, dtype, shape, inputs.BASE_SEED + 77)
    ob = [b.copy() for b in bufs]
    ridx = pyoracle.run(kind, dtype, ob, n)
    st = Stencil(kind, shape[::-1], dtype, variant=variant)
    if fusion is not None:
        st.set_fusion(fusion)
    gb = [guarded(b) for b in bufs]
    d = [v for v, _ in gb]
    gidx = st.run(d, n)
    torch.cuda.synchronize()
    check_guards([w for _, w in gb], f"{kind} {dtype} {shape} {variant} n={n} fusion={fusion}")
    nres = 1 if ar["n_bufs"] == 2 or (ar["n_bufs"] == 3 and ar["n_in"] == 2) else ar["n_out"]
    lo, hi = ar["lo"], ar["hi"]
    sl = tuple(slice(lo, m - hi) for m in shape)
    for k in range(nres):
        g = d[gidx + k].cpu().numpy()
        assert_parity(g[sl], ob[ridx + k][sl], dtype, f"{kind} {dtype} {shape} {variant} n={n} fusion={fusion}")
    st.close()
    n_checked += 1


for kind in KINDS2 + KINDS3:
    for dt in dtypes(kind):
        for shape in (SH2 if kind in KINDS2 else SH3):
            if min(shape) < 6:
                continue
            for var in ("shuffle", "plain"):
                check_run(kind, dt, shape, var, 1)
                check_run(kind, dt, shape, var, 3)
    print("ok", kind, flush=True)

# fused 2-D paths: ktb2r (auto for L2-resident grids), ktb2d (-S with the smem
# kernel is selected by env only), k2d2 two / three sweeps
for kind in ("jacobi2d5", "jacobi2d9", "gaussblur5x5", "gameoflife"):
    dt = "i32" if kind == "gameoflife" else "f32"
    for var in ("shuffle", "plain"):
        check_run(kind, dt, (70, 516), var, 10, fusion=-10)
        check_run(kind, dt, (70, 516), var, 6, fusion=2)
        if kind == "jacobi2d5":
            check_run(kind, dt, (70, 516), var, 6, fusion=3)
    print("ok fused", kind, flush=True)

# the paper-literal family (fp32 / int32)
for kind in ("jacobi2d5", "gameoflife", "laplacian3d7", "wave13pt", "gradient", "tricubic"):
    dt = "i32" if kind == "gameoflife" else "f32"
    shape = (37, 260) if kind in KINDS2 else (9, 35, 132)
    for var in (PAPER if not a.quick else ["paper_ptxasw", "paper_original"]):
        if var in ("paper_noload", "paper_nocorner"):
            # ablations are invalid at warp edges by design: launch only
            st = Stencil(kind, shape[::-1], dt, variant=var)
            ar, bufs = bufs_of(kind, dt, shape, 5)
            gb = [guarded(b) for b in bufs]
            st.run([v for v, _ in gb], 1)
            torch.cuda.synchronize()
            check_guards([w for _, w in gb], f"{kind} {var}")
            st.close()
        else:
            check_run(kind, dt, shape, var, 2)
    print("ok paper", kind, flush=True)

print(f"sanitize_run: {n_checked} oracle-checked runs OK")
