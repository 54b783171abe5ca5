"""Parity helpers: run the CUDA path (through the C ABI) and the CPU oracle on
the same seeded inputs and compare them element by element.

Tolerance: integer kinds bit-exact; floating point passes iff
for every compared point p

    |g_p - r_p| <= tol * max(|r_p|, S),   S = mean |r| over the compared points,

with tol = 1e-5 (fp32) / 1e-12 (fp64) — BASELINE.json north_star's relative
error bound, with the floor S for outputs that cancel to ~0 (reading R13).
"""
from __future__ import annotations

import numpy as np

TOL = {"f32": 1e-5, "f64": 1e-12}
NP = {"f32": np.float32, "f64": np.float64, "i32": np.int32}


def assert_parity(g: np.ndarray, r: np.ndarray, dtype: str, what: str = ""):
    assert g.shape == r.shape, (g.shape, r.shape)
    if dtype == "i32":
        bad = np.argwhere(g != r)
        assert bad.size == 0, f"{what}: {len(bad)} integer mismatches, first at {bad[:5].tolist()}"
        return
    g64, r64 = g.astype(np.float64), r.astype(np.float64)
    assert np.all(np.isfinite(g64)), f"{what}: non-finite GPU output"
    S = float(np.mean(np.abs(r64))) if r64.size else 0.0
    lim = TOL[dtype] * np.maximum(np.abs(r64), S)
    err = np.abs(g64 - r64)
    bad = err > lim
    if bad.any():
        idx = np.argwhere(bad)[:5].tolist()
        worst = float(np.max(err / np.maximum(lim, 1e-300)))
        raise AssertionError(f"{what}: {int(bad.sum())} points beyond tolerance "
                             f"(worst {worst:.3g}x the bound) e.g. {idx}")


def interior(shape, lo, hi):
    return tuple(slice(lo, n - hi) for n in shape)


def ring_mask(shape, lo, hi):
    m = np.ones(shape, bool)
    m[interior(shape, lo, hi)] = False
    return m


# ------------------------------------------------------------- GPU side
def to_dev(a: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_step(kind, dtype, ins, n_out, coeffs=None, variant="shuffle", fill=0):
    """One stencil_step; returns the output arrays (boundary left at `fill`)."""
    import torch
    from paper_2301_11389_b200.binding import Stencil
    dims = ins[0].shape[::-1]
    st = Stencil(kind, dims, dtype, coeffs=coeffs, variant=variant)
    dins = [to_dev(a) for a in ins]
    douts = [torch.full_like(dins[0], fill) for _ in range(n_out)]
    st.step(dins, douts)
    torch.cuda.synchronize()
    res = [d.cpu().numpy() for d in douts]
    st.close()
    return res


def gpu_run(kind, dtype, bufs, n_iters, coeffs=None, variant="shuffle"):
    """stencil_run over copies of `bufs`; returns (result index, all buffers)."""
    import torch
    from paper_2301_11389_b200.binding import Stencil
    dims = bufs[0].shape[::-1]
    st = Stencil(kind, dims, dtype, coeffs=coeffs, variant=variant)
    dbufs = [to_dev(a) for a in bufs]
    idx = st.run(dbufs, n_iters)
    torch.cuda.synchronize()
    res = [d.cpu().numpy() for d in dbufs]
    st.close()
    return idx, res


# ---------------------------------------------------------- oracle side
def oracle_window_run(oracle, kind, dtype, fields, n_iters, window, radius, coeffs=None,
                      nthreads=1):
    """Oracle result of `n_iters` sweeps restricted to `window` (tuple of
    slices, numpy axis order) of the full-grid run, computed on the
    dependence cone only: the window grown by (n_iters+1)*radius, clipped to
    the grid.  Cells of the cut-out's outer ring that are not on the global
    boundary are stale after sweep 1, and staleness advances `radius` cells
    per sweep, so after n sweeps it stays more than n*radius cells away from
    the window.  `fields` are the run buffers' initial contents (current
    field(s) first, as stencil_run expects)."""
    grow = (n_iters + 1) * radius
    sub, inner = [], []
    for sl, n in zip(window, fields[0].shape):
        a, b = max(0, sl.start - grow), min(n, sl.stop + grow)
        sub.append(slice(a, b))
        inner.append(slice(sl.start - a, sl.stop - a))
    bufs = [np.ascontiguousarray(f[tuple(sub)]) for f in fields]
    idx = oracle.run(kind, dtype, bufs, n_iters, coeffs=coeffs, nthreads=nthreads)
    return bufs[idx][tuple(inner)]
