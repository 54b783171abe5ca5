"""N ranks emulated on one GPU: the slab decomposition of S9 with device copies
standing in for NCCL.

Every rank holds lo + n/N + hi planes (stencil_slab_plan); each sweep
copies the halo planes between the ranks' device buffers with the plan's
offsets and counts, then runs stencil_step_range on the rank's owned
interior planes — the same kernels and plane ranges dist.cu launches around
its NCCL group.  Result must equal the single-GPU stencil_run bit for bit.
"""
import numpy as np
import pytest
import torch

from paper_2301_11389_b200 import inputs

pytestmark = pytest.mark.gpu


def _run_fake(kind, dtype, shape, world, n_iters, variant="shuffle"):
    from paper_2301_11389_b200.binding import Stencil, slab_plan
    from oracle import pyoracle
    ar = pyoracle.arity(kind)
    lo, hi = ar["lo"], ar["hi"]
    n = shape[0]
    m = n // world
    fields = [inputs.generate_torch(shape, dtype, inputs.BASE_SEED + 13, a) for a in range(ar["n_in"])]
    plans = [slab_plan(n, lo, hi, r, world) for r in range(world)]
    ranks = []
    for r, p in enumerate(plans):
        loc = []
        for f in fields:
            t = torch.zeros((p["local_n"],) + tuple(shape[1:]), dtype=f.dtype, device="cuda")
            for L in range(p["local_n"]):
                G = p["own_begin"] - lo + L
                if 0 <= G < n:
                    t[L] = f[G]
            loc.append(t)
        st = Stencil(kind, tuple(shape[1:][::-1]) + (p["local_n"],) if len(shape) == 3
                     else (shape[1], p["local_n"]), dtype, variant=variant)
        a = max(p["own_begin"], lo) - p["own_begin"] + lo
        b = min(p["own_end"], n - hi) - p["own_begin"] + lo
        if kind == "wave13pt":
            bufs = [loc[0], loc[1], loc[1].clone()]
        else:
            bufs = [loc[0], loc[0].clone()]
        ranks.append(dict(st=st, plan=p, bufs=bufs, a=a, b=b))
    # Dirichlet ring of the current field into the other buffers (as stencil_run)
    for rk in ranks:
        if kind == "wave13pt":
            cur = rk["bufs"][1]
            ring = torch.ones_like(cur, dtype=torch.bool)
            p = rk["plan"]
            for L in range(p["local_n"]):
                if lo <= p["own_begin"] - lo + L < n - hi:
                    ring[L][tuple(slice(lo, s - hi) for s in shape[1:])] = False
            rk["bufs"][0][ring] = cur[ring]
    cur_i, nxt_i, prv_i = (1, 2, 0) if kind == "wave13pt" else (0, 1, None)
    for _ in range(n_iters):
        for r, rk in enumerate(ranks):                     # halo exchange (device copies)
            p = rk["plan"]
            buf = rk["bufs"][cur_i]
            if p["recv_lo_at"] >= 0:
                q = ranks[r - 1]
                src = q["bufs"][cur_i]
                buf[p["recv_lo_at"]:p["recv_lo_at"] + p["n_lo"]] = \
                    src[q["plan"]["send_hi_from"]:q["plan"]["send_hi_from"] + p["n_lo"]]
            if p["recv_hi_at"] >= 0:
                q = ranks[r + 1]
                src = q["bufs"][cur_i]
                buf[p["recv_hi_at"]:p["recv_hi_at"] + p["n_hi"]] = \
                    src[q["plan"]["send_lo_from"]:q["plan"]["send_lo_from"] + p["n_hi"]]
        for rk in ranks:
            bf = rk["bufs"]
            if kind == "wave13pt":
                rk["st"].step_range([bf[prv_i], bf[cur_i]], [bf[nxt_i]], rk["a"], rk["b"])
            else:
                rk["st"].step_range([bf[cur_i]], [bf[nxt_i]], rk["a"], rk["b"])
        if kind == "wave13pt":
            prv_i, cur_i, nxt_i = cur_i, nxt_i, prv_i
        else:
            cur_i, nxt_i = nxt_i, cur_i
    torch.cuda.synchronize()
    out = torch.cat([rk["bufs"][cur_i][lo:lo + m] for rk in ranks], 0)
    for rk in ranks:
        rk["st"].close()
    return fields, out


@pytest.mark.parametrize("kind,dtype,shape,world", [
    ("gaussblur5x5", "f32", (64, 260), 4),
    ("jacobi2d9", "f64", (48, 130), 3),
    ("laplacian3d7", "f64", (32, 45, 130), 2),
    ("jacobi3d7", "f32", (40, 33, 132), 4),
    ("wave13pt", "f64", (24, 20, 66), 2),
])
def test_fake_ranks_equal_single_gpu(kind, dtype, shape, world):
    from paper_2301_11389_b200.binding import Stencil
    fields, got = _run_fake(kind, dtype, shape, world, 6)
    st = Stencil(kind, tuple(shape[::-1]), dtype)
    if kind == "wave13pt":
        bufs = [fields[0].clone(), fields[1].clone(), torch.zeros_like(fields[0])]
    else:
        bufs = [fields[0].clone(), torch.zeros_like(fields[0])]
    idx = st.run(bufs, 6)
    torch.cuda.synchronize()
    assert torch.equal(got, bufs[idx])
    st.close()
