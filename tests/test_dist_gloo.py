"""Multi-rank slab decomposition on CPU: world_size 2 (and 3) over gloo.

Each rank builds its local slab (lo + n/N + hi planes) from the global
initial field exactly as stencil_slab_plan (the C library's host plan, the
one dist.cu executes) says, exchanges halo planes with gloo send/recv using
the plan's offsets and counts, sweeps its slab with the CPU oracle and
restores the global Dirichlet planes it owns.  The gathered owned planes
must equal the single-domain oracle run bit for bit (slab decomposition
changes no per-point arithmetic).  This is the host logic of S9; the NCCL
transport itself needs >= 2 GPUs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_from_global(g, plan, lo, axis0_n):
    """Local slab: local plane L <-> global plane own_begin - lo + L (zeros outside)."""
    loc = np.zeros((plan["local_n"],) + g.shape[1:], g.dtype)
    for L in range(plan["local_n"]):
        G = plan["own_begin"] - lo + L
        if 0 <= G < axis0_n:
            loc[L] = g[G]
    return loc


def _exchange(buf, plan, rank, world):
    """Halo exchange with the plan's offsets (same as dist.cu's NCCL group)."""
    n_lo, n_hi = plan["n_lo"], plan["n_hi"]
    reqs = []
    if plan["send_lo_from"] >= 0:       # to rank-1: my bottom n_hi owned planes
        s = torch.from_numpy(np.ascontiguousarray(buf[plan["send_lo_from"]:plan["send_lo_from"] + n_hi]))
        reqs.append(dist.isend(s, rank - 1))
    if plan["send_hi_from"] >= 0:       # to rank+1: my top n_lo owned planes
        s = torch.from_numpy(np.ascontiguousarray(buf[plan["send_hi_from"]:plan["send_hi_from"] + n_lo]))
        reqs.append(dist.isend(s, rank + 1))
    if plan["recv_lo_at"] >= 0:
        r = torch.empty((n_lo,) + buf.shape[1:], dtype=torch.from_numpy(buf[:1]).dtype)
        dist.recv(r, rank - 1)
        buf[plan["recv_lo_at"]:plan["recv_lo_at"] + n_lo] = r.numpy()
    if plan["recv_hi_at"] >= 0:
        r = torch.empty((n_hi,) + buf.shape[1:], dtype=torch.from_numpy(buf[:1]).dtype)
        dist.recv(r, rank + 1)
        buf[plan["recv_hi_at"]:plan["recv_hi_at"] + n_hi] = r.numpy()
    for q in reqs:
        q.wait()


def _worker(rank, world, port, kind, dtype, shape, n_iters, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle
        from paper_2301_11389_b200 import binding, inputs
        ar = pyoracle.arity(kind)
        lo, hi = ar["lo"], ar["hi"]
        n = shape[0]                                  # slow axis (numpy axis 0)
        plan = binding.slab_plan(n, lo, hi, rank, world)
        fields = [inputs.generate_np(shape, dtype, inputs.BASE_SEED + 11, a) for a in range(ar["n_in"])]
        loc = [_local_from_global(f, plan, lo, n) for f in fields]
        # global Dirichlet planes owned by this rank (local indices)
        keep = [L for L in range(plan["local_n"])
                if 0 <= plan["own_begin"] - lo + L < n
                and not (lo <= plan["own_begin"] - lo + L < n - hi)]
        if kind == "wave13pt":
            # Dirichlet ring of cur copied into prev and next (stencil_run / oracle_run)
            ring = np.ones(loc[1].shape, bool)
            for L in range(plan["local_n"]):
                G = plan["own_begin"] - lo + L
                if lo <= G < n - hi:
                    ring[L][tuple(slice(lo, m - hi) for m in loc[1].shape[1:])] = False
            prev = loc[0].copy()
            prev[ring] = loc[1][ring]
            bufs = [prev, loc[1], loc[1].copy()]
            p, c, nx = 0, 1, 2
            for _ in range(n_iters):
                _exchange(bufs[c], plan, rank, world)
                out = bufs[nx].copy()
                pyoracle.step(kind, dtype, [bufs[p], bufs[c]], [out])
                for L in keep:
                    out[L] = bufs[c][L]
                bufs[nx] = out
                p, c, nx = c, nx, p
            res = bufs[c]
        else:
            cur, nxt = loc[0], loc[0].copy()
            for _ in range(n_iters):
                _exchange(cur, plan, rank, world)
                out = nxt.copy()
                pyoracle.step(kind, dtype, [cur], [out])
                for L in keep:
                    out[L] = cur[L]
                cur, nxt = out, cur
            res = cur
        owned = res[lo:lo + plan["own_end"] - plan["own_begin"]]
        q.put((rank, plan["own_begin"], owned))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,dtype,shape,world", [
    ("jacobi2d9", "f64", (16, 24), 2),
    ("gaussblur5x5", "f32", (20, 36), 2),
    ("laplacian3d7", "f64", (12, 9, 10), 2),
    ("wave13pt", "f64", (12, 8, 9), 2),
    ("laplacian3d7", "f32", (15, 7, 8), 3),
])
def test_slab_decomposition_matches_single_domain(oracle, kind, dtype, shape, world):
    from paper_2301_11389_b200 import build, inputs
    build.build()
    ar = oracle.arity(kind)
    n_iters = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, dtype, shape, n_iters, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([o for _, _, o in sorted(parts, key=lambda t: t[0])], axis=0)
    fields = [inputs.generate_np(shape, dtype, inputs.BASE_SEED + 11, a) for a in range(ar["n_in"])]
    if kind == "wave13pt":
        bufs = [fields[0], fields[1], fields[1].copy()]
    else:
        bufs = [fields[0], fields[0].copy()]
    idx = oracle.run(kind, dtype, bufs, n_iters)
    assert np.array_equal(got, bufs[idx])


def test_slab_plan_fields(oracle):
    from paper_2301_11389_b200 import binding
    p = binding.slab_plan(1024, 1, 1, 0, 4)
    assert (p["own_begin"], p["own_end"], p["local_n"]) == (0, 256, 258)
    assert p["recv_lo_at"] == -1 and p["send_lo_from"] == -1
    assert (p["recv_hi_at"], p["send_hi_from"], p["n_lo"], p["n_hi"]) == (257, 256, 1, 1)
    p = binding.slab_plan(1024, 1, 2, 2, 4)
    assert (p["own_begin"], p["recv_lo_at"], p["send_lo_from"], p["recv_hi_at"], p["send_hi_from"]) == \
        (512, 0, 1, 257, 256)
    p = binding.slab_plan(1024, 2, 2, 3, 4)
    assert p["recv_hi_at"] == -1 and p["send_hi_from"] == -1 and p["local_n"] == 260
    with pytest.raises(Exception):
        binding.slab_plan(1023, 1, 1, 0, 4)        # not divisible
    with pytest.raises(Exception):
        binding.slab_plan(8, 2, 2, 0, 8)           # slab thinner than the halo
