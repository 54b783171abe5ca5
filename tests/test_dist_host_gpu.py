"""The attached multi-rank paths for real: two (three) processes on one GPU.

transport "p2p": stencil_dist_attach_p2p — the fused peer-store halo
exchange (CUDA IPC peer pointers, epoch flags with stream memory
operations), the path that moves halos without any copy kernel or NCCL.

Each process is one rank of a world-size-2 gloo group; the stencil handle is
attached with stencil_dist_attach_host, whose exchange callback moves the
halo planes with torch.distributed send/recv.  Everything of the multi-GPU
step except the NCCL calls runs: the slab layout, the plan's offsets, the
interior / halo-slab launches, the slab ring copy of stencil_run, the owned
interior point count.  The ranks' owned planes, gathered on rank 0, must
equal the single-GPU run bit for bit and the CPU oracle's run of the same
global fields within the DESIGN.md §7 tolerance.  Every case also runs with
the local buffers' halo planes (and, for p2p, the other run buffers)
starting as NaN garbage instead of the global field's planes: the exchange
alone must fill them (the p2p ring copy used to run before the
prologue exchange and carried the caller's halo contents into the x-edge
cells of the other buffer).  (NCCL refuses two ranks on one GPU;
the NCCL transport shares all of this code but its calls need >= 2 GPUs.)
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(peer, send, recv):
    req = dist.isend(torch.from_numpy(send), peer)
    dist.recv(torch.from_numpy(recv), peer)
    req.wait()


def _allgather(blob):
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, blob)
    return parts


def _rank(rank, world, port, kind, dtype, dims, n_iters, q, transport="host", runs=1, halo="global"):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2301_11389_b200 import inputs
        from paper_2301_11389_b200.binding import Stencil
        st = Stencil(kind, dims, dtype)
        if transport == "host":
            st.attach_host(rank, world, _exchange)
        else:
            st.attach_p2p(rank, world)
        info = st.info()
        n_in, n_out, n_bufs = st.arity()
        lo, hi = info["lo"], info["hi"]
        shape = tuple(dims[::-1])
        n = shape[0]
        m = n // world
        local_n = info["local_dims"][len(dims) - 1]
        assert local_n == m + lo + hi
        fields = [inputs.generate_torch(shape, dtype, inputs.BASE_SEED + 19, a) for a in range(n_in)]

        def slab(t):
            out = torch.zeros((local_n,) + shape[1:], dtype=t.dtype, device="cuda")
            for L in range(local_n):
                G = rank * m - lo + L
                owned = lo <= L < lo + m
                if 0 <= G < n and (owned or halo == "global"):
                    out[L] = t[G]
                elif halo == "garbage":
                    out[L] = float("nan")
            return out

        def other():
            return torch.full((local_n,) + shape[1:], float("nan") if halo == "garbage" else 0.0,
                              dtype=fields[0].dtype, device="cuda")

        loc = [slab(f) for f in fields]
        if n_bufs == 2:
            bufs = [loc[0], other()]
        elif kind == "wave13pt":
            bufs = [loc[0], loc[1], other()]
        else:
            bufs = loc + [other() for _ in range(n_out)]
        if transport == "p2p":
            st.p2p_register(bufs, _allgather)
        for _ in range(runs - 1):          # consecutive runs on the same buffers (epochs carry over)
            i = st.run(bufs, n_iters)
            if n_bufs == 2:                  # attached runs are single sweeps: no rotation needed
                assert i == n_iters % 2
        idx = st.run(bufs, n_iters)
        torch.cuda.synchronize()
        nres = n_out if n_bufs > 3 else 1
        owned = [bufs[idx + k][lo:lo + m].cpu() for k in range(nres)]
        parts = [None] * world
        dist.all_gather_object(parts, owned)
        if rank == 0:
            ref = Stencil(kind, dims, dtype)
            if n_bufs == 2:
                rb = [fields[0].clone(), torch.zeros_like(fields[0])]
            elif kind == "wave13pt":
                rb = [fields[0].clone(), fields[1].clone(), torch.zeros_like(fields[0])]
            else:
                rb = [f.clone() for f in fields] + [torch.zeros_like(fields[0]) for _ in range(n_out)]
            for _ in range(runs - 1):
                i = ref.run(rb, n_iters)
                if n_bufs == 2 and i == 1:   # a fused 1-GPU run may end in bufs[1] (stencil.h)
                    rb = [rb[1], rb[0]]
            ridx = ref.run(rb, n_iters)
            torch.cuda.synchronize()
            # the CPU oracle on the same global fields
            from oracle import pyoracle
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from parity import assert_parity
            pyoracle.build()
            npf = [f.cpu().numpy() for f in fields]
            if n_bufs == 2:
                ob = [npf[0].copy(), np.zeros_like(npf[0])]
            elif kind == "wave13pt":
                ob = [npf[0].copy(), npf[1].copy(), np.zeros_like(npf[0])]
            else:
                ob = [a.copy() for a in npf] + [np.zeros_like(npf[0]) for _ in range(n_out)]
            oidx = 0
            for _ in range(runs):
                oidx = pyoracle.run(kind, dtype, ob, n_iters)
            ok = True
            for k in range(nres):
                got = torch.cat([parts[r][k] for r in range(world)], 0)
                exp = rb[ridx + k].cpu()
                # compare interior points (the global ring is held; the ring of a
                # non-iterable kind's output is never written and may be garbage)
                sl = tuple(slice(lo, e - hi) for e in shape)
                ok = ok and torch.equal(got[sl], exp[sl])
                try:
                    assert_parity(got.numpy()[sl], ob[oidx + k][sl], dtype, f"{kind} rank-gathered vs oracle")
                except AssertionError as err:
                    print(err, flush=True)
                    ok = False
            q.put(ok)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,dtype,dims,world", [
    ("jacobi3d7", "f32", (132, 20, 24), 2),
    ("wave13pt", "f64", (66, 18, 16), 2),
    ("gaussblur5x5", "f32", (260, 48), 2),
    ("laplacian3d7", "f64", (66, 16, 30), 3),
    ("divergence", "f32", (132, 12, 16), 2),
    ("tricubic", "f32", (132, 20, 16), 2),
])
@pytest.mark.parametrize("transport", ["host", "p2p"])
@pytest.mark.parametrize("halo", ["global", "garbage"])
def test_two_processes_one_gpu_equal_single(kind, dtype, dims, world, transport, halo):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, kind, dtype, dims, 4, q, transport, 2, halo))
             for r in range(world)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
