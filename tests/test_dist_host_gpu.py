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
equal the single-GPU run bit for bit.  (NCCL refuses two ranks on one GPU;
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


def _rank(rank, world, port, kind, dtype, dims, n_iters, q, transport="host", runs=1):
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
                if 0 <= G < n:
                    out[L] = t[G]
            return out

        loc = [slab(f) for f in fields]
        if n_bufs == 2:
            bufs = [loc[0], torch.zeros_like(loc[0])]
        elif kind == "wave13pt":
            bufs = [loc[0], loc[1], torch.zeros_like(loc[0])]
        else:
            bufs = loc + [torch.zeros_like(loc[0]) for _ in range(n_out)]
        if transport == "p2p":
            st.p2p_register(bufs, _allgather)
        for _ in range(runs - 1):          # consecutive runs on the same buffers (epochs carry over)
            st.run(bufs, n_iters)
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
                ref.run(rb, n_iters)
            ridx = ref.run(rb, n_iters)
            torch.cuda.synchronize()
            ok = True
            for k in range(nres):
                got = torch.cat([parts[r][k] for r in range(world)], 0)
                exp = rb[ridx + k].cpu()
                # compare the interior of the slow axis (the global ring planes are held)
                ok = ok and torch.equal(got[lo:n - hi], exp[lo:n - hi])
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
def test_two_processes_one_gpu_equal_single(kind, dtype, dims, world, transport):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, kind, dtype, dims, 4, q, transport, 2))
             for r in range(world)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
