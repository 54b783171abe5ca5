"""The NCCL-attached path on one GPU (a group of one rank).

stencil_dist_attach with nranks = 1 runs everything the multi-GPU step runs
(libnccl.so.2 dlopen, ncclCommInitRank, the grouped send/recv issue with no
peer, the comm-stream events, the interior/halo slab launches, the slab
ring copy) except the transfers themselves.  Its local buffers have the slab
layout (lo dead planes + n planes + hi dead planes); results must equal the
unattached single-GPU run bit for bit.
"""
import numpy as np
import pytest
import torch

from paper_2301_11389_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,dtype,dims", [
    ("jacobi3d7", "f32", (132, 40, 24)),
    ("wave13pt", "f64", (66, 20, 16)),
    ("gaussblur5x5", "f32", (260, 48)),
])
def test_attached_single_rank_equals_unattached(kind, dtype, dims):
    from oracle import pyoracle
    from paper_2301_11389_b200.binding import Stencil, dist_get_id
    ar = pyoracle.arity(kind)
    lo, hi = ar["lo"], ar["hi"]
    shape = tuple(dims[::-1])
    fields = [inputs.generate_torch(shape, dtype, inputs.BASE_SEED + 17, a) for a in range(ar["n_in"])]

    ref = Stencil(kind, dims, dtype)
    rb = ([fields[0].clone(), fields[1].clone(), torch.zeros_like(fields[0])] if kind == "wave13pt"
          else [fields[0].clone(), torch.zeros_like(fields[0])])
    ridx = ref.run(rb, 5)

    st = Stencil(kind, dims, dtype)
    st.attach(dist_get_id(), 0, 1)
    info = st.info()
    n = shape[0]
    assert info["nranks"] == 1 and info["local_dims"][len(dims) - 1] == n + lo + hi
    assert info["interior_points"] == ref.info()["interior_points"]

    def pad(t):
        out = torch.zeros((n + lo + hi,) + shape[1:], dtype=t.dtype, device="cuda")
        out[lo:lo + n] = t
        return out

    lb = ([pad(fields[0]), pad(fields[1]), torch.zeros((n + lo + hi,) + shape[1:], dtype=fields[0].dtype,
                                                        device="cuda")] if kind == "wave13pt"
          else [pad(fields[0]), torch.zeros((n + lo + hi,) + shape[1:], dtype=fields[0].dtype,
                                            device="cuda")])
    idx = st.run(lb, 5)
    torch.cuda.synchronize()
    assert idx == ridx
    assert torch.equal(lb[idx][lo:lo + n], rb[ridx])
    st.close()
    ref.close()
