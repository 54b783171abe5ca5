"""Maximum sizes: grids of more than 2^31 elements per buffer (64-bit
offsets in every kernel path), checked against the oracle on windows cut
out with their dependence cone (one step: the cone is the radius).

jacobi2d5 fp32 65536 x 32800 and laplacian3d7 fp32 1024 x 1024 x 2100 are
8.6 GB per buffer (two buffers each); the windows sit at the far end of the
arrays, where element offsets exceed 2^31, plus one at the start.
"""
import numpy as np
import pytest
import torch

from paper_2301_11389_b200 import inputs
from parity import assert_parity

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TWO31 = 1 << 31


def _check_windows(oracle, kind, dtype, f_dev, g_dev, wins, lo, hi):
    n = f_dev.shape
    for w in wins:
        sub = tuple(slice(max(0, s.start - lo), min(d, s.stop + hi)) for s, d in zip(w, n))
        f = f_dev[sub].cpu().numpy()
        ref = np.zeros_like(f)
        oracle.step(kind, dtype, [f], [ref])
        inner = tuple(slice(s.start - u.start, s.stop - u.start) for s, u in zip(w, sub))
        g = g_dev[w].cpu().numpy()
        r = ref[inner]
        # points interior to the global grid AND to the cut-out (the oracle
        # leaves the cut-out's own ring untouched)
        m = np.ones(g.shape, bool)
        for ax, (s, u, d) in enumerate(zip(w, sub, n)):
            idx = np.arange(s.start, s.stop)
            ok = (idx >= lo) & (idx < d - hi) & (idx - u.start >= lo) & (idx - u.start < (u.stop - u.start) - hi)
            shp = [1] * len(n)
            shp[ax] = -1
            m &= ok.reshape(shp)
        assert m.any()
        assert_parity(g[m], r[m], dtype, f"{kind} window {w}")


@pytest.mark.parametrize("variant", ["shuffle", "plain"])
def test_jacobi2d_beyond_2e31_elements(oracle, variant):
    from paper_2301_11389_b200.binding import Stencil
    shape = (32800, 65536)                       # (ny, nx)
    assert shape[0] * shape[1] > TWO31
    f = inputs.generate_torch(shape, "f32", inputs.BASE_SEED + 71)
    g = torch.zeros_like(f)
    st = Stencil("jacobi2d5", shape[::-1], "f32", variant=variant)
    st.step([f], [g])
    torch.cuda.synchronize()
    ny, nx = shape
    wins = [(slice(0, 8), slice(0, 300)),
            (slice(ny - 9, ny), slice(nx - 300, nx)),                  # offsets > 2^31
            (slice(ny - 40, ny - 30), slice(nx // 2 - 150, nx // 2 + 150))]
    assert (ny - 9) * nx > TWO31
    _check_windows(oracle, "jacobi2d5", "f32", f, g, wins, 1, 1)
    st.close()
    del f, g
    torch.cuda.empty_cache()


@pytest.mark.parametrize("variant", ["shuffle", "plain"])
def test_laplacian3d_beyond_2e31_elements(oracle, variant):
    from paper_2301_11389_b200.binding import Stencil
    shape = (2100, 1024, 1024)                   # (nz, ny, nx)
    assert shape[0] * shape[1] * shape[2] > TWO31
    f = inputs.generate_torch(shape, "f32", inputs.BASE_SEED + 72)
    g = torch.zeros_like(f)
    st = Stencil("laplacian3d7", shape[::-1], "f32", variant=variant)
    st.step([f], [g])
    torch.cuda.synchronize()
    nz, ny, nx = shape
    wins = [(slice(0, 4), slice(0, 6), slice(0, 140)),
            (slice(nz - 5, nz), slice(ny - 8, ny), slice(nx - 140, nx)),  # offsets > 2^31
            (slice(nz - 30, nz - 26), slice(500, 520), slice(380, 520))]
    assert (nz - 30) * ny * nx > TWO31
    _check_windows(oracle, "laplacian3d7", "f32", f, g, wins, 1, 1)
    st.close()
    del f, g
    torch.cuda.empty_cache()
