"""The paper-literal variant family (kpaper.cuh) on the GPU.

ORIGINAL (all loads), PTXASW (Listing 6 code shape) and UNIFORM (warp-uniform
branch) must equal the oracle within tolerance and the register-cache SHUFFLE
kernel bit for bit — shuffles move bits unchanged (SPEC.md
warp-sim "Shuffle bit-transparency").  The ablations are intentionally
invalid: NOCORNER is exact on every lane that has a
shuffle source inside a complete warp and wrong at the warp edges; NOLOAD
differs.  Widths leave the last warp of each row incomplete (the paper's
%incomplete case).
"""
import numpy as np
import pytest

from paper_2301_11389_b200 import inputs
from parity import assert_parity, gpu_step

pytestmark = pytest.mark.gpu

CASES = [("jacobi2d5", "f32", 1), ("jacobi2d9", "f32", 1), ("gaussblur5x5", "f32", 2),
         ("gameoflife", "i32", 1)]
SHAPES = [(9, 36), (17, 132), (6, 516), (5, 1060)]     # nx - 2R not a multiple of 32


@pytest.mark.parametrize("kind,dtype,r", CASES)
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_valid_paper_variants_match(oracle, kind, dtype, r, shape):
    f = inputs.generate_np(shape, dtype, inputs.BASE_SEED + 21)
    ref = np.zeros_like(f)
    oracle.step(kind, dtype, [f], [ref])
    (rc,) = gpu_step(kind, dtype, [f], 1, variant="shuffle")
    sl = (slice(r, -r), slice(r, -r))
    for var in ("paper_original", "paper_ptxasw", "paper_uniform"):
        (g,) = gpu_step(kind, dtype, [f], 1, variant=var)
        assert_parity(g[sl], ref[sl], dtype, f"{kind} {var} {shape}")
        assert np.array_equal(g.view(np.uint8), rc.view(np.uint8)), f"{var} != register-cache SHUFFLE"


@pytest.mark.parametrize("kind,dtype,r", CASES)
def test_ablations_are_invalid_only_at_corners(kind, dtype, r):
    shape = (12, 264 if r == 1 else 268)     # 8 complete warps + one incomplete (6/8 lanes) per row
    f = inputs.generate_np(shape, dtype, inputs.BASE_SEED + 22)
    (good,) = gpu_step(kind, dtype, [f], 1, variant="paper_original")
    (nc,) = gpu_step(kind, dtype, [f], 1, variant="paper_nocorner")
    (nl,) = gpu_step(kind, dtype, [f], 1, variant="paper_noload")
    i = np.arange(shape[1])
    lane = (i - r) % 32
    complete = (i >= r) & (i < r + 256)
    has_src = complete & (lane <= 31 - 2 * r)
    rows = slice(r, -r)
    assert np.array_equal(nc[rows][:, has_src], good[rows][:, has_src])
    assert not np.array_equal(nc[rows][:, r:-r], good[rows][:, r:-r])
    assert not np.array_equal(nl[rows][:, r:-r], good[rows][:, r:-r])


def test_paper_variants_rejected_for_3d_and_fp64():
    from paper_2301_11389_b200.binding import Stencil, StencilError
    st = Stencil("laplacian3d7", (8, 8, 8), "f32")
    with pytest.raises(StencilError):
        st.set_variant("paper_ptxasw")
    st2 = Stencil("jacobi2d9", (8, 8), "f64")
    with pytest.raises(StencilError):
        st2.set_variant("paper_original")
