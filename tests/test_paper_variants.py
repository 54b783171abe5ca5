"""The paper-literal variant family (kpaper.cuh) on the GPU.

2-D (kpaper.cuh) and 3-D (kpaper3d.cuh) suite members.  ORIGINAL (all
loads), PTXASW (Listing 6 code shape) and UNIFORM (warp-uniform branch) must
equal the oracle within tolerance and the register-cache SHUFFLE
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
    # gaussblur: a rank-2 weight matrix, so the register-cache kernel also
    # runs the 25-tap form (rank-1 weights take the separable form,
    # DESIGN.md §5.1a, whose rounding differs from the paper's 25-term chain)
    c = list(np.linspace(0.01, 0.07, 25)) if kind == "gaussblur5x5" else None
    f = inputs.generate_np(shape, dtype, inputs.BASE_SEED + 21)
    ref = np.zeros_like(f)
    oracle.step(kind, dtype, [f], [ref], coeffs=c)
    (rc,) = gpu_step(kind, dtype, [f], 1, coeffs=c, variant="shuffle")
    sl = (slice(r, -r), slice(r, -r))
    for var in ("paper_original", "paper_ptxasw", "paper_uniform"):
        (g,) = gpu_step(kind, dtype, [f], 1, coeffs=c, variant=var)
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


CASES_3D = [("laplacian3d7", 1, 1), ("jacobi3d7", 1, 1), ("wave13pt", 2, 2), ("divergence", 1, 1),
            ("gradient", 1, 1), ("tricubic", 1, 2)]
SHAPES_3D = [(5, 6, 36), (6, 9, 132), (5, 5, 520)]    # (nz, ny, nx); rows end in an incomplete warp


@pytest.mark.parametrize("kind,lo,hi", CASES_3D)
@pytest.mark.parametrize("shape", SHAPES_3D, ids=lambda s: "x".join(map(str, s)))
def test_valid_paper_variants_3d(oracle, kind, lo, hi, shape):
    """3-D suite members (kpaper3d.cuh): ORIGINAL / PTXASW / UNIFORM equal the
    oracle; they are bit-identical to each other and, for the k3d kinds
    (same term order), to the register-cache SHUFFLE kernel."""
    ar = oracle.arity(kind)
    ins = [inputs.generate_np(shape, "f32", inputs.BASE_SEED + 23, a) for a in range(ar["n_in"])]
    refs = [np.zeros_like(ins[0]) for _ in range(ar["n_out"])]
    oracle.step(kind, "f32", ins, refs)
    sl = (slice(lo, -hi),) * 3
    rc = gpu_step(kind, "f32", ins, ar["n_out"], variant="shuffle")
    outs = {}
    for var in ("paper_original", "paper_ptxasw", "paper_uniform"):
        gs = gpu_step(kind, "f32", ins, ar["n_out"], variant=var)
        for k in range(ar["n_out"]):
            assert_parity(gs[k][sl], refs[k][sl], "f32", f"{kind} {var} {shape} out{k}")
            if kind != "tricubic":
                assert np.array_equal(gs[k].view(np.uint8), rc[k].view(np.uint8)), f"{var} != SHUFFLE"
        outs[var] = gs
    for var in ("paper_ptxasw", "paper_uniform"):
        for a, b in zip(outs[var], outs["paper_original"]):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), f"{var} != ORIGINAL"


def test_ablations_3d_laplacian():
    """NOCORNER is exact on lanes whose destinations (deltas 1, 2) have their
    source inside a complete warp and wrong at warp edges; NOLOAD differs."""
    shape = (4, 5, 260)                      # x interior 1..258: 8 complete warps + 2 lanes
    f = inputs.generate_np(shape, "f32", inputs.BASE_SEED + 24)
    (good,) = gpu_step("laplacian3d7", "f32", [f], 1, variant="paper_original")
    (nc,) = gpu_step("laplacian3d7", "f32", [f], 1, variant="paper_nocorner")
    (nl,) = gpu_step("laplacian3d7", "f32", [f], 1, variant="paper_noload")
    i = np.arange(shape[2])
    lane = (i - 1) % 32
    has_src = (i >= 1) & (i < 257) & (lane <= 29)
    inner = (slice(1, -1), slice(1, -1))
    assert np.array_equal(nc[inner][..., has_src], good[inner][..., has_src])
    assert not np.array_equal(nc[inner][..., 1:-1], good[inner][..., 1:-1])
    assert not np.array_equal(nl[inner][..., 1:-1], good[inner][..., 1:-1])


def test_paper_variants_rejected_for_fp64():
    from paper_2301_11389_b200.binding import Stencil, StencilError
    st = Stencil("laplacian3d7", (8, 8, 8), "f64")
    with pytest.raises(StencilError):
        st.set_variant("paper_ptxasw")
    st2 = Stencil("jacobi2d9", (8, 8), "f64")
    with pytest.raises(StencilError):
        st2.set_variant("paper_original")
