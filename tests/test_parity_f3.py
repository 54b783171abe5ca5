"""GPU parity of the SURVEY §8(f) row-f3 kernels (csrc/kf3.cuh; tricubic2 on
the tricubic kernels) against the CPU oracle, through the C ABI.

Sizes that span several warp tiles (128 fp32 / 64 fp64 columns), CTA row
groups (8 rows), z chunks (16 planes) and ragged tails; the minimum grids;
SHUFFLE == PLAIN bit for bit; runs; closed forms on the device; and the
paper's problem sizes (uxx1 512x512x1024, whispering
8192x16384, lapgsrb 512x1024x1024) on dependence-cone windows in the launch
configuration bench.py times.
"""
import zlib

import numpy as np
import pytest
import torch

from paper_2301_11389_b200 import inputs
from parity import assert_parity, gpu_run, gpu_step, interior, oracle_window_run, ring_mask

pytestmark = pytest.mark.gpu

SHAPES3 = {  # (nz, ny, nx)
    "f32": [(4, 4, 4), (5, 6, 8), (7, 11, 36), (19, 13, 132), (21, 18, 260), (5, 9, 516)],
    "f64": [(4, 4, 4), (6, 5, 6), (9, 10, 66), (18, 12, 130)],
}
SHAPES2 = {  # (ny, nx)
    "f32": [(3, 4), (5, 8), (29, 36), (70, 132), (41, 1028), (9, 2052)],
    "f64": [(3, 4), (6, 6), (45, 66), (37, 258)],
}
# lapgsrb's kernel (klap2.cuh) tiles 30 output rows per CTA: several row
# tiles with ragged tails, and z extents the one-wave grid splits into parts
LAP_SHAPES = {"f32": [(11, 67, 260), (40, 33, 516), (3, 95, 132)], "f64": [(9, 64, 130), (33, 31, 66)]}
COEFFS = {"uxx1": [0.3, 1.2, -0.07], "lapgsrb": [0.15]}


def seed_of(*key):
    return inputs.BASE_SEED + zlib.crc32(repr(key).encode()) % 1000


def cases():
    for kind in ("tricubic2", "uxx1", "lapgsrb", "whispering"):
        need = 4 if kind in ("tricubic2", "uxx1") else 3
        for dt in ("f32", "f64"):
            extra = LAP_SHAPES[dt] if kind == "lapgsrb" else []
            for shape in (SHAPES2 if kind == "whispering" else SHAPES3)[dt] + extra:
                if min(shape) >= need:
                    yield kind, dt, shape


@pytest.mark.parametrize("kind,dtype,shape", list(cases()),
                         ids=lambda v: v if isinstance(v, str) else "x".join(map(str, v)))
@pytest.mark.parametrize("coeffs", ["default", "distinct"])
def test_step_parity_and_variants(oracle, kind, dtype, shape, coeffs):
    if coeffs == "distinct" and kind not in COEFFS:
        pytest.skip("kind takes no coefficients")
    c = COEFFS.get(kind) if coeffs == "distinct" else None
    ar = oracle.arity(kind)
    ins = [inputs.generate_np(shape, dtype, seed_of(kind, dtype, shape), a) for a in range(ar["n_in"])]
    refs = [np.zeros_like(ins[0]) for _ in range(ar["n_out"])]
    oracle.step(kind, dtype, ins, refs, coeffs=c)
    sl = interior(shape, ar["lo"], ar["hi"])
    outs = {}
    for var in ("shuffle", "plain"):
        gs = gpu_step(kind, dtype, ins, ar["n_out"], coeffs=c, variant=var, fill=0)
        for k, (g, r) in enumerate(zip(gs, refs)):
            assert_parity(g[sl], r[sl], dtype, f"{kind} {dtype} {shape} {var} out{k}")
            assert np.all(g[ring_mask(shape, ar["lo"], ar["hi"])] == 0), "boundary ring written"
        outs[var] = gs
    for a, b in zip(outs["shuffle"], outs["plain"]):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), "SHUFFLE and PLAIN differ"


@pytest.mark.parametrize("kind,dtype,shape", [
    ("lapgsrb", "f32", (21, 18, 260)), ("lapgsrb", "f64", (9, 10, 66)), ("lapgsrb", "f32", (11, 67, 260)),
    ("uxx1", "f32", (19, 13, 132)), ("whispering", "f32", (70, 132)), ("tricubic2", "f32", (19, 13, 132))])
def test_run_parity(oracle, kind, dtype, shape):
    """stencil_run: lapgsrb ping-pongs (Dirichlet ring held), the others
    re-apply the step; the result index equals the oracle's."""
    ar = oracle.arity(kind)
    ins = [inputs.generate_np(shape, dtype, inputs.BASE_SEED + 41, a) for a in range(ar["n_in"])]
    if ar["n_bufs"] == 2:
        bufs = [ins[0], np.zeros_like(ins[0])]
    else:
        bufs = ins + [np.zeros_like(ins[0]) for _ in range(ar["n_out"])]
    ob = [b.copy() for b in bufs]
    ridx = oracle.run(kind, dtype, ob, 5)
    for var in ("shuffle", "plain"):
        gidx, gb = gpu_run(kind, dtype, [b.copy() for b in bufs], 5, variant=var)
        assert gidx == ridx
        for k in range(ar["n_out"] if ar["n_bufs"] > 2 else 1):
            assert_parity(gb[gidx + k], ob[ridx + k], dtype, f"{kind} run {var} out{k}")


def test_lapgsrb_checkerboard_on_gpu():
    """u = (-1)^(i+j+k), w = 1/8: red points -> -6w, black -> -36 w^2 exactly
    away from the boundary (the oracle pin, on the device)."""
    shape = (12, 13, 132)
    k, j, i = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    u = ((-1.0) ** (i + j + k)).astype(np.float32)
    (g,) = gpu_step("lapgsrb", "f32", [u], 1, coeffs=[0.125])
    red = ((i + j + k) % 2) == 0
    deep = (i >= 2) & (i <= shape[2] - 3) & (j >= 2) & (j <= shape[1] - 3) & (k >= 2) & (k <= shape[0] - 3)
    assert np.all(g[deep & red] == -0.75) and np.all(g[deep & ~red] == -36 / 64)


def test_whispering_quadratic_on_gpu():
    """Ez = i^2 + j^2, H = 0, da = 1, db = 1/4, cb = 1/2: Ez' = Ez + 2 * 2 * 1/8."""
    shape = (40, 260)
    j, i = np.meshgrid(np.arange(shape[0], dtype=np.float32), np.arange(shape[1], dtype=np.float32),
                       indexing="ij")
    z, one = np.zeros(shape, np.float32), np.ones(shape, np.float32)
    outs = gpu_step("whispering", "f32", [z, z, i * i + j * j, one, one / 4, one, one / 4, one / 2], 3)
    np.testing.assert_array_equal(outs[2][1:-1, 1:-1], (i * i + j * j)[1:-1, 1:-1] + 0.5)


def test_uxx1_cubic_on_gpu():
    """xx = i^3, d1 = 1: out = u1 + dth * 3 (i - 1/2)^2 (the 4th-order stagger
    is exact on cubics); fp64, 1e-12."""
    shape = (6, 7, 66)
    k, j, i = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")
    z = np.zeros(shape)
    (g,) = gpu_step("uxx1", "f64", [j.copy(), np.ones(shape), i ** 3, z, z], 1)
    exp = j + 0.25 * 3 * (i - 0.5) ** 2
    np.testing.assert_allclose(g[2:-1, 2:-1, 2:-1], exp[2:-1, 2:-1, 2:-1], rtol=1e-12)


def test_f3_kinds_reject_attach_and_paper_variants():
    from paper_2301_11389_b200.binding import Stencil, StencilError
    for kind, dims in (("uxx1", (8, 8, 8)), ("whispering", (8, 8)), ("lapgsrb", (8, 8, 8)),
                       ("tricubic2", (8, 8, 8))):
        st = Stencil(kind, dims, "f32")
        with pytest.raises(StencilError) as e:
            st.set_variant("paper_ptxasw")
        assert e.value.code == -2
        with pytest.raises(StencilError) as e:
            st.attach_p2p(0, 2)
        assert e.value.code == -2
        st.close()


# ------------------------------------------------- the paper's problem sizes
def _windows3(shape):
    nz, ny, nx = shape
    return [(slice(0, 8), slice(0, 8), slice(0, 40)),
            (slice(nz // 2, nz // 2 + 8), slice(ny // 3, ny // 3 + 10), slice(nx - 70, nx - 6)),
            (slice(nz - 8, nz), slice(ny - 9, ny), slice(nx - 40, nx))]


def _check_windows(oracle, kind, dtype, dev_in, dev_out, n_iters, radius, windows, coeffs=None):
    ar = oracle.arity(kind)
    shape = tuple(dev_in[0].shape)
    grow = (n_iters + 1) * radius
    for w in windows:
        # cut-outs start at even indices: lapgsrb's colour is (i+j+k) & 1 of the
        # oracle's local indices, which then equals the global colour
        sub = tuple(slice(max(0, s.start - grow) & ~1, min(n, s.stop + grow)) for s, n in zip(w, shape))
        fields = [t[sub].cpu().numpy() for t in dev_in]
        inner = tuple(slice(s.start - u.start, s.stop - u.start) for s, u in zip(w, sub))
        if ar["n_bufs"] == 2:                                   # iterable: dependence cone
            full_w = tuple(slice(0, u.stop - u.start) for u in sub)
            ref = oracle_window_run(oracle, kind, dtype, [fields[0], np.zeros_like(fields[0])], n_iters,
                                    full_w, radius, coeffs=coeffs, nthreads=8)
            refs = [ref[inner]]
        else:                                                   # one step on the cut-out
            outs = [np.zeros_like(fields[0]) for _ in range(ar["n_out"])]
            oracle.step(kind, dtype, fields, outs, coeffs=coeffs, nthreads=8)
            refs = [o[inner] for o in outs]
        # compare the points that are interior both globally and in the cut-out
        gidx = [np.arange(s.start, s.stop) for s in w]
        m = np.ones(tuple(len(g) for g in gidx), bool)
        for ax, (g, u, n) in enumerate(zip(gidx, sub, shape)):
            ok = (g >= ar["lo"]) & (g < n - ar["hi"]) & (g - u.start >= ar["lo"]) & (g - u.start < u.stop - u.start - ar["hi"])
            sh = [1] * len(shape)
            sh[ax] = len(g)
            m &= ok.reshape(sh)
        for k, r in enumerate(refs):
            got = dev_out[k][w].cpu().numpy()
            assert_parity(got[m], r[m], dtype, f"{kind} out{k} window {w}")


@pytest.mark.slow
@pytest.mark.parametrize("variant", ["shuffle", "plain"])
def test_uxx1_paper_size_windows(oracle, variant):
    from paper_2301_11389_b200.binding import Stencil
    dims = (512, 512, 1024)
    shape = dims[::-1]
    ins = [inputs.generate_torch(shape, "f32", inputs.BASE_SEED + 6, a) for a in range(5)]
    out = torch.zeros_like(ins[0])
    st = Stencil("uxx1", dims, "f32", variant=variant)
    st.step(ins, [out])
    torch.cuda.synchronize()
    _check_windows(oracle, "uxx1", "f32", ins, [out], 1, 2, _windows3(shape))
    st.close()


@pytest.mark.slow
@pytest.mark.parametrize("variant", ["shuffle", "plain"])
def test_whispering_paper_size_windows(oracle, variant):
    from paper_2301_11389_b200.binding import Stencil
    dims = (8192, 16384)
    shape = dims[::-1]
    ins = [inputs.generate_torch(shape, "f32", inputs.BASE_SEED + 7, a) for a in range(8)]
    outs = [torch.zeros_like(ins[0]) for _ in range(3)]
    st = Stencil("whispering", dims, "f32", variant=variant)
    st.step(ins, outs)
    torch.cuda.synchronize()
    ny, nx = shape
    wins = [(slice(0, 40), slice(0, 300)), (slice(ny // 2, ny // 2 + 33), slice(nx // 3, nx // 3 + 260)),
            (slice(ny - 40, ny), slice(nx - 300, nx)), (slice(31, 34), slice(8000, 8192))]
    _check_windows(oracle, "whispering", "f32", ins, outs, 1, 1, wins)
    st.close()


@pytest.mark.slow
@pytest.mark.parametrize("variant", ["shuffle", "plain"])
def test_lapgsrb_paper_size_x10_windows(oracle, variant):
    """512x1024x1024 (nx, ny, nz) fp32, 10 iterations: each iteration reaches
    two cells (red then black), so the dependence cone grows by 2 per sweep."""
    from paper_2301_11389_b200.binding import Stencil
    dims = (512, 1024, 1024)
    shape = dims[::-1]
    f = inputs.generate_torch(shape, "f32", inputs.BASE_SEED + 8)
    bufs = [f.clone(), torch.zeros_like(f)]
    st = Stencil("lapgsrb", dims, "f32", variant=variant)
    idx = st.run(bufs, 10)
    torch.cuda.synchronize()
    res = bufs[idx]
    del bufs
    _check_windows(oracle, "lapgsrb", "f32", [f], [res], 10, 2, _windows3(shape))
    st.close()


@pytest.mark.slow
def test_tricubic2_256_samples(oracle):
    from paper_2301_11389_b200.binding import Stencil
    n = 256
    shape = (n, n, n)
    ins = [inputs.generate_torch(shape, "f32", inputs.BASE_SEED + 9, a) for a in range(4)]
    out = torch.zeros_like(ins[0])
    st = Stencil("tricubic2", shape, "f32")
    st.step(ins, [out])
    torch.cuda.synchronize()
    _check_windows(oracle, "tricubic2", "f32", ins, [out], 1, 2, _windows3(shape))
    st.close()
