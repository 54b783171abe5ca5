"""GPU parity of the 3-D kernels (TMA plane ring) against the CPU oracle.

Small grids spanning several x-tiles (128 fp32 / 64 fp64), several CTA row
tiles (8 rows), ragged tails in every axis and the minimum grids; SHUFFLE vs
PLAIN bit identity; runs (ping-pong, the wave13pt 3-level rotation, repeated
steps); closed-form pins on the device; and the BASELINE configs at full
size on dependence-cone windows (laplacian / wave13pt fp64 512^3, jacobi3d
fp32 1024^3, divergence / gradient fp32 512^3), in bench.py's launch
configuration.
"""
import zlib

import numpy as np
import pytest
import torch

from paper_2301_11389_b200 import inputs
from parity import (assert_parity, gpu_run, gpu_step, interior, oracle_window_run, ring_mask)

pytestmark = pytest.mark.gpu

KINDS_3D = ["laplacian3d7", "jacobi3d7", "wave13pt", "divergence", "gradient", "tricubic"]
SHAPES = {  # (nz, ny, nx) numpy order
    "f32": [(3, 3, 4), (5, 5, 8), (7, 9, 36), (12, 17, 132), (10, 33, 260), (6, 8, 516)],
    "f64": [(3, 3, 4), (5, 5, 6), (6, 11, 66), (9, 13, 130), (7, 20, 258)],
}


def cases():
    for kind in KINDS_3D:
        need = 5 if kind == "wave13pt" else 4 if kind == "tricubic" else 3
        for dt in ("f32", "f64"):
            for shape in SHAPES[dt] + ([(4, 4, 4), (19, 20, 132)] if kind == "tricubic" else []):
                if min(shape) >= need and shape[2] * (8 if dt == "f64" else 4) % 16 == 0:
                    yield kind, dt, shape


def seed_of(*key):
    return inputs.BASE_SEED + zlib.crc32(repr(key).encode()) % 1000


@pytest.mark.parametrize("kind,dtype,shape", list(cases()),
                         ids=lambda v: v if isinstance(v, str) else "x".join(map(str, v)))
def test_step_parity_and_variants(oracle, kind, dtype, shape):
    ar = oracle.arity(kind)
    ins = [inputs.generate_np(shape, dtype, seed_of(kind, dtype, shape), a)
           for a in range(ar["n_in"])]
    refs = [np.zeros_like(ins[0]) for _ in range(ar["n_out"])]
    oracle.step(kind, dtype, ins, refs)
    sl = interior(shape, ar["lo"], ar["hi"])
    outs = {}
    for var in ("shuffle", "plain"):
        gs = gpu_step(kind, dtype, ins, ar["n_out"], variant=var, fill=0)
        for k, (g, r) in enumerate(zip(gs, refs)):
            assert_parity(g[sl], r[sl], dtype, f"{kind} {dtype} {shape} {var} out{k}")
            assert np.all(g[ring_mask(shape, ar["lo"], ar["hi"])] == 0), "boundary written"
        outs[var] = gs
    for a, b in zip(outs["shuffle"], outs["plain"]):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), "SHUFFLE and PLAIN differ"


@pytest.mark.parametrize("kind,dtype,shape", [
    ("laplacian3d7", "f64", (9, 13, 130)), ("jacobi3d7", "f32", (12, 17, 132)),
    ("wave13pt", "f64", (10, 12, 66)), ("wave13pt", "f32", (9, 10, 132)),
    ("divergence", "f32", (7, 9, 36)), ("gradient", "f64", (6, 11, 66)),
    ("tricubic", "f32", (19, 20, 132))])
def test_run_parity(oracle, kind, dtype, shape):
    ar = oracle.arity(kind)
    ins = [inputs.generate_np(shape, dtype, inputs.BASE_SEED + 5, a) for a in range(ar["n_in"])]
    if ar["n_bufs"] == 2:
        bufs = [ins[0], np.zeros_like(ins[0])]
    elif kind == "wave13pt":
        bufs = [ins[0], ins[1], np.zeros_like(ins[0])]
    else:
        bufs = ins + [np.zeros_like(ins[0]) for _ in range(ar["n_out"])]
    ob = [b.copy() for b in bufs]
    ridx = oracle.run(kind, dtype, ob, 5)
    for var in ("shuffle", "plain"):
        gidx, gb = gpu_run(kind, dtype, [b.copy() for b in bufs], 5, variant=var)
        assert gidx == ridx
        for k in range(ar["n_out"] if ar["n_bufs"] > 3 else 1):
            assert_parity(gb[gidx + k], ob[ridx + k], dtype, f"{kind} run {var} out{k}")


@pytest.mark.parametrize("shape", [(64, 50, 260), (40, 23, 516)])
def test_tricubic_multi_plane_ranges(oracle, shape):
    """fp32 tricubic (ktricubic2) on grids where each SM gets several planes
    and the equal flattened ranges cross column boundaries (pipeline
    restarts): full-grid parity, both variants bit-identical."""
    ins = [inputs.generate_np(shape, "f32", inputs.BASE_SEED + 11, a) for a in range(4)]
    ref = np.zeros_like(ins[0])
    oracle.step("tricubic", "f32", ins, [ref])
    sl = interior(shape, 1, 2)
    outs = {}
    for var in ("shuffle", "plain"):
        (g,) = gpu_step("tricubic", "f32", ins, 1, variant=var, fill=0)
        assert_parity(g[sl], ref[sl], "f32", f"tricubic {shape} {var}")
        assert np.all(g[ring_mask(shape, 1, 2)] == 0), "boundary written"
        outs[var] = g
    assert np.array_equal(outs["shuffle"].view(np.uint32), outs["plain"].view(np.uint32))


def test_laplacian_closed_form_on_gpu():
    """i^2+j^2+k^2 -> 6 exactly; a linear field -> 0 exactly."""
    k, j, i = np.meshgrid(np.arange(20.0), np.arange(24.0), np.arange(132.0), indexing="ij")
    for f, v in (((i * i + j * j + k * k).astype(np.float32), 6.0),
                 ((3 * i - 2 * j + k).astype(np.float32), 0.0)):
        (g,) = gpu_step("laplacian3d7", "f32", [f], 1)
        assert np.all(g[1:-1, 1:-1, 1:-1] == v)


def test_divergence_gradient_closed_forms_on_gpu():
    k, j, i = np.meshgrid(np.arange(10.0), np.arange(12.0), np.arange(68.0), indexing="ij")
    (d,) = gpu_step("divergence", "f64", [i.copy(), j.copy(), k.copy()], 1)
    assert np.all(d[1:-1, 1:-1, 1:-1] == 3.0)
    gs = gpu_step("gradient", "f64", [3 * i - 2 * j + 5 * k], 3)
    for g, v in zip(gs, (3.0, -2.0, 5.0)):
        assert np.all(g[1:-1, 1:-1, 1:-1] == v)


def test_tricubic_special_offsets_on_gpu():
    """X=Y=Z=0 selects f[k][j][i] exactly; X=Y=Z=1 selects f[k+1][j+1][i+1]."""
    shape = (9, 20, 136)
    f = inputs.generate_np(shape, "f32", 3)
    for t, sl in ((0.0, (slice(1, -2),) * 3), (1.0, (slice(2, -1),) * 3)):
        c = np.full(shape, t, np.float32)
        (g,) = gpu_step("tricubic", "f32", [f, c, c, c], 1)
        np.testing.assert_array_equal(g[1:-2, 1:-2, 1:-2], f[sl])


def test_tricubic_reproduces_cubics_on_gpu():
    """Degree-3 polynomial per axis: g = p(i+X) q(j+Y) r(k+Z) (fp64, 1e-12)."""
    rng = np.random.default_rng(5)
    shape = (8, 19, 66)
    k, j, i = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")
    p = np.polynomial.Polynomial([0.3, -0.11, 0.025, 0.0005])
    q = np.polynomial.Polynomial([1.0, 0.05, -0.02, 0.001])
    r = np.polynomial.Polynomial([-0.7, 0.2, 0.1, -0.03])
    X, Y, Z = (rng.uniform(size=shape) for _ in range(3))
    (g,) = gpu_step("tricubic", "f64", [p(i) * q(j) * r(k), X, Y, Z], 1)
    exp = p(i + X) * q(j + Y) * r(k + Z)
    sl = (slice(1, -2),) * 3
    np.testing.assert_allclose(g[sl], exp[sl], rtol=1e-11, atol=1e-11)


# ----------------------------------------------------- BASELINE configs
def _dev_fields(shape, dtype, seed, n):
    return [inputs.generate_torch(shape, dtype, seed, a) for a in range(n)]


def _window_check(oracle, kind, dtype, dev_init, dev_result, n_iters, r, windows):
    """Compare device results against the oracle on dependence-cone windows;
    the oracle reads the initial fields' sub-blocks copied from the device."""
    shape = tuple(dev_init[0].shape)
    grow = (n_iters + 1) * r
    for w in windows:
        sub = tuple(slice(max(0, s.start - grow), min(n, s.stop + grow)) for s, n in zip(w, shape))
        fields = [t[sub].cpu().numpy() for t in dev_init]
        inner = tuple(slice(s.start - u.start, s.stop - u.start) for s, u in zip(w, sub))
        full_w = tuple(slice(0, u.stop - u.start) for u in sub)
        ref = oracle_window_run(oracle, kind, dtype, fields, n_iters, full_w, r, nthreads=8)
        assert_parity(dev_result[w].cpu().numpy(), ref[inner], dtype, f"{kind} window {w}")


@pytest.mark.slow
@pytest.mark.parametrize("kind,dtype,dims,iters", [
    ("laplacian3d7", "f64", (512, 512, 512), 10), ("wave13pt", "f64", (512, 512, 512), 10),
    ("jacobi3d7", "f32", (1024, 1024, 1024), 10)])
def test_configs_full_size_windows(oracle, kind, dtype, dims, iters):
    from paper_2301_11389_b200.binding import Stencil
    shape = dims[::-1]
    ar = oracle.arity(kind)
    init = _dev_fields(shape, dtype, inputs.BASE_SEED + 2, ar["n_in"])
    if kind == "wave13pt":
        bufs = [init[0].clone(), init[1].clone(), torch.zeros_like(init[0])]
        oinit = [init[0], init[1], torch.zeros_like(init[0])]
    else:
        bufs = [init[0].clone(), torch.zeros_like(init[0])]
        oinit = [init[0], torch.zeros_like(init[0])]
    st = Stencil(kind, dims, dtype)
    idx = st.run(bufs, iters)
    torch.cuda.synchronize()
    r = ar["hi"]
    n = shape[0]
    wins = [(slice(0, 8), slice(0, 8), slice(0, 40)),
            (slice(n // 2, n // 2 + 8), slice(n // 3, n // 3 + 8), slice(n - 70, n - 6)),
            (slice(n - 8, n), slice(n - 8, n), slice(n - 40, n))]
    _window_check(oracle, kind, dtype, oinit, bufs[idx], iters, r, wins)
    st.close()


@pytest.mark.slow
@pytest.mark.parametrize("kind,n", [("divergence", 512), ("gradient", 512), ("tricubic", 256)])
def test_suite_single_step_samples(oracle, kind, n):
    from paper_2301_11389_b200.binding import Stencil
    shape = (n, n, n)
    ar = oracle.arity(kind)
    ins = _dev_fields(shape, "f32", inputs.BASE_SEED + 9, ar["n_in"])
    outs = [torch.zeros_like(ins[0]) for _ in range(ar["n_out"])]
    st = Stencil(kind, shape[::-1], "f32")
    st.step(ins, outs)
    torch.cuda.synchronize()
    for w in [(slice(0, 6), slice(0, 6), slice(0, 140)), (slice(n // 2 - 6, n // 2), slice(n - 12, n),
                                                           slice(n - 132, n))]:
        sub = tuple(slice(max(0, s.start - 2), min(n, s.stop + 2)) for s in w)
        f = [t[sub].cpu().numpy() for t in ins]
        refs = [np.zeros_like(f[0]) for _ in range(ar["n_out"])]
        oracle.step(kind, "f32", f, refs)
        inner = tuple(slice(s.start - u.start, s.stop - u.start) for s, u in zip(w, sub))
        # compare interior points of the window only
        for k in range(ar["n_out"]):
            g = outs[k][w].cpu().numpy()
            rr = refs[k][inner]
            m = np.zeros(g.shape, bool)
            lo, hi = ar["lo"], ar["hi"]
            gi = [np.arange(s.start, s.stop) for s in w]
            ok = [(a >= lo) & (a < n - hi) for a in gi]
            m[np.ix_(*ok)] = True
            sub_in = tuple(slice(s.start - u.start, s.stop - u.start) for s, u in zip(w, sub))
            # the oracle only wrote the cut-out's own interior: exclude its ring
            ring = np.zeros(f[0].shape, bool)
            ring[lo:-hi, lo:-hi, lo:-hi] = True
            m &= ring[sub_in]
            assert_parity(g[m], rr[m], "f32", f"{kind} out{k} window {w}")
    st.close()


@pytest.mark.parametrize("dtype,shape", [("f32", (29, 37, 260)), ("f64", (27, 19, 130)),
                                         ("f32", (3, 3, 4)), ("f32", (20, 3, 132))])
def test_gradient_kgrad_chunks(oracle, dtype, shape):
    """kgrad (csrc/kgrad.cuh): z chunks of 8 planes with a ragged last chunk,
    row groups of 8 with a ragged last group, a ragged x-tile (260 = 2*128+4,
    130 = 2*64+2) and the degenerate one-plane / one-row cases, element by
    element against the oracle; SHUFFLE and PLAIN bit-identical."""
    u = inputs.generate_np(shape, dtype, seed_of("kgrad", dtype, shape))
    refs = [np.zeros_like(u) for _ in range(3)]
    oracle.step("gradient", dtype, [u], refs)
    sl = interior(shape, 1, 1)
    got = {}
    for var in ("shuffle", "plain"):
        gs = gpu_step("gradient", dtype, [u], 3, variant=var, fill=0)
        for k, (g, r) in enumerate(zip(gs, refs)):
            assert_parity(g[sl], r[sl], dtype, f"gradient {dtype} {shape} {var} out{k}")
            assert np.all(g[ring_mask(shape, 1, 1)] == 0), "boundary written"
        got[var] = gs
    for a, b in zip(got["shuffle"], got["plain"]):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), "SHUFFLE and PLAIN differ"
