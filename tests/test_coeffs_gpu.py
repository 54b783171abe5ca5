"""GPU parity with non-default, distinct coefficients through every kernel
family that takes coefficients.

The defaults hide mistakes: jacobi2d5's centre weight defaults to 0 and
divergence / gradient default to equal per-axis weights, so a kernel that
drops the centre tap or applies ay to the x difference passes every
default-coefficient test.  Here every kind runs with coefficients whose
every term is distinct and non-zero, through

  k2d (stencil_step), k2d2 with two and three sweeps per launch
  (stencil_set_fusion 2 / 3), ktb2d (the tile kernel, fusion -S), k3d
  (stencil_step; gradient on k3d via STB200_GRAD_K3D in a subprocess), kgrad
  (gradient's default kernel), kpaper and kpaper3d (the paper-literal
  variants),

element by element against the oracle (tolerance of DESIGN.md §7) and
SHUFFLE == PLAIN bit for bit.  Closed forms with distinct per-axis
coefficients (the oracle pins of test_oracle_pins.py) are re-run on the
device.  Also the BASELINE-size window check of jacobi2d5 fp32 32768^2 x10
on the three-sweep streaming path (k2d2 NSW=3, strips of H=128 rows),
which is the launch configuration of the DESIGN.md 32768^2 figures.
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2301_11389_b200 import inputs
from parity import assert_parity, gpu_step, interior, oracle_window_run

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# distinct, non-default, non-dyadic coefficients for every term
COEFFS = {
    "jacobi2d5": [0.3, 0.175],
    "jacobi2d9": [0.2, 0.15, 0.05],
    "gaussblur5x5": list(np.linspace(-0.3, 0.5, 25) * np.cos(np.arange(25))),
    "laplacian3d7": [-5.5, 0.875],
    "jacobi3d7": [0.2, 0.1333],
    "wave13pt": [1.1, 0.21, -0.013],
    "divergence": [0.5, 0.25, 0.125],
    "gradient": [0.5, 0.25, 0.125],
}
R = {"jacobi2d5": 1, "jacobi2d9": 1, "gaussblur5x5": 2}


def _ins(oracle, kind, dtype, shape, seed):
    ar = oracle.arity(kind)
    return [inputs.generate_np(shape, dtype, seed, a) for a in range(ar["n_in"])]


def _step_both_variants(oracle, kind, dtype, shape, variants=("shuffle", "plain")):
    ar = oracle.arity(kind)
    ins = _ins(oracle, kind, dtype, shape, inputs.BASE_SEED + 31)
    refs = [np.zeros_like(ins[0]) for _ in range(ar["n_out"])]
    oracle.step(kind, dtype, ins, refs, coeffs=COEFFS[kind])
    sl = interior(shape, ar["lo"], ar["hi"])
    got = {}
    for var in variants:
        gs = gpu_step(kind, dtype, ins, ar["n_out"], coeffs=COEFFS[kind], variant=var)
        for k, (g, r) in enumerate(zip(gs, refs)):
            assert_parity(g[sl], r[sl], dtype, f"{kind} {dtype} {shape} {var} out{k} coeffs")
        got[var] = gs
    first = got[variants[0]]
    for var in variants[1:]:
        for a, b in zip(first, got[var]):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), f"{variants[0]} != {var}"
    return got


# ----------------------------------------------------------------- k2d / k3d
@pytest.mark.parametrize("kind", ["jacobi2d5", "jacobi2d9", "gaussblur5x5"])
@pytest.mark.parametrize("dtype,shape", [("f32", (37, 516)), ("f64", (29, 258))])
def test_k2d_step_coeffs(oracle, kind, dtype, shape):
    _step_both_variants(oracle, kind, dtype, shape)


@pytest.mark.parametrize("kind", ["laplacian3d7", "jacobi3d7", "wave13pt", "divergence", "gradient"])
@pytest.mark.parametrize("dtype,shape", [("f32", (9, 21, 260)), ("f64", (8, 13, 130))])
def test_k3d_kgrad_step_coeffs(oracle, kind, dtype, shape):
    _step_both_variants(oracle, kind, dtype, shape)


def test_gradient_k3d_kernel_coeffs(oracle, tmp_path):
    """gradient's k3d instantiation (the fused peer-store path uses it; the
    single-GPU default is kgrad) selected with STB200_GRAD_K3D=1, which is
    read once per process: run in a subprocess."""
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from test_coeffs_gpu import _k3d_gradient_child; _k3d_gradient_child()\n"
    ) % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ, STB200_GRAD_K3D="1")
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "k3d-gradient-ok" in p.stdout


def _k3d_gradient_child():
    from oracle import pyoracle
    pyoracle.build()
    for dtype, shape in (("f32", (9, 21, 260)), ("f64", (8, 13, 130))):
        _step_both_variants(pyoracle, "gradient", dtype, shape)
    print("k3d-gradient-ok")


# --------------------------------------------------- paper-literal families
@pytest.mark.parametrize("kind,shape", [("jacobi2d5", (9, 132)), ("jacobi2d9", (9, 132)),
                                        ("gaussblur5x5", (8, 268)),
                                        ("laplacian3d7", (6, 9, 132)), ("jacobi3d7", (6, 9, 132)),
                                        ("wave13pt", (7, 8, 132)), ("divergence", (6, 9, 132)),
                                        ("gradient", (6, 9, 132))])
def test_paper_variants_coeffs(oracle, kind, shape):
    """kpaper / kpaper3d: ORIGINAL, PTXASW and UNIFORM equal the oracle with
    distinct coefficients and equal each other (and the register-cache
    SHUFFLE kernel) bit for bit."""
    _step_both_variants(oracle, kind, "f32", shape,
                        variants=("shuffle", "paper_original", "paper_ptxasw", "paper_uniform"))


# ------------------------------------------------------- fused 2-D run paths
def _run(kind, dtype, f, n, fusion, variant):
    from paper_2301_11389_b200.binding import Stencil
    st = Stencil(kind, f.shape[::-1], dtype, coeffs=COEFFS[kind], variant=variant)
    st.set_fusion(fusion)
    d = [torch.from_numpy(f.copy()).cuda(), torch.zeros(f.shape, dtype=torch.from_numpy(f).dtype,
                                                       device="cuda")]
    spl = st.info()["sweeps_per_launch"]
    idx = st.run(d, n)
    torch.cuda.synchronize()
    out = d[idx].cpu().numpy()
    st.close()
    return out, spl


@pytest.mark.parametrize("kind,fusion", [("jacobi2d5", 2), ("jacobi2d5", 3), ("jacobi2d9", 2),
                                         ("jacobi2d9", 3), ("gaussblur5x5", 2),
                                         ("jacobi2d5", -6), ("jacobi2d9", -6), ("gaussblur5x5", -4)])
@pytest.mark.parametrize("dtype,shape", [("f32", (70, 1028)), ("f64", (45, 514))])
def test_fused_runs_coeffs(oracle, kind, fusion, dtype, shape):
    """k2d2 (streaming, 2 or 3 sweeps per launch) and ktb2d (tile kernel)
    with distinct coefficients: oracle parity after 9 sweeps (a remainder
    sweep plus fused launches), both variants bit-identical to each other
    and to one sweep per launch."""
    n = 9
    f = inputs.generate_np(shape, dtype, inputs.BASE_SEED + 33)
    bufs = [f.copy(), np.zeros_like(f)]
    ridx = oracle.run(kind, dtype, bufs, n, coeffs=COEFFS[kind])
    single, _ = _run(kind, dtype, f, n, 1, "shuffle")
    for var in ("shuffle", "plain"):
        g, spl = _run(kind, dtype, f, n, fusion, var)
        assert spl == abs(fusion) or fusion < 0
        assert_parity(g, bufs[ridx], dtype, f"{kind} fusion {fusion} {var}")
        assert np.array_equal(g.view(np.uint8), single.view(np.uint8)), f"{var} fused != single sweeps"


# ------------------------------------------------------ closed forms on GPU
def test_per_axis_closed_forms_on_gpu():
    """The oracle pins of test_oracle_pins.py with distinct per-axis
    coefficients, on k3d (divergence) and kgrad (gradient): div of
    (2i, -5j, 7k) with (1/2, 1/4, 1/8) is 1.25 exactly; grad of 3i-2j+5k is
    (3, -1, 1.25) exactly."""
    for dtype, npdt, nx in (("f32", np.float32, 132), ("f64", np.float64, 66)):
        k, j, i = np.meshgrid(np.arange(10.0), np.arange(12.0), np.arange(float(nx)), indexing="ij")
        ins = [(2 * i).astype(npdt), (-5 * j).astype(npdt), (7 * k).astype(npdt)]
        (d,) = gpu_step("divergence", dtype, ins, 1, coeffs=[0.5, 0.25, 0.125])
        assert np.all(d[1:-1, 1:-1, 1:-1] == 1.25)
        gs = gpu_step("gradient", dtype, [(3 * i - 2 * j + 5 * k).astype(npdt)], 3,
                      coeffs=[0.5, 0.25, 0.125])
        for g, v in zip(gs, (3.0, -1.0, 1.25)):
            assert np.all(g[1:-1, 1:-1, 1:-1] == v)


def test_jacobi_centre_weight_closed_form_on_gpu():
    """(c0, c1) = (1/2, 1/8): i^2 + j^2 -> +1/2 exactly, through k2d, the
    two- and three-sweep streaming kernel and the tile kernel (after n
    sweeps: + n/2)."""
    j, i = np.meshgrid(np.arange(300.0), np.arange(260.0), indexing="ij")
    f = (i * i + j * j).astype(np.float32)
    (g,) = gpu_step("jacobi2d5", "f32", [f], 1, coeffs=[0.5, 0.125])
    np.testing.assert_array_equal(g[1:-1, 1:-1], f[1:-1, 1:-1] + 0.5)
    from paper_2301_11389_b200.binding import Stencil
    for fusion in (2, 3, -4):
        st = Stencil("jacobi2d5", f.shape[::-1], "f32", coeffs=[0.5, 0.125])
        st.set_fusion(fusion)
        d = [torch.from_numpy(f.copy()).cuda(), torch.zeros(f.shape, device="cuda")]
        idx = st.run(d, 6)
        torch.cuda.synchronize()
        g = d[idx].cpu().numpy()
        # after 6 sweeps the Dirichlet ring has influenced cells within 6 of it
        np.testing.assert_array_equal(g[7:-7, 7:-7], f[7:-7, 7:-7] + 3.0)
        st.close()


# ------------------------------------- 32768^2 on the three-sweep streaming path
@pytest.mark.slow
@pytest.mark.parametrize("variant", ["shuffle", "plain"])
def test_jacobi2d5_32768_x10_windows(oracle, variant):
    """jacobi2d5 fp32 32768^2 x10 through stencil_run in its default
    configuration: one single sweep, then three k2d2 launches of three
    sweeps each (NSW=3, strips of H=128 rows), the configuration DESIGN.md
    §5.5 times.  Dependence-cone windows at the corners, the edges, strip
    boundaries and a random interior spot, against the oracle."""
    from paper_2301_11389_b200.binding import Stencil
    n, iters = 32768, 10
    st = Stencil("jacobi2d5", (n, n), "f32", variant=variant)
    assert st.info()["sweeps_per_launch"] == 3
    f = inputs.generate_torch((n, n), "f32", inputs.BASE_SEED + 0)
    bufs = [f.clone(), torch.zeros_like(f)]
    idx = st.run(bufs, iters)
    torch.cuda.synchronize()
    res = bufs[idx]
    del bufs[1 - idx]
    rng = np.random.default_rng(1)
    y, x = (int(v) for v in rng.integers(200, n - 400, size=2))
    wins = [(slice(0, 40), slice(0, 160)), (slice(n - 40, n), slice(n - 160, n)),
            (slice(0, 40), slice(n - 300, n)), (slice(n - 64, n), slice(0, 200)),
            (slice(120, 140), slice(4000, 4400)), (slice(1 + 128 * 77 - 8, 1 + 128 * 77 + 8),
                                                   slice(119 * 40, 119 * 41 + 16)),
            (slice(y, y + 48), slice(x, x + 300))]
    grow = (iters + 1) * 1
    for w in wins:
        sub = tuple(slice(max(0, s.start - grow), min(n, s.stop + grow)) for s in w)
        fw = f[sub].cpu().numpy()
        inner = tuple(slice(s.start - u.start, s.stop - u.start) for s, u in zip(w, sub))
        full_w = tuple(slice(0, u.stop - u.start) for u in sub)
        ref = oracle_window_run(oracle, "jacobi2d5", "f32", [fw, np.zeros_like(fw)], iters,
                                full_w, 1)
        assert_parity(res[w].cpu().numpy(), ref[inner], "f32", f"jacobi 32768^2 window {w}")
    st.close()
