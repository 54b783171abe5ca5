"""Pins of the CPU oracle against what the paper and mathematics fix.

None of these compares the oracle with itself or with a retyped copy of its
formula: each checks a value printed in the paper (Table 1 counts, Listing 5
hand grids), a closed form, an invariant, a textbook pattern, or a library
routine that reduces to the same operation (scipy.ndimage.correlate on
integer data, where fp64 arithmetic is exact).  DESIGN.md §4 lists which pin
guards which part of each definition.
"""
import os
from collections import defaultdict

import numpy as np
import pytest
import scipy.ndimage as ndi

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ALL_KINDS = ["jacobi2d5", "jacobi2d9", "gaussblur5x5", "gameoflife", "laplacian3d7",
             "jacobi3d7", "wave13pt", "divergence", "gradient", "tricubic",
             "tricubic2", "uxx1", "lapgsrb", "whispering"]


def read_sections(path):
    """Parse a golden grid file: '# section NAME' headers followed by rows."""
    secs, cur = {}, None
    for line in open(path):
        s = line.strip()
        if s.startswith("# section"):
            cur = s.split()[2]
            secs[cur] = []
        elif s and not s.startswith("#") and cur:
            secs[cur].append([float(v) for v in s.split()])
    return {k: np.array(v) for k, v in secs.items()}


def grid(shape, dtype, fill=0):
    return np.full(shape, fill, dtype={"f32": np.float32, "f64": np.float64,
                                       "i32": np.int32}[dtype])


def interior(kind_ar, shape):
    lo, hi = kind_ar["lo"], kind_ar["hi"]
    return tuple(slice(lo, n - hi) for n in shape)


# --------------------------------------------------------------- Table 1
def _dependencies(oracle, kind, seed=1, centres=None):
    """Brute force: which (array, offset) inputs change the output at a point
    (the union over `centres`: lapgsrb's red and black points take different
    branches)."""
    ar = oracle.arity(kind)
    nd = ar["ndims"]
    n = 11
    shape = (n,) * nd
    dtype = "i32" if kind == "gameoflife" else "f64"
    rng = np.random.default_rng(seed)
    deps = set()
    for centre in centres or [(n // 2,) * nd]:
        deps |= _deps_at(oracle, kind, ar, nd, shape, dtype, rng, centre)
    return deps


def _deps_at(oracle, kind, ar, nd, shape, dtype, rng, centre):
    deps = set()
    trials = 40 if kind == "gameoflife" else 2
    for _ in range(trials):
        if dtype == "i32":
            ins = [rng.integers(0, 2, size=shape).astype(np.int32) for _ in range(ar["n_in"])]
        else:
            ins = [rng.uniform(0.05, 0.95, size=shape) for _ in range(ar["n_in"])]
        outs = [grid(shape, dtype) for _ in range(ar["n_out"])]
        oracle.step(kind, dtype, ins, outs)
        base = [o[centre] for o in outs]
        for a in range(ar["n_in"]):
            for off in np.ndindex(*(7,) * nd):
                off = tuple(o - 3 for o in off)
                pos = tuple(c + o for c, o in zip(centre, off))
                pert = [x.copy() for x in ins]
                if dtype == "i32":
                    pert[a][pos] = 1 - pert[a][pos]
                else:
                    pert[a][pos] += 0.37
                outs2 = [grid(shape, dtype) for _ in range(ar["n_out"])]
                oracle.step(kind, dtype, pert, outs2)
                if any(o2[centre] != b for o2, b in zip(outs2, base)):
                    deps.add((a, off[::-1]))        # store offset as (dx, dy[, dz])
    return deps


def _table1_counts_ordered(loads):
    """The paper's selection rule on a load sequence in program order: loads
    of one array that differ only along x share a source, the first of them
    in program order; every later one is a shuffle of delta |x - x_source|
    (a shuffled load is never a source)."""
    src, shuffles, delta_sum = {}, 0, 0
    for a, off in loads:
        key = (a, off[1:])
        if key not in src:
            src[key] = off[0]
        else:
            shuffles += 1
            delta_sum += abs(off[0] - src[key])
    return shuffles, len(loads), (delta_sum / shuffles if shuffles else 0.0)


def _table1_counts(deps):
    """Shuffles/loads/avg delta by the paper's selection rule:
    loads of one array that differ only along x (the thread dimension,
    PAPER.md:505-507) share a source; delta N = x distance to the source;
    the x-end tap is the source (DESIGN.md §3 R1)."""
    groups = defaultdict(list)
    for a, off in deps:
        groups[(a, off[1:])].append(off[0])
    shuffles, delta_sum = 0, 0
    for xs in groups.values():
        xs.sort()
        shuffles += len(xs) - 1
        delta_sum += sum(x - xs[0] for x in xs[1:])
    return shuffles, len(deps), (delta_sum / shuffles if shuffles else 0.0)


def _table1_rows():
    rows = []
    for line in open(os.path.join(GOLDEN, "table1.txt")):
        if line.strip() and not line.startswith("#"):
            p = line.split()
            rows.append((p[0], p[1], int(p[2]), int(p[3]), float(p[4])))
    return rows


@pytest.mark.parametrize("row", _table1_rows(), ids=lambda r: r[0])
def test_table1_load_and_shuffle_counts(oracle, row):
    """Table 1: loads, shuffles and average delta follow
    from the tap set of each stencil — pins radius, tap set and arity."""
    _, kind, shuffles, loads, delta = row
    if kind == "lapgsrb":                  # union of a black (5,5,5) and a red (6,5,5) point
        deps = _dependencies(oracle, kind, centres=[(5, 5, 5), (5, 5, 6)])
        assert len(deps) == 25 and all(sum(map(abs, o)) <= 2 for _, o in deps)   # the L1 ball
    else:
        deps = _dependencies(oracle, kind)
    if kind == "whispering":
        seq = [(int(r[0]), (int(r[1]), int(r[2])))
               for r in (l.split() for l in open(os.path.join(GOLDEN, "whispering_loads.txt")))
               if r and not r[0].startswith("#")]
        assert set(seq) == deps            # the reading's load sequence covers exactly the oracle's taps
        s, l, d = _table1_counts_ordered(seq)
    else:
        s, l, d = _table1_counts(deps)
    assert (s, l) == (shuffles, loads)
    assert abs(d - delta) < 0.005


# --------------------------------------------------- hand grids (Listing 5)
def test_jacobi2d5_hand_4x4(oracle):
    g = read_sections(os.path.join(GOLDEN, "jacobi2d5_4x4.txt"))
    for dtype in ("f32", "f64"):
        inp = g["input"].astype(np.float32 if dtype == "f32" else np.float64)
        out = np.full_like(inp, -1)
        oracle.step("jacobi2d5", dtype, [inp], [out], coeffs=[0.0, 0.25])
        np.testing.assert_array_equal(out, g["output"])


def test_jacobi2d9_hand_impulse_4x4(oracle):
    g = read_sections(os.path.join(GOLDEN, "jacobi2d9_impulse_4x4.txt"))
    inp = g["input"].astype(np.float64)
    out = np.full_like(inp, -1)
    oracle.step("jacobi2d9", "f64", [inp], [out], coeffs=[0.25, 0.125, 0.0625])
    np.testing.assert_array_equal(out, g["output"])


def test_default_coeffs_are_the_documented_values(oracle):
    """DESIGN.md §3 R2: the defaults, written as exact rationals."""
    np.testing.assert_array_equal(oracle.default_coeffs("jacobi2d5"), [0, 1 / 4])
    np.testing.assert_array_equal(oracle.default_coeffs("jacobi2d9"), [1 / 4, 1 / 8, 1 / 16])
    b = np.array([1, 4, 6, 4, 1]) / 16
    np.testing.assert_array_equal(oracle.default_coeffs("gaussblur5x5"), np.outer(b, b).ravel())
    np.testing.assert_array_equal(oracle.default_coeffs("laplacian3d7"), [-6, 1])
    assert oracle.default_coeffs("jacobi3d7")[0] == 0
    assert abs(oracle.default_coeffs("jacobi3d7")[1] - 1 / 6) < 1e-17
    lam = 1 / 8
    np.testing.assert_allclose(oracle.default_coeffs("wave13pt"),
                               [2 - 7.5 * lam, 4 * lam / 3, -lam / 12], rtol=1e-16)
    np.testing.assert_array_equal(oracle.default_coeffs("divergence"), [0.5] * 3)
    np.testing.assert_array_equal(oracle.default_coeffs("gradient"), [0.5] * 3)
    assert len(oracle.default_coeffs("tricubic")) == 0
    assert len(oracle.default_coeffs("gameoflife")) == 0


# ----------------------------------------------------------- closed forms
def _ij(shape):
    return np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("kind,coeffs,shift", [
    ("jacobi2d5", [0, 0.25], 1.0),                  # variance 1/2 per axis
    ("jacobi2d9", [0.25, 0.125, 0.0625], 1.0),      # variance 1/2 per axis
    ("gaussblur5x5", None, 2.0),                    # binomial(4): variance 1 per axis
])
def test_2d_quadratic_moves_by_variance(oracle, dtype, kind, coeffs, shift):
    """sum_w w*(i+di)^2 = i^2 + sum_w w di^2 for a normalised symmetric stencil."""
    j, i = _ij((37, 53))
    f = (i * i + j * j).astype(np.float32 if dtype == "f32" else np.float64)
    out = np.zeros_like(f)
    oracle.step(kind, dtype, [f], [out], coeffs=coeffs)
    ar = oracle.arity(kind)
    sl = interior(ar, f.shape)
    np.testing.assert_array_equal(out[sl], f[sl] + shift)


@pytest.mark.parametrize("kind,coeffs", [("jacobi2d5", [0, 0.25]),
                                         ("jacobi2d9", [0.25, 0.125, 0.0625]),
                                         ("gaussblur5x5", None)])
def test_2d_constant_and_linear_preserved(oracle, kind, coeffs):
    j, i = _ij((21, 34))
    for f in (np.full((21, 34), 7.0), 3 * i - 5 * j + 11):
        out = np.zeros_like(f)
        oracle.step(kind, "f64", [f], [out], coeffs=coeffs)
        sl = interior(oracle.arity(kind), f.shape)
        np.testing.assert_array_equal(out[sl], f[sl])


@pytest.mark.parametrize("kind,ncoef", [("jacobi2d5", 2), ("jacobi2d9", 3),
                                        ("gaussblur5x5", 25), ("laplacian3d7", 2),
                                        ("wave13pt", 3)])
def test_library_correlate_on_integer_data(oracle, kind, ncoef):
    """Reduction to a library routine: each linear kind equals
    scipy.ndimage.correlate with the kind's tap weights (exact: integer data,
    dyadic weights).  Pins orientation (correlation, not convolution, R4),
    every tap position and weight assignment."""
    rng = np.random.default_rng(7)
    c = rng.integers(-8, 9, size=ncoef) / 8.0
    ar = oracle.arity(kind)
    shape = (9, 10, 11) if ar["ndims"] == 3 else (13, 17)
    f = rng.integers(-50, 50, size=shape).astype(np.float64)
    if kind == "jacobi2d5":
        W = np.array([[0, c[1], 0], [c[1], c[0], c[1]], [0, c[1], 0]])
    elif kind == "jacobi2d9":
        W = np.array([[c[2], c[1], c[2]], [c[1], c[0], c[1]], [c[2], c[1], c[2]]])
    elif kind == "gaussblur5x5":
        W = c.reshape(5, 5)
    elif kind == "laplacian3d7":
        W = np.zeros((3, 3, 3))
        W[1, 1, 1] = c[0]
        for ax in range(3):
            for s in (0, 2):
                idx = [1, 1, 1]
                idx[ax] = s
                W[tuple(idx)] = c[1]
    else:  # wave13pt with prev = 0
        W = np.zeros((5, 5, 5))
        W[2, 2, 2] = c[0]
        for ax in range(3):
            for s, m in ((1, c[1]), (3, c[1]), (0, c[2]), (4, c[2])):
                idx = [2, 2, 2]
                idx[ax] = s
                W[tuple(idx)] = m
    ref = ndi.correlate(f, W, mode="constant")
    out = np.zeros_like(f)
    ins = [np.zeros_like(f), f] if kind == "wave13pt" else [f]
    oracle.step(kind, "f64", ins, [out], coeffs=c)
    sl = interior(ar, shape)
    np.testing.assert_array_equal(out[sl], ref[sl])


def test_gaussblur_asymmetric_impulse_orientation(oracle):
    """Correlation (R4): an impulse at (j0,i0) lands weight w[dj][di] at
    (j0-dj, i0-di).  Asymmetric weights make a transposition visible."""
    w = np.arange(1, 26, dtype=np.float64)
    f = np.zeros((11, 11))
    f[5, 5] = 1.0
    out = np.zeros_like(f)
    oracle.step("gaussblur5x5", "f64", [f], [out], coeffs=w)
    for dj in range(-2, 3):
        for di in range(-2, 3):
            assert out[5 - dj, 5 - di] == w[(dj + 2) * 5 + di + 2]


def test_gaussblur_separable_equals_two_1d_passes(oracle):
    """Binomial blur = row pass then column pass (exact on integer data)."""
    rng = np.random.default_rng(3)
    f = rng.integers(0, 256, size=(24, 31)).astype(np.float64)
    b = np.array([1, 4, 6, 4, 1]) / 16.0
    two_pass = ndi.correlate1d(ndi.correlate1d(f, b, axis=1, mode="constant"), b, axis=0,
                               mode="constant")
    out = np.zeros_like(f)
    oracle.step("gaussblur5x5", "f64", [f], [out])
    np.testing.assert_array_equal(out[2:-2, 2:-2], two_pass[2:-2, 2:-2])


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_laplacian_closed_forms(oracle, dtype):
    """Linear field -> 0 exactly; i^2+j^2+k^2 -> 6 exactly (the discrete
    Laplacian is exact on quadratics); 4x4x4: all 8 interior outputs = 6."""
    npdt = np.float32 if dtype == "f32" else np.float64
    for shape in ((4, 4, 4), (9, 13, 17)):
        k, j, i = _ij(shape)
        lin = (2 * i - 3 * j + 5 * k + 1).astype(npdt)
        quad = (i * i + j * j + k * k).astype(npdt)
        for f, val in ((lin, 0.0), (quad, 6.0)):
            out = np.full_like(f, -99)
            oracle.step("laplacian3d7", dtype, [f], [out])
            assert np.all(out[1:-1, 1:-1, 1:-1] == val)
            # boundary ring untouched
            mask = np.ones(shape, bool)
            mask[1:-1, 1:-1, 1:-1] = False
            assert np.all(out[mask] == -99)


def test_jacobi3d7_invariants(oracle):
    k, j, i = _ij((8, 9, 10))
    for f in (np.full((8, 9, 10), 3.0), 2 * i + j - 4 * k):
        out = np.zeros_like(f)
        oracle.step("jacobi3d7", "f64", [f], [out], coeffs=[0.25, 0.125])
        np.testing.assert_array_equal(out[1:-1, 1:-1, 1:-1], f[1:-1, 1:-1, 1:-1])
    f = np.full((8, 9, 10), 0.7)
    out = np.zeros_like(f)
    oracle.step("jacobi3d7", "f64", [f], [out])     # default (0, 1/6)
    np.testing.assert_allclose(out[1:-1, 1:-1, 1:-1], 0.7, rtol=2.3e-16)


def test_wave13pt_closed_forms(oracle):
    """Constant and linear fields are stationary (prev = cur); the 4th-order
    Laplacian is exact on i^2, so next = 2 i^2 + lam*2 - i^2 = i^2 + 2 lam."""
    lam = 0.125
    shape = (9, 10, 11)
    k, j, i = _ij(shape)
    for f in (np.full(shape, 2.5), 3 * i - j + 2 * k):
        out = np.zeros_like(f)
        oracle.step("wave13pt", "f64", [f.copy(), f.copy()], [out])
        np.testing.assert_allclose(out[2:-2, 2:-2, 2:-2], f[2:-2, 2:-2, 2:-2], rtol=1e-15,
                                   atol=1e-13)
    for f in (i * i, j * j, k * k):
        out = np.zeros_like(f)
        oracle.step("wave13pt", "f64", [f.copy(), f.copy()], [out])
        np.testing.assert_allclose(out[2:-2, 2:-2, 2:-2], f[2:-2, 2:-2, 2:-2] + 2 * lam,
                                   rtol=1e-14, atol=1e-13)


def test_wave13pt_prev_enters_with_minus_sign(oracle):
    shape = (7, 7, 7)
    cur = np.zeros(shape)
    prev = np.zeros(shape)
    prev[3, 3, 3] = 5.0
    out = np.zeros(shape)
    oracle.step("wave13pt", "f64", [prev, cur], [out])
    assert out[3, 3, 3] == -5.0 and np.count_nonzero(out) == 1


def test_divergence_closed_forms(oracle):
    shape = (6, 7, 8)
    k, j, i = _ij(shape)
    out = np.zeros(shape)
    oracle.step("divergence", "f64", [i.copy(), j.copy(), k.copy()], [out])
    assert np.all(out[1:-1, 1:-1, 1:-1] == 3.0)
    oracle.step("divergence", "f64", [j.copy(), k.copy(), i.copy()], [out])
    assert np.all(out[1:-1, 1:-1, 1:-1] == 0.0)
    # solenoidal-looking field with distinct slopes per component
    oracle.step("divergence", "f64", [2 * i, -5 * j, 7 * k], [out])
    assert np.all(out[1:-1, 1:-1, 1:-1] == 4.0)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_gradient_closed_form(oracle, dtype):
    shape = (6, 7, 8)
    k, j, i = _ij(shape)
    u = (3 * i - 2 * j + 5 * k).astype(np.float32 if dtype == "f32" else np.float64)
    outs = [np.zeros_like(u) for _ in range(3)]
    oracle.step("gradient", dtype, [u], outs)
    for o, v in zip(outs, (3.0, -2.0, 5.0)):
        assert np.all(o[1:-1, 1:-1, 1:-1] == v)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_divergence_per_axis_coefficients(oracle, dtype):
    """R9 with distinct per-axis coefficients (ax, ay, az) = (1/2, 1/4, 1/8):
    (u, v, w) = (2i, -5j, 7k) has central differences (4, -10, 14), so
    div = 2 - 2.5 + 1.75 = 1.25 exactly.  Any coefficient->axis permutation
    gives another value (ax<->ay: 1 - 5 + 1.75 = -2.25; ax<->az: 0.5 - 2.5
    + 7 = 5.0; ay<->az: 2 - 1.25 + 3.5 = 4.25), as does a coefficient applied
    to the wrong array."""
    npdt = np.float32 if dtype == "f32" else np.float64
    shape = (6, 7, 12)
    k, j, i = _ij(shape)
    out = np.zeros(shape, npdt)
    ins = [(2 * i).astype(npdt), (-5 * j).astype(npdt), (7 * k).astype(npdt)]
    oracle.step("divergence", dtype, ins, [out], coeffs=[0.5, 0.25, 0.125])
    assert np.all(out[1:-1, 1:-1, 1:-1] == 1.25)
    oracle.step("divergence", dtype, ins, [out], coeffs=[0.25, 0.5, 0.125])
    assert np.all(out[1:-1, 1:-1, 1:-1] == -2.25)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_gradient_per_axis_coefficients(oracle, dtype):
    """R10 with (ax, ay, az) = (1/2, 1/4, 1/8): u = 3i - 2j + 5k has central
    differences (6, -4, 10), so (gx, gy, gz) = (3, -1, 1.25) exactly; each
    output carries its own axis' coefficient."""
    npdt = np.float32 if dtype == "f32" else np.float64
    shape = (6, 7, 12)
    k, j, i = _ij(shape)
    u = (3 * i - 2 * j + 5 * k).astype(npdt)
    outs = [np.zeros_like(u) for _ in range(3)]
    oracle.step("gradient", dtype, [u], outs, coeffs=[0.5, 0.25, 0.125])
    for o, v in zip(outs, (3.0, -1.0, 1.25)):
        assert np.all(o[1:-1, 1:-1, 1:-1] == v)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_jacobi_centre_coefficient(oracle, dtype):
    """A non-zero centre weight (the default jacobi2d5 / jacobi3d7 centre
    weight is 0): with (c0, c1) = (1/2, 1/8), i^2+j^2 -> (1/2 + 4/8) f +
    (1/8)*4 = f + 1/2; in 3-D with (a, b) = (1/4, 1/8), i^2+j^2+k^2 ->
    (1/4 + 6/8) f + (1/8)*6 = f + 3/4.  Exact (dyadic)."""
    npdt = np.float32 if dtype == "f32" else np.float64
    j, i = _ij((19, 24))
    f = (i * i + j * j).astype(npdt)
    out = np.zeros_like(f)
    oracle.step("jacobi2d5", dtype, [f], [out], coeffs=[0.5, 0.125])
    np.testing.assert_array_equal(out[1:-1, 1:-1], f[1:-1, 1:-1] + 0.5)
    k, j, i = _ij((7, 9, 12))
    f = (i * i + j * j + k * k).astype(npdt)
    out = np.zeros_like(f)
    oracle.step("jacobi3d7", dtype, [f], [out], coeffs=[0.25, 0.125])
    np.testing.assert_array_equal(out[1:-1, 1:-1, 1:-1], f[1:-1, 1:-1, 1:-1] + 0.75)


def _tri_inputs(shape, X, Y, Z, f):
    return [f, np.full(shape, X) if np.isscalar(X) else X,
            np.full(shape, Y) if np.isscalar(Y) else Y,
            np.full(shape, Z) if np.isscalar(Z) else Z]


def test_tricubic_special_offsets(oracle):
    """t=0 selects the node 0 sample; t=1 selects node +1 (Lagrange
    cardinality).  Exact in fp64."""
    rng = np.random.default_rng(11)
    shape = (7, 8, 9)
    f = rng.uniform(size=shape)
    out = np.zeros(shape)
    oracle.step("tricubic", "f64", _tri_inputs(shape, 0.0, 0.0, 0.0, f), [out])
    np.testing.assert_array_equal(out[1:-2, 1:-2, 1:-2], f[1:-2, 1:-2, 1:-2])
    oracle.step("tricubic", "f64", _tri_inputs(shape, 1.0, 1.0, 1.0, f), [out])
    np.testing.assert_array_equal(out[1:-2, 1:-2, 1:-2], f[2:-1, 2:-1, 2:-1])
    # mixed: X=1 only moves along x (the fastest axis)
    oracle.step("tricubic", "f64", _tri_inputs(shape, 1.0, 0.0, 0.0, f), [out])
    np.testing.assert_array_equal(out[1:-2, 1:-2, 1:-2], f[1:-2, 1:-2, 2:-1])


def test_tricubic_reproduces_cubic_polynomials(oracle):
    """Cubic Lagrange interpolation is exact on polynomials of degree <= 3
    per axis: g = p(i+X) q(j+Y) r(k+Z).  Distinct polynomials and offsets per
    axis expose any axis mix-up."""
    rng = np.random.default_rng(5)
    shape = (8, 9, 10)
    k, j, i = _ij(shape)
    p = np.polynomial.Polynomial([0.3, -1.1, 0.25, 0.05])
    q = np.polynomial.Polynomial([1.0, 0.5, -0.2, 0.01])
    r = np.polynomial.Polynomial([-0.7, 0.2, 0.1, -0.03])
    f = p(i) * q(j) * r(k)
    X, Y, Z = (rng.uniform(size=shape) for _ in range(3))
    out = np.zeros(shape)
    oracle.step("tricubic", "f64", _tri_inputs(shape, X, Y, Z, f), [out])
    exp = p(i + X) * q(j + Y) * r(k + Z)
    sl = (slice(1, -2),) * 3
    np.testing.assert_allclose(out[sl], exp[sl], rtol=1e-12, atol=1e-12)


def test_tricubic_partition_of_unity(oracle):
    rng = np.random.default_rng(9)
    shape = (6, 6, 6)
    X, Y, Z = (rng.uniform(size=shape) for _ in range(3))
    out = np.zeros(shape)
    oracle.step("tricubic", "f64", _tri_inputs(shape, X, Y, Z, np.full(shape, 1.25)), [out])
    np.testing.assert_allclose(out[1:-2, 1:-2, 1:-2], 1.25, rtol=1e-14)


# ----------------------------------------------------------- game of life
def _life(cells, shape, gens, oracle):
    g = np.zeros(shape, np.int32)
    for (r, c) in cells:
        g[r, c] = 1
    bufs = [g, np.zeros_like(g)]
    idx = oracle.run("gameoflife", "i32", bufs, gens)
    return {tuple(x) for x in np.argwhere(bufs[idx] == 1)}


def test_life_blinker_period_2(oracle):
    horiz = {(2, 1), (2, 2), (2, 3)}
    vert = {(1, 2), (2, 2), (3, 2)}
    assert _life(horiz, (5, 5), 1, oracle) == vert
    assert _life(horiz, (5, 5), 2, oracle) == horiz


def test_life_still_lifes(oracle):
    block = {(3, 3), (3, 4), (4, 3), (4, 4)}
    beehive = {(3, 4), (3, 5), (4, 3), (4, 6), (5, 4), (5, 5)}
    for s in (block, beehive):
        for gens in (1, 2, 5):
            assert _life(s, (10, 10), gens, oracle) == s


def test_life_glider_translates(oracle):
    glider = {(1, 2), (2, 3), (3, 1), (3, 2), (3, 3)}
    for n in (1, 2, 3):
        moved = {(r + n, c + n) for (r, c) in glider}
        assert _life(glider, (16, 16), 4 * n, oracle) == moved


def test_life_brute_force_neighbour_sets(oracle):
    """Random 3..16-wide soups: every interior cell against a set-based
    neighbour count; the border is never written (fixed, R5)."""
    rng = np.random.default_rng(2)
    for _ in range(25):
        shape = tuple(int(x) for x in rng.integers(3, 17, size=2))
        g = rng.integers(0, 2, size=shape).astype(np.int32)
        out = np.full(shape, 7, np.int32)
        oracle.step("gameoflife", "i32", [g], [out])
        live = {tuple(x) for x in np.argwhere(g == 1)}
        for r in range(shape[0]):
            for c in range(shape[1]):
                if 0 < r < shape[0] - 1 and 0 < c < shape[1] - 1:
                    nb = {(r + a, c + b) for a in (-1, 0, 1) for b in (-1, 0, 1)} - {(r, c)}
                    n = len(nb & live)
                    alive = (r, c) in live
                    assert out[r, c] == int(n == 3 or (alive and n == 2))
                else:
                    assert out[r, c] == 7


# ------------------------------------------------------ linearity / runs
@pytest.mark.parametrize("kind", ["jacobi2d5", "jacobi2d9", "gaussblur5x5", "laplacian3d7",
                                  "jacobi3d7", "wave13pt", "divergence", "gradient"])
def test_linearity_exact_on_small_integers(oracle, kind):
    ar = oracle.arity(kind)
    shape = (7, 8, 9) if ar["ndims"] == 3 else (11, 12)
    rng = np.random.default_rng(4)
    x = [rng.integers(-20, 20, size=shape).astype(np.float64) for _ in range(ar["n_in"])]
    y = [rng.integers(-20, 20, size=shape).astype(np.float64) for _ in range(ar["n_in"])]
    coeffs = np.array([0.5, -0.25, 0.125][: ar["ncoeffs"]]) if kind != "gaussblur5x5" else None

    def A(ins):
        outs = [np.zeros(shape) for _ in range(ar["n_out"])]
        oracle.step(kind, "f64", ins, outs, coeffs=coeffs)
        return outs

    for a, b, c in zip(A([p + q for p, q in zip(x, y)]), A(x), A(y)):
        np.testing.assert_array_equal(a, b + c)


def test_run_pingpong_keeps_dirichlet_ring(oracle):
    rng = np.random.default_rng(8)
    f = rng.uniform(size=(12, 14))
    bufs = [f.copy(), np.zeros_like(f)]
    idx = oracle.run("jacobi2d5", "f64", bufs, 3)
    assert idx == 1
    ring = np.ones(f.shape, bool)
    ring[1:-1, 1:-1] = False
    np.testing.assert_array_equal(bufs[0][ring], f[ring])
    np.testing.assert_array_equal(bufs[1][ring], f[ring])
    # 3 sweeps of a row-constant field with zero... invariant: constant field
    c = np.full((12, 14), 2.0)
    bufs = [c.copy(), np.zeros_like(c)]
    idx = oracle.run("jacobi2d9", "f64", bufs, 4, coeffs=[0.25, 0.125, 0.0625])
    np.testing.assert_array_equal(bufs[idx], c)


def test_run_wave13pt_rotation_conserves_linear_field(oracle):
    shape = (9, 9, 9)
    k, j, i = _ij(shape)
    f = 0.5 * i + 0.25 * j - k
    bufs = [f.copy(), f.copy(), np.zeros(shape)]
    idx = oracle.run("wave13pt", "f64", bufs, 5)
    assert idx == (1 + 5) % 3
    np.testing.assert_allclose(bufs[idx], f, rtol=0, atol=1e-12)


def test_errors_are_reported(oracle):
    f = np.zeros((4, 4), np.float32)
    with pytest.raises(ValueError):
        oracle.step("nosuchkind", "f32", [f], [f.copy()])
    with pytest.raises(ValueError):
        oracle.step("gameoflife", "f32", [f], [f.copy()])
    with pytest.raises(ValueError):
        oracle.step("gaussblur5x5", "f32", [f], [f.copy()])   # 4 < lo+hi+1 = 5
    with pytest.raises(ValueError):
        oracle.step("jacobi2d5", "f32", [f], [f.copy()], coeffs=[1.0, 2.0, 3.0])
