"""Pins of the oracle's SURVEY §8(f) row-f3 kinds (DESIGN.md §3 R19-R22):
tricubic2, uxx1, lapgsrb, whispering.

As in test_oracle_pins.py, nothing here re-types the oracle's formula: each
test checks a closed form, an invariant, or a textbook algorithm that
reaches the same result by a different route (the in-place red-black
Gauss-Seidel sweep for lapgsrb, the unfused two-half-step Yee leapfrog for
whispering), exact in fp64 on integer data with dyadic weights.  Table 1
counts for these kinds are pinned in test_oracle_pins.py.
"""
import numpy as np
import pytest


def _ij(shape):
    return np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")


# ------------------------------------------------------------ tricubic2
def _tri_inputs(shape, X, Y, Z, f):
    return [f] + [np.full(shape, t) if np.isscalar(t) else t for t in (X, Y, Z)]


def test_tricubic2_special_offsets_exact(oracle):
    """Cardinality of the Lagrange weights: t = 0 selects node 0, t = 1 node
    +1; every expanded term is then an exact 0 or 1 times a sample."""
    rng = np.random.default_rng(12)
    shape = (7, 8, 9)
    f = rng.uniform(size=shape)
    out = np.zeros(shape)
    for t, sl in ((0.0, (slice(1, -2),) * 3), (1.0, (slice(2, -1),) * 3)):
        oracle.step("tricubic2", "f64", _tri_inputs(shape, t, t, t, f), [out])
        np.testing.assert_array_equal(out[1:-2, 1:-2, 1:-2], f[sl])
    oracle.step("tricubic2", "f64", _tri_inputs(shape, 0.0, 1.0, 0.0, f), [out])   # Y moves y only
    np.testing.assert_array_equal(out[1:-2, 1:-2, 1:-2], f[1:-2, 2:-1, 1:-2])


def test_tricubic2_reproduces_cubic_polynomials(oracle):
    """Exact (to rounding) on a product of cubics, distinct per axis."""
    rng = np.random.default_rng(6)
    shape = (8, 9, 10)
    k, j, i = _ij(shape)
    p = np.polynomial.Polynomial([0.2, -0.9, 0.3, 0.04])
    q = np.polynomial.Polynomial([1.1, 0.4, -0.25, 0.02])
    r = np.polynomial.Polynomial([-0.6, 0.3, 0.05, -0.02])
    X, Y, Z = (rng.uniform(size=shape) for _ in range(3))
    out = np.zeros(shape)
    oracle.step("tricubic2", "f64", _tri_inputs(shape, X, Y, Z, p(i) * q(j) * r(k)), [out])
    exp = p(i + X) * q(j + Y) * r(k + Z)
    sl = (slice(1, -2),) * 3
    np.testing.assert_allclose(out[sl], exp[sl], rtol=1e-12, atol=1e-12)


def test_tricubic2_partition_of_unity(oracle):
    rng = np.random.default_rng(13)
    shape = (6, 6, 6)
    X, Y, Z = (rng.uniform(size=shape) for _ in range(3))
    out = np.zeros(shape)
    oracle.step("tricubic2", "f64", _tri_inputs(shape, X, Y, Z, np.full(shape, -2.5)), [out])
    np.testing.assert_allclose(out[1:-2, 1:-2, 1:-2], -2.5, rtol=1e-14)


# ----------------------------------------------------------------- uxx1
UXX1 = [0.25, 9 / 8, -1 / 24]


def _uxx1(oracle, shape, u1, d1, xx, xy, xz, coeffs=UXX1, dtype="f64"):
    out = np.zeros(shape)
    oracle.step("uxx1", dtype, [u1, d1, xx, xy, xz], [out], coeffs=coeffs)
    return out[2:-1, 2:-1, 2:-1]


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_uxx1_linear_stress_per_axis(oracle, axis):
    """A linear stress along one axis only (xx = 3i, or xy = 3j, or xz = 3k):
    both differences see the slope (the c2 term over a distance of 3), so
    out = u1 + dth * 3 * (c1 + 3 c2) = u1 + 0.75 exactly with c1 + 3 c2 = 1.
    With distinct c1 / c2 the result names which difference carries which
    weight: (c1, c2) = (1/2, 1/4) gives u1 + dth*3*(1/2 + 3/4)."""
    shape = (7, 8, 9)
    k, j, i = _ij(shape)
    z = np.zeros(shape)
    u1 = 5.0 * i - 2.0 * j + k
    stress = [z, z, z]
    stress[axis] = 3.0 * (i, j, k)[axis]
    got = _uxx1(oracle, shape, u1, np.ones(shape), *stress)
    np.testing.assert_array_equal(got, u1[2:-1, 2:-1, 2:-1] + 0.75)
    got = _uxx1(oracle, shape, u1, np.ones(shape), *stress, coeffs=[0.25, 0.5, 0.25])
    np.testing.assert_array_equal(got, u1[2:-1, 2:-1, 2:-1] + 0.25 * 3 * (0.5 + 0.75))


def test_uxx1_staggered_derivative_of_a_cubic(oracle):
    """c1 = 9/8, c2 = -1/24 is the 4th-order staggered first derivative,
    exact on cubics at the half point i - 1/2: xx = i^3 gives
    out = u1 + dth * 3 (i - 1/2)^2 (d1 = 1).  Pins the offsets i-2..i+1, the
    left stagger and the weight assignment (exact in fp64: the result is a
    multiple of 1/16)."""
    shape = (6, 6, 12)
    k, j, i = _ij(shape)
    z = np.zeros(shape)
    got = _uxx1(oracle, shape, z, np.ones(shape), i ** 3, z, z)
    np.testing.assert_array_equal(got, (0.25 * 3 * (i - 0.5) ** 2)[2:-1, 2:-1, 2:-1])
    got = _uxx1(oracle, shape, z, np.ones(shape), z, z, k ** 3)
    np.testing.assert_array_equal(got, (0.25 * 3 * (k - 0.5) ** 2)[2:-1, 2:-1, 2:-1])


def test_uxx1_density_average(oracle):
    """d1 linear in (j, k): d = 0.25*(d1[j][k] + d1[j-1][k] + d1[j][k-1] +
    d1[j-1][k-1]) = 2(j - 1/2) + 4(k - 1/2) + 64 + i, so with a unit stress
    slope in x, out = u1 + dth / d.  Checks the four density taps."""
    shape = (6, 7, 8)
    k, j, i = _ij(shape)
    z = np.zeros(shape)
    d1 = 2.0 * j + 4.0 * k + 64.0 + i
    got = _uxx1(oracle, shape, z, d1, i.copy(), z, z)
    d = 2.0 * (j - 0.5) + 4.0 * (k - 0.5) + 64.0 + i
    np.testing.assert_allclose(got, (0.25 / d)[2:-1, 2:-1, 2:-1], rtol=1e-15)


# -------------------------------------------------------------- lapgsrb
def _gsrb_inplace(u, w):
    """Textbook red-black Gauss-Seidel (in place, numpy): update every red
    interior point from its six neighbours, then every black one from the
    updated field; the boundary is held."""
    u = u.copy()
    nz, ny, nx = u.shape
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    inner = (i > 0) & (i < nx - 1) & (j > 0) & (j < ny - 1) & (k > 0) & (k < nz - 1)
    for colour in (0, 1):
        nb = np.zeros_like(u)
        c = (slice(1, -1),) * 3
        nb[c] = (u[1:-1, 1:-1, :-2] + u[1:-1, 1:-1, 2:] + u[1:-1, :-2, 1:-1] + u[1:-1, 2:, 1:-1]
                 + u[:-2, 1:-1, 1:-1] + u[2:, 1:-1, 1:-1])
        m = inner & (((i + j + k) & 1) == colour)
        u[m] = w * nb[m]
    return u


@pytest.mark.parametrize("shape", [(3, 3, 4), (6, 7, 9), (9, 8, 11)])
def test_lapgsrb_equals_inplace_red_black_sweep(oracle, shape):
    """One out-of-place lapgsrb step = one red-then-black in-place
    Gauss-Seidel iteration (exact: integer data, w = 1/8)."""
    rng = np.random.default_rng(sum(shape))
    u = rng.integers(-64, 64, size=shape).astype(np.float64)
    out = u.copy()
    oracle.step("lapgsrb", "f64", [u], [out], coeffs=[0.125])
    np.testing.assert_array_equal(out, _gsrb_inplace(u, 0.125))


def test_lapgsrb_run_equals_repeated_sweeps(oracle):
    rng = np.random.default_rng(3)
    u = rng.integers(-64, 64, size=(7, 8, 10)).astype(np.float64)
    bufs = [u.copy(), np.zeros_like(u)]
    idx = oracle.run("lapgsrb", "f64", bufs, 3, coeffs=[0.125])
    ref = u
    for _ in range(3):
        ref = _gsrb_inplace(ref, 0.125)
    np.testing.assert_array_equal(bufs[idx], ref)


def test_lapgsrb_harmonic_field_is_a_fixed_point(oracle):
    """A linear field is discrete-harmonic: the Gauss-Seidel update with
    w = 1/6 leaves it unchanged (to rounding of the 1/6 weight)."""
    shape = (8, 9, 10)
    k, j, i = _ij(shape)
    u = 3.0 * i - 2.0 * j + 0.5 * k + 7.0
    out = np.zeros(shape)
    oracle.step("lapgsrb", "f64", [u], [out])
    np.testing.assert_allclose(out[1:-1, 1:-1, 1:-1], u[1:-1, 1:-1, 1:-1], rtol=4e-16, atol=4e-15)


def test_lapgsrb_checkerboard_closed_form(oracle):
    """u = (-1)^(i+j+k): a red point's neighbours are all -1, so r = -6w;
    a black point's neighbours are red points with r = -6w, so out = -36 w^2
    (points whose red neighbours are all interior)."""
    shape = (9, 9, 10)
    k, j, i = _ij(shape)
    u = (-1.0) ** (i + j + k)
    out = np.zeros(shape)
    w = 0.125
    oracle.step("lapgsrb", "f64", [u], [out], coeffs=[w])
    red = ((i + j + k) % 2) == 0
    deep = (i >= 2) & (i <= shape[2] - 3) & (j >= 2) & (j <= shape[1] - 3) & (k >= 2) & (k <= shape[0] - 3)
    assert np.all(out[deep & red] == -6 * w)
    assert np.all(out[deep & ~red] == -36 * w * w)


# ----------------------------------------------------------- whispering
def _yee_two_half_steps(Hx, Hy, Ez, dax, dbx, day, dby, cb):
    """Textbook unfused TM-mode Yee leapfrog (numpy): the H half step on
    every cell that has its Ez neighbours, then the E step on the interior
    from the updated H."""
    Hx1, Hy1, Ez1 = Hx.copy(), Hy.copy(), Ez.copy()
    Hx1[:-1, :] = dax[:-1, :] * Hx[:-1, :] - dbx[:-1, :] * (Ez[1:, :] - Ez[:-1, :])
    Hy1[:, :-1] = day[:, :-1] * Hy[:, :-1] + dby[:, :-1] * (Ez[:, 1:] - Ez[:, :-1])
    Ez1[1:-1, 1:-1] = Ez[1:-1, 1:-1] + cb[1:-1, 1:-1] * (
        (Hy1[1:-1, 1:-1] - Hy1[1:-1, :-2]) - (Hx1[1:-1, 1:-1] - Hx1[:-2, 1:-1]))
    return Hx1, Hy1, Ez1


@pytest.mark.parametrize("shape", [(3, 4), (9, 12), (17, 13)])
def test_whispering_equals_unfused_yee_step(oracle, shape):
    """The fused step (neighbouring H recomputed inside the Ez update) equals
    the two half steps of the textbook scheme on the interior (exact: integer
    fields, dyadic material arrays)."""
    rng = np.random.default_rng(shape[0] * 31 + shape[1])
    Hx, Hy, Ez = (rng.integers(-32, 32, size=shape).astype(np.float64) for _ in range(3))
    dax, dbx, day, dby, cb = (rng.integers(-8, 9, size=shape) / 8.0 for _ in range(5))
    outs = [np.zeros(shape) for _ in range(3)]
    oracle.step("whispering", "f64", [Hx, Hy, Ez, dax, dbx, day, dby, cb], outs)
    ref = _yee_two_half_steps(Hx, Hy, Ez, dax, dbx, day, dby, cb)
    for o, r in zip(outs, ref):
        np.testing.assert_array_equal(o[1:-1, 1:-1], r[1:-1, 1:-1])


def test_whispering_linear_field_closed_form(oracle):
    """Ez = a i + b j, H = 0, da = 1, db = beta: H picks up the curl of Ez
    (Hx' = -beta b, Hy' = beta a) and Ez is unchanged (the curl of a uniform
    H is zero).  Distinct a, b pin the axes and the signs."""
    shape = (10, 12)
    j, i = _ij(shape)
    z, one = np.zeros(shape), np.ones(shape)
    beta, gamma, a, b = 0.25, 0.5, 3.0, -2.0
    outs = [np.zeros(shape) for _ in range(3)]
    oracle.step("whispering", "f64", [z, z, a * i + b * j, one, beta * one, one, beta * one, gamma * one], outs)
    sl = (slice(1, -1), slice(1, -1))
    assert np.all(outs[0][sl] == -beta * b) and np.all(outs[1][sl] == beta * a)
    np.testing.assert_array_equal(outs[2][sl], (a * i + b * j)[sl])


@pytest.mark.parametrize("axis", [0, 1])
def test_whispering_quadratic_field_closed_form(oracle, axis):
    """Ez = i^2 (or j^2), H = 0: the discrete curl-curl of the Yee scheme is
    the 5-point Laplacian, exact on quadratics: Ez' = Ez + 2 beta gamma."""
    shape = (10, 12)
    j, i = _ij(shape)
    z, one = np.zeros(shape), np.ones(shape)
    beta, gamma = 0.25, 0.5
    Ez = (i * i, j * j)[axis]
    outs = [np.zeros(shape) for _ in range(3)]
    oracle.step("whispering", "f64", [z, z, Ez, one, beta * one, one, beta * one, gamma * one], outs)
    sl = (slice(1, -1), slice(1, -1))
    np.testing.assert_array_equal(outs[2][sl], Ez[sl] + 2 * beta * gamma)
