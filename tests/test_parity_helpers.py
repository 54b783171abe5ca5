"""Host-side checks of the parity machinery itself (CPU only)."""
import numpy as np

from paper_2301_11389_b200 import inputs
from parity import assert_parity, oracle_window_run


def test_window_run_equals_full_run(oracle):
    """The dependence-cone window reproduces the full-grid oracle run."""
    for kind, dtype, r, shape, n in [("gaussblur5x5", "f32", 2, (90, 120), 6),
                                     ("gameoflife", "i32", 1, (70, 80), 9),
                                     ("jacobi2d9", "f64", 1, (60, 64), 8)]:
        f = inputs.generate_np(shape, dtype, 11)
        bufs = [f.copy(), np.zeros_like(f)]
        idx = oracle.run(kind, dtype, bufs, n)
        for w in [(slice(0, 10), slice(0, 12)), (slice(30, 41), slice(50, 64)),
                  (slice(shape[0] - 8, shape[0]), slice(shape[1] - 20, shape[1]))]:
            got = oracle_window_run(oracle, kind, dtype, [f, np.zeros_like(f)], n, w, r)
            assert np.array_equal(got, bufs[idx][w]), (kind, w)


def test_wave_window_run_equals_full_run(oracle):
    shape = (30, 31, 32)
    prev = inputs.generate_np(shape, "f64", 1, 0)
    cur = inputs.generate_np(shape, "f64", 1, 1)
    bufs = [prev.copy(), cur.copy(), np.zeros(shape)]
    idx = oracle.run("wave13pt", "f64", bufs, 3)
    w = (slice(10, 16), slice(3, 9), slice(20, 28))
    got = oracle_window_run(oracle, "wave13pt", "f64", [prev, cur, np.zeros(shape)], 3, w, 2)
    assert np.array_equal(got, bufs[idx][w])


def test_assert_parity_floor_metric():
    r = np.array([1.0, -1.0, 1e-9], np.float32)
    assert_parity(r + np.float32(5e-6) * np.sign(r), r, "f32")     # within 1e-5 relative
    g = r.copy()
    g[2] = 5e-6                                                     # under the floor S*tol
    assert_parity(g, r, "f32")
    g[0] = 1.0001
    try:
        assert_parity(g, r, "f32")
        raise RuntimeError("should have failed")
    except AssertionError:
        pass
    assert_parity(np.array([3], np.int32), np.array([3], np.int32), "i32")
