"""The seeded input generator (paper_2301_11389_b200/inputs.py)."""
import numpy as np
import torch

from paper_2301_11389_b200 import inputs


def test_splitmix64_known_answer():
    """Reference splitmix64 (Steele/Lea/Flood; Vigna's splitmix64.c): seeded
    with 0, the first output is 0xE220A8397B1DCDAF, the second 0x6E789E6AA1B965F4."""
    with np.errstate(over="ignore"):
        x = np.array([1, 2], dtype=np.uint64) * np.uint64(inputs.GOLDEN)
        z = inputs._mix_np(x)
    assert int(z[0]) == 0xE220A8397B1DCDAF
    assert int(z[1]) == 0x6E789E6AA1B965F4


def test_ranges_and_determinism():
    a = inputs.generate_np((33, 17), "f32", 5)
    b = inputs.generate_np((33, 17), "f32", 5)
    assert a.dtype == np.float32 and np.array_equal(a, b)
    assert a.min() >= 0 and a.max() < 1
    d = inputs.generate_np((1000,), "f64", 5)
    assert d.min() >= 0 and d.max() < 1
    g = inputs.generate_np((100, 100), "i32", 5)
    assert set(np.unique(g)) == {0, 1} and 0.4 < g.mean() < 0.6
    assert not np.array_equal(inputs.generate_np((50,), "f32", 5, 0),
                              inputs.generate_np((50,), "f32", 5, 1))


def test_chunking_does_not_change_values():
    a = inputs.generate_np((1001,), "f64", 9, chunk=1 << 20)
    b = inputs.generate_np((1001,), "f64", 9, chunk=7)
    assert np.array_equal(a, b)


def test_torch_generator_matches_numpy_on_cpu():
    for dt in ("f32", "f64", "i32"):
        a = inputs.generate_np((5, 7, 9), dt, inputs.BASE_SEED + 3, 2)
        b = inputs.generate_torch((5, 7, 9), dt, inputs.BASE_SEED + 3, 2, device="cpu",
                                  chunk=50).numpy()
        assert np.array_equal(a, b), dt
