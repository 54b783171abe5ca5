"""The device-side input generator equals the host one bit for bit."""
import numpy as np
import pytest

from paper_2301_11389_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["f32", "f64", "i32"])
def test_torch_cuda_generator_matches_numpy(dtype):
    shape = (37, 41, 66)
    a = inputs.generate_np(shape, dtype, inputs.BASE_SEED + 4, 1)
    b = inputs.generate_torch(shape, dtype, inputs.BASE_SEED + 4, 1, device="cuda",
                              chunk=10000).cpu().numpy()
    assert np.array_equal(a, b)
