"""Pins of the counter-based Gaussian generator spec on the host."""
import numpy as np

from synth import counter_rng


def test_splitmix64_reference_vector():
    """SplitMix64 from state 0: the published first output 0xE220A8397B1DCDAF."""
    out = counter_rng._splitmix64(np.array([0], dtype=np.uint64))
    assert int(out[0]) == 0xE220A8397B1DCDAF


def test_gaussian_moments_and_determinism():
    a = counter_rng.counter_gaussian(7, 0, 2000, 100)
    assert np.array_equal(a, counter_rng.counter_gaussian(7, 0, 2000, 100))
    assert abs(a.mean()) < 0.01 and abs(a.var() - 1) < 0.01
    assert abs((a ** 4).mean() - 3) < 0.05                    # Gaussian kurtosis
    b = counter_rng.counter_gaussian(7, 1, 2000, 100)
    assert abs(np.corrcoef(a.ravel(), b.ravel())[0, 1]) < 0.01   # sides are independent streams


def test_prefix_property():
    """Element (i, j) depends only on (seed, side, i, j): a sub-block is a prefix."""
    a = counter_rng.counter_gaussian(3, 1, 50, 20)
    b = counter_rng.counter_gaussian(3, 1, 30, 5)
    assert np.array_equal(a[:30, :5], b)
