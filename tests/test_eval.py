"""F2 evaluation helpers (host, -m "not gpu"): AP and MSE against their definitions."""
import itertools

import numpy as np

from paper_2401_09703_b200 import evaluate as ev


def test_average_precision_brute_force():
    rng = np.random.default_rng(0)
    for _ in range(20):
        n = int(rng.integers(1, 12))
        s = rng.standard_normal(n)
        y = rng.random(n) < 0.5
        if not y.any():
            assert ev.average_precision(s, y) == 0.0
            continue
        order = sorted(range(n), key=lambda i: (-s[i], i))
        precs = []
        for r, i in enumerate(order, 1):
            if y[i]:
                precs.append(sum(y[j] for j in order[:r]) / r)
        assert np.isclose(ev.average_precision(s, y), np.mean(precs))


def test_average_precision_extremes():
    assert ev.average_precision([3, 2, 1, 0], [1, 1, 0, 0]) == 1.0
    assert np.isclose(ev.average_precision([3, 2, 1, 0], [0, 0, 1, 1]), (1 / 3 + 2 / 4) / 2)


def test_mse():
    assert ev.mse([1, 2, 3], [1, 2, 5]) == 4 / 3
    assert ev.mse([], []) == 0.0
