"""Counter-based Gaussian generator — the random start blocks of the
approximate augmented space (RPI Ω; GKL p1) when
they are not passed in explicitly.

An input generator, not method arithmetic: it serves the oracle side, and the CUDA path
implements the same published spec independently (csrc/variants.cu K12).  Element (i, j)
of the s x l block of side `side` (0 = U side, 1 = V side) under `seed`:

    c  = (side << 60) | (i << 20) | j                       (i < 2^40, j < 2^20)
    z1 = splitmix64(seed ^ 2c),  z2 = splitmix64(seed ^ (2c + 1))
    u1 = ((z1 >> 11) + 0.5) 2^-53,  u2 = (z2 >> 11) 2^-53
    x  = sqrt(-2 ln u1) cos(2 pi u2)                         (Box–Muller)

splitmix64(x): x += 0x9E3779B97F4A7C15; z = (x ^ x>>30) * 0xBF58476D1CE4E5B9;
z = (z ^ z>>27) * 0x94D049BB133111EB; return z ^ z>>31   (all mod 2^64).
"""
from __future__ import annotations

import numpy as np

_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        z = x
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def counter_gaussian(seed: int, side: int, s: int, l: int) -> np.ndarray:
    """s x l row-major standard-normal block."""
    i = np.arange(s, dtype=np.uint64)[:, None]
    j = np.arange(l, dtype=np.uint64)[None, :]
    c = (np.uint64(side) << np.uint64(60)) | (i << np.uint64(20)) | j
    sd = np.uint64(seed)
    with np.errstate(over="ignore"):
        z1 = _splitmix64(sd ^ (c * np.uint64(2)))
        z2 = _splitmix64(sd ^ (c * np.uint64(2) + np.uint64(1)))
    u1 = ((z1 >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
    u2 = (z2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
