"""Parity metrics (TEST INFRASTRUCTURE ONLY).  BASELINE.json north_star tolerances:
singular values within 1e-10 relative; sin of the largest principal angle between the
GPU and oracle U_k / V_k subspaces below 1e-8.
"""
from __future__ import annotations

import numpy as np


def orthonormalize(X):
    q, _ = np.linalg.qr(np.asarray(X, dtype=np.float64))
    return q


def sin_theta(X, Y) -> float:
    """sin θ_max between range(X) and range(Y) as ||Y - X (X^T Y)||_2 with X, Y
    orthonormalised by fp64 QR.  Never sqrt(1 - cos^2): that has a ~1.5e-8 floor
    (SURVEY §0.4)."""
    X = orthonormalize(X)
    Y = orthonormalize(Y)
    Mres = Y - X @ (X.T @ Y)
    r = np.linalg.qr(Mres, mode="r")
    return float(np.linalg.norm(r, 2)) if r.size else 0.0


def sigma_relerr(s_test, s_ref, floor_frac=1e-3, abs_floor=1e-13) -> float:
    """max_i |σ_i - σ_i^ref| / σ_i^ref; for σ_i^ref < floor_frac σ_1 the error is taken
    relative to σ_1 with an absolute floor abs_floor σ_1."""
    s_test = np.asarray(s_test, dtype=np.float64)
    s_ref = np.asarray(s_ref, dtype=np.float64)
    s1 = max(float(s_ref[0]), 1e-300) if s_ref.size else 1.0
    err = 0.0
    for a, b in zip(s_test, s_ref):
        if b >= floor_frac * s1:
            e = abs(a - b) / b
        else:
            e = max(abs(a - b) - abs_floor * s1, 0.0) / s1
        err = max(err, e)
    return err


def gap_rank(theta_all, k, min_gap=1e-6) -> int:
    """Largest k' <= k with relative gap (θ_k' - θ_k'+1)/θ_k' >= min_gap: the leading
    subspace that is unique and therefore pinned (SURVEY §8(c) gap guard)."""
    th = np.asarray(theta_all, dtype=np.float64)
    th = np.concatenate([th, np.zeros(max(0, k + 1 - th.size))])
    for kk in range(k, 0, -1):
        if th[kk - 1] > 0 and (th[kk - 1] - th[kk]) / th[kk - 1] >= min_gap:
            return kk
    return 0


def orth_err(X) -> float:
    X = np.asarray(X)
    return float(np.abs(X.T @ X - np.eye(X.shape[1])).max())
