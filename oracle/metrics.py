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


def sigma_relerr(s_test, s_ref, floor_frac=1e-3) -> float:
    """max_i |σ_i - σ_i^ref| / max(σ_i^ref, floor_frac·σ_1^ref).

    With the 1e-10 tolerance this is SURVEY §8(c)'s rule |Δσ_i| <= max(1e-10 σ_i,
    1e-13 σ_1): relative below the tolerance for σ_i >= 1e-3 σ_1, and an absolute floor
    of 1e-13 σ_1 (= 1e-10 x 1e-3 σ_1) for the tiny ones (σ_k -> 0)."""
    s_test = np.asarray(s_test, dtype=np.float64)
    s_ref = np.asarray(s_ref, dtype=np.float64)
    if s_ref.size == 0:
        return 0.0
    s1 = max(float(s_ref[0]), 1e-300)
    den = np.maximum(s_ref, floor_frac * s1)
    n = min(s_test.size, s_ref.size)
    return float(np.max(np.abs(s_test[:n] - s_ref[:n]) / den[:n])) if n else 0.0


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
