"""Shared helpers for the GPU parity tests (tests only)."""
from __future__ import annotations

import numpy as np

from oracle import metrics, zha_simon

# BASELINE.json north_star tolerances (fp64)
SIGMA_TOL = 1e-10
ANGLE_TOL = 1e-8


def compare(Ug, Sg, Vg, Uo, So, Vo, theta_all, k, sigma_tol=SIGMA_TOL, angle_tol=ANGLE_TOL):
    """σ within sigma_tol relative; sin θ_max of U_k', V_k' below angle_tol, where k' <= k
    is the largest leading block with a relative gap >= 1e-6 (gap guard)."""
    es = metrics.sigma_relerr(Sg, So)
    kk = metrics.gap_rank(theta_all, k)
    eu = metrics.sin_theta(Ug[:, :kk], Uo[:, :kk]) if kk else 0.0
    ev = metrics.sin_theta(Vg[:, :kk], Vo[:, :kk]) if kk else 0.0
    ok = es <= sigma_tol and eu <= angle_tol and ev <= angle_tol
    return ok, dict(sigma=es, angle_u=eu, angle_v=ev, kk=kk)


def run_oracle(w, n_batches=None):
    U, S, V = w.U0.copy(), w.S0.copy(), w.V0.copy()
    out = []
    for b in w.batches[:n_batches]:
        U, S, V, th = zha_simon.apply_batch(U, S, V, b)
        out.append((U, S, V, th))
    return out


def gpu_state(P, w, device="cuda"):
    import torch
    m, n = w.final_dims()
    t = P.TSVD(w.k, m_capacity=m, n_capacity=n)
    t.init(torch.from_numpy(w.U0).to(device), torch.from_numpy(w.S0).to(device), torch.from_numpy(w.V0).to(device))
    return t


def gpu_apply(P, t, b, opts=None, device="cuda"):
    E = P.Sparse.from_scipy(b.E, device=device)
    D = P.Sparse.from_scipy(b.D, device=device) if b.D is not None else None
    t.update(b.kind, E, D, opts)


def gpu_factors(t):
    return t.get_U(), t.get_S(), t.get_V()
