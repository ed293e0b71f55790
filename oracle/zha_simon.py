"""Exact update oracle: Zha–Simon dense augmented projection (TEST INFRASTRUCTURE ONLY).

PAPER.md:86-116 (Eq 1, add columns), PAPER.md:118-160 (Eq 2, update weights); add rows
is Eq (1) applied to the transpose (Theorem 1 'Add rows'; Alg 9
PAPER.md:1186-1201 with the core block read as E_r V_k).

All inputs fp64.  U: m x k, S: (k,), V: n x k (orthonormal columns, S descending).
Sparse update blocks use the library's convention of s update vectors stored as CSR
rows:  rows -> E_r (s x n);  cols -> E_c^T (s x m);  weights -> D^T (s x m), E_m^T (s x n).

Each function returns (U_new, S_new, V_new, theta_all) with theta_all the full
singular spectrum of the core (for the gap guard and the energy pin).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import la


def _dense(X) -> np.ndarray:
    return X.toarray() if sp.issparse(X) else np.asarray(X, dtype=np.float64)


def _svd(K):
    """Dense LAPACK SVD of the core (gesdd, falling back to gesvd on non-convergence)."""
    try:
        F, th, Gt = sla.svd(K, full_matrices=False, lapack_driver="gesdd")
    except np.linalg.LinAlgError:  # pragma: no cover
        F, th, Gt = sla.svd(K, full_matrices=False, lapack_driver="gesvd")
    return F, th, Gt.T


def add_columns(U, S, V, EcT):
    """Eq (1), verbatim.

    (I - U_k U_k^T) E_c = Q R                       (dense Householder QR)
    K = [[Σ_k, U_k^T E_c], [0, R]]                  ((k+q) x (k+s))
    F, Θ, G = SVD(K)
    U ← [U_k Q] F[:, :k],  Σ ← Θ[:k],  V ← [[V_k, 0], [0, I]] G[:, :k]
    """
    k = S.size
    Ec = _dense(EcT).T                       # m x s
    s = Ec.shape[1]
    C0 = U.T @ Ec                            # k x s
    Z = Ec - U @ C0                          # augmented matrix
    Q, R = la.qr(Z)                          # m x q, q x s (Householder)
    q = Q.shape[1]
    K = np.zeros((k + q, k + s))
    K[:k, :k] = np.diag(S)
    K[:k, k:] = C0
    K[k:, k:] = R
    F, th, G = _svd(K)
    Un = np.hstack([U, Q]) @ F[:, :k]
    Vn = np.vstack([V @ G[:k, :k], G[k:, :k]])
    return Un, th[:k].copy(), Vn, th


def add_rows(U, S, V, Er):
    """Theorem 1 'Add rows' = Eq (1) on the transpose [Ã; E_r]^T = [Ã^T, E_r^T].

    (I - V V^T) E_r^T = Q R;  K = [[Σ, 0], [E_r V, R^T]]  ((k+s) x (k+q))
    U ← [[U, 0], [0, I]] F[:, :k],  V ← [V Q] G[:, :k]
    """
    Vn, Sn, Un, th = add_columns(V, S, U, Er)
    return Un, Sn, Vn, th


def update_weights(U, S, V, DT, EmT):
    """Eq (2), verbatim.

    (I - U U^T) D = Q_D R_D,  (I - V V^T) E_m = Q_E R_E
    K = [[Σ, 0], [0, 0]] + [U^T D; R_D] [V^T E_m; R_E]^T
    U ← [U Q_D] F[:, :k],  Σ ← Θ[:k],  V ← [V Q_E] G[:, :k]
    """
    k = S.size
    D = _dense(DT).T                         # m x s
    Em = _dense(EmT).T                       # n x s
    C0D = U.T @ D
    C0E = V.T @ Em
    QD, RD = la.qr(D - U @ C0D)
    QE, RE = la.qr(Em - V @ C0E)
    LD = np.vstack([C0D, RD])                # (k+qD) x s
    LE = np.vstack([C0E, RE])                # (k+qE) x s
    K = LD @ LE.T
    K[:k, :k] += np.diag(S)
    F, th, G = _svd(K)
    Un = np.hstack([U, QD]) @ F[:, :k]
    Vn = np.hstack([V, QE]) @ G[:, :k]
    return Un, th[:k].copy(), Vn, th


def apply_batch(U, S, V, batch):
    """Dispatch on synth.Batch.kind."""
    if batch.kind == "rows":
        return add_rows(U, S, V, batch.E)
    if batch.kind == "cols":
        return add_columns(U, S, V, batch.E)
    if batch.kind == "weights":
        return update_weights(U, S, V, batch.D, batch.E)
    raise ValueError(batch.kind)


def reconstruct(U, S, V):
    """Ã = U Σ V^T (dense)."""
    return (U * S) @ V.T
