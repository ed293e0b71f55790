"""Plain definitions of the intermediate quantities on the path (TEST INFRASTRUCTURE ONLY).

Used by kernel-level parity tests (tests/test_gpu_kernels.py) to check one step of the
CUDA path at a time.  Each is the textbook definition written out, citing the passage.

Notation: the update block is E^T stored as s sparse rows (s x d), X' the
lift-side base factor (d x k) and M_X its k x k multiplier (Eq (4)),
so X = X' M_X.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def lift(ET, Xp, MX):
    """Lemma 1 under the extended decomposition:
    W = E^T X' (s x k, a gather of the X' rows E touches) and C0^T = W M_X = E^T X."""
    ET = sp.csr_matrix(ET)
    W = np.asarray(ET @ Xp)
    return W, W @ MX


def sparse_gram(ET):
    """Lemma 2 inner product of the raw sparse parts: (E^T E)_{ij} = <e_i, e_j>."""
    ET = sp.csr_matrix(ET)
    return np.asarray((ET @ ET.T).toarray())


def svlcov_gram(ET, C0T):
    """Gram of the SV-LCOV tuples (e_i, c_i): <e_i,e_j> - <c_i,c_j> (Lemma 2)."""
    return sparse_gram(ET) - C0T @ C0T.T


def chol_deflate(G, enorm2, tau=1e-12):
    """Cholesky G = R^T R (R upper, R_ii >= 0) in outer-product order, with the deflation
    reading of Alg 2's unguarded division (R8/R9): pivot i is deflated when its
    Schur-complement diagonal d_i <= tau * ||e_i||^2 or ||e_i|| = 0; its row of R is 0.

    Alg 2 computes the same R in exact arithmetic (row i of R holds
    <q_i, q_j>, which is what the Gram's Cholesky factor holds)."""
    A = np.array(G, dtype=np.float64, copy=True)
    s = A.shape[0]
    R = np.zeros((s, s))
    keep = np.zeros(s, dtype=bool)
    for i in range(s):
        d = A[i, i]
        if enorm2[i] == 0.0 or d <= tau * enorm2[i]:
            continue
        keep[i] = True
        R[i, i] = np.sqrt(d)
        R[i, i + 1:] = A[i, i + 1:] / R[i, i]
        A[i + 1:, i + 1:] -= np.outer(R[i, i + 1:], R[i, i + 1:])
    return R, keep


def core_rows(S, C0T, R, keep):
    """Alg 9 line 2 (block read as E_r V_k):
    K = [[Σ, 0], [E_r V_k, R^T]] with the zero columns of deflated pivots dropped:
    (k+s) x (k+r)."""
    k = S.size
    s = C0T.shape[0]
    r = int(keep.sum())
    K = np.zeros((k + s, k + r))
    K[:k, :k] = np.diag(S)
    K[k:, :k] = C0T
    K[k:, k:] = R[keep].T
    return K


def core_weights(S, C0T_D, R_D, keep_D, C0T_E, R_E, keep_E):
    """Alg 4 line 3: diag(Σ,0) + [U^T D; R_D][V^T E; R_E]^T, deflated
    rows of R dropped: (k+r_D) x (k+r_E)."""
    k = S.size
    LD = np.vstack([C0T_D.T, R_D[keep_D]])
    LE = np.vstack([C0T_E.T, R_E[keep_E]])
    K = LD @ LE.T
    K[:k, :k] += np.diag(S)
    return K


def cond1(M):
    """1-norm condition number ||M||_1 ||M^-1||_1 (the MII reset test, R18)."""
    return float(np.linalg.norm(M, 1) * np.linalg.norm(np.linalg.inv(M), 1))
