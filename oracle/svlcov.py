"""SV-LCOV tuple algebra and the two orthogonalisers of §3.1 (TEST INFRASTRUCTURE ONLY).

Def 1: (b, c)_{U_k} with c = U_k^T b represents z = (I - U_k U_k^T) b.
Lemma 2: scale, add, inner product <(b1,c1),(b2,c2)> = b1.b2 - c1.c2.
Alg 1: dense modified Gram–Schmidt on the densified augmented matrix.
Alg 2: the same MGS run on tuples.

Pure-Python loops, dense numpy vectors: for the small cases of the pin tests only.

Reading (R8/R9): Alg 2 divides by α with no guard.  A
vector whose remaining squared length α² <= tau * ||e_i||² (or whose input is empty)
is *deflated*: R[i, :] = 0 and the tuple is zeroed, so it contributes nothing later.
A negative α² from rounding is clamped to 0 and deflated.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def lift(E, U):
    """Lemma 1: columns of E (m x s) -> tuples (B = E, C = U^T E)."""
    Ed = E.toarray() if sp.issparse(E) else np.asarray(E, dtype=np.float64)
    return Ed.copy(), U.T @ Ed


def materialize(b, c, U):
    """Def 1: (b, c)_{U} -> b - U c."""
    return b - U @ c


def dot(b1, c1, b2, c2):
    """Lemma 2 inner product: <b1,b2> - <c1,c2>."""
    return float(b1 @ b2 - c1 @ c2)


def alg1_mgs(E, U):
    """Alg 1, line by line (no deflation: full column rank inputs)."""
    Ed = E.toarray() if sp.issparse(E) else np.asarray(E, dtype=np.float64)
    Q = Ed - U @ (U.T @ Ed)                           # line 1
    s = Q.shape[1]
    R = np.zeros((s, s))
    for i in range(s):                                # line 2
        alpha = np.sqrt(Q[:, i] @ Q[:, i])            # line 3
        R[i, i] = alpha                               # line 4
        Q[:, i] = Q[:, i] / alpha                     # line 5
        for j in range(i + 1, s):                     # line 6
            beta = Q[:, i] @ Q[:, j]                  # line 7
            R[i, j] = beta                            # line 8
            Q[:, j] = Q[:, j] - beta * Q[:, i]        # line 9
    return Q, R


def alg2_svlcov_qr(E, U, tau: float = 1e-12):
    """Alg 2, line by line on tuples, with the deflation reading.

    Returns B (m x s), C (k x s), R (s x s upper, zero rows for deflated), keep (bool s)."""
    B, C = lift(E, U)                                  # line 1
    s = B.shape[1]
    norms2 = np.einsum("ij,ij->j", B, B)               # ||e_i||^2 of the input vectors
    R = np.zeros((s, s))
    keep = np.zeros(s, dtype=bool)
    for i in range(s):                                 # line 2
        a2 = dot(B[:, i], C[:, i], B[:, i], C[:, i])   # line 3 (radicand)
        if norms2[i] == 0.0 or a2 <= tau * norms2[i]:
            B[:, i] = 0.0
            C[:, i] = 0.0
            continue                                   # deflated: R[i, :] stays 0
        keep[i] = True
        alpha = np.sqrt(a2)
        R[i, i] = alpha                                # line 4
        B[:, i] /= alpha                               # line 5
        C[:, i] /= alpha
        for j in range(i + 1, s):                      # line 6
            beta = dot(B[:, i], C[:, i], B[:, j], C[:, j])   # line 7
            R[i, j] = beta                             # line 8
            B[:, j] -= beta * B[:, i]                  # line 9
            C[:, j] -= beta * C[:, i]
    return B, C, R, keep
