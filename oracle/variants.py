"""Dense approximate-augmented-space oracles (TEST INFRASTRUCTURE ONLY).

GKL: Alg 5.  RPI: Alg 7.  Cores and updates:
App D.3, PAPER.md:933-971 ("Add columns / Update weights with approximated augmented
space"); add rows is the transpose (as in zha_simon.add_rows).

Z is applied as an operator x -> E x - U (U^T E x) (matrix-free; the paper times its
baselines as the best of direct and matrix-free Z), so the oracle
also runs at sizes where the dense augmented matrix does not fit.

Readings (DESIGN.md §"Readings"):
  * GKL's H is l x (l+1): H[i,i] = α_i, H[i,i+1] = β_i, so P = P_{l+1} H^T is s x l and
    Q^T Z = P^T (PAPER.md:834-835 prints shapes that do not compose).
  * Q has the lift side's row count (PAPER.md:821 says n x l).
  * RPI's random start is passed in (Omega, s x l); P is orthonormalised at the top of
    each iteration exactly as Alg 7 line 4.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import la
from .zha_simon import _svd


class AugmentedOp:
    """Z = (I - X X^T) E with E given as s sparse update vectors (CSR rows, s x d).

    Z is d x s.  matvec/matmat: Z p;  rmatmat: Z^T q."""

    def __init__(self, X, ET):
        self.X = X
        self.ET = sp.csr_matrix(ET)          # s x d
        self.E = self.ET.T.tocsr()           # d x s
        self.C0 = (self.ET @ X).T            # k x s  = X^T E

    def mat(self, P):                        # d x l
        return self.E @ P - self.X @ (self.C0 @ P)

    def rmat(self, Q):                       # s x l
        return self.ET @ Q - self.C0.T @ (self.X.T @ Q)


def rpi_dense(Zop: AugmentedOp, Omega: np.ndarray, t: int):
    """Alg 7: for i=1..t: P,R=QR(P); Q=ZP; Q,R=QR(Q); P=Z^T Q."""
    P = np.array(Omega, dtype=np.float64, copy=True)
    Q = None
    for _ in range(t):
        P, _ = la.qr(P)
        Q = Zop.mat(P)
        Q, _ = la.qr(Q)
        P = Zop.rmat(Q)
    return Q, P


def gkl_dense(Zop: AugmentedOp, p1: np.ndarray, l: int):
    """Alg 5 with full reorthogonalisation of p (line 9) and the
    l x (l+1) reading of H.  Returns Q (d x l), P = P_{l+1} H^T (s x l)."""
    s = p1.size
    d = Zop.X.shape[0]
    Pm = np.zeros((s, l + 1))
    Qm = np.zeros((d, l))
    alpha = np.zeros(l)
    beta = np.zeros(l)
    Pm[:, 0] = p1 / np.linalg.norm(p1)
    q_prev = np.zeros(d)
    b_prev = 0.0
    for i in range(l):
        q = Zop.mat(Pm[:, i:i + 1])[:, 0] - b_prev * q_prev          # line 4
        alpha[i] = np.linalg.norm(q)                                  # line 5
        q = q / alpha[i]                                              # line 6
        p = Zop.rmat(q[:, None])[:, 0] - alpha[i] * Pm[:, i]          # line 7
        p = p - Pm[:, :i + 1] @ (Pm[:, :i + 1].T @ p)                 # line 8 (orthogonalise)
        beta[i] = np.linalg.norm(p)                                   # line 9
        Pm[:, i + 1] = p / beta[i]                                    # line 10
        Qm[:, i] = q
        q_prev, b_prev = q, beta[i]
    H = np.zeros((l, l + 1))
    H[np.arange(l), np.arange(l)] = alpha
    H[np.arange(l), np.arange(1, l + 1)] = beta
    return Qm, Pm @ H.T


def _basis(mode, Zop, sketch, l, t):
    if mode == "rpi":
        return rpi_dense(Zop, sketch, t)
    if mode == "gkl":
        return gkl_dense(Zop, sketch, l)
    raise ValueError(mode)


def add_columns(U, S, V, EcT, mode, sketch, l=10, t=3):
    """App D.3 'Add columns with approximated augmented space':
    K = [[Σ, U^T E], [0, P^T]] ((k+l) x (k+s));  U ← [U Q] F;  V ← [[V,0],[0,I]] G."""
    k = S.size
    Zop = AugmentedOp(U, EcT)
    Q, P = _basis(mode, Zop, sketch, l, t)
    s = EcT.shape[0]
    lq = Q.shape[1]
    K = np.zeros((k + lq, k + s))
    K[:k, :k] = np.diag(S)
    K[:k, k:] = Zop.C0
    K[k:, k:] = P.T
    F, th, G = _svd(K)
    Un = np.hstack([U, Q]) @ F[:, :k]
    Vn = np.vstack([V @ G[:k, :k], G[k:, :k]])
    return Un, th[:k].copy(), Vn, th


def add_rows(U, S, V, Er, mode, sketch, l=10, t=3):
    """Transpose of add_columns (lift on the V side, append on the U side)."""
    Vn, Sn, Un, th = add_columns(V, S, U, Er, mode, sketch, l, t)
    return Un, Sn, Vn, th


def update_weights(U, S, V, DT, EmT, mode, sketch_D, sketch_E, l=10, t=3):
    """App D.3 'Update weights with approximated augmented space':
    K = diag(Σ,0) + [U^T D; P_D^T][V^T E; P_E^T]^T  ((k+l) x (k+l))."""
    k = S.size
    ZD = AugmentedOp(U, DT)
    ZE = AugmentedOp(V, EmT)
    QD, PD = _basis(mode, ZD, sketch_D, l, t)
    QE, PE = _basis(mode, ZE, sketch_E, l, t)
    LD = np.vstack([ZD.C0, PD.T])
    LE = np.vstack([ZE.C0, PE.T])
    K = LD @ LE.T
    K[:k, :k] += np.diag(S)
    F, th, G = _svd(K)
    Un = np.hstack([U, QD]) @ F[:, :k]
    Vn = np.hstack([V, QE]) @ G[:, :k]
    return Un, th[:k].copy(), Vn, th
