"""Dense LAPACK primitives of the oracle (TEST INFRASTRUCTURE ONLY).

`qr(Z)` is the reduced Householder QR `numpy.linalg.qr(Z)` computes (LAPACK geqrf +
orgqr): Z = Q R, Q with orthonormal columns, R upper triangular.  For tall inputs it is
taken from PyTorch's CPU LAPACK (the same geqrf/orgqr, MKL-threaded) instead of numpy's
OpenBLAS build, whose QR runs ~10x slower on 1e5-1e6-row blocks (configs[1]'s 50000 x 5000
augmented block, configs[3]'s 1e6 x 256 RPI block).  Same definition, a faster library
call; plain CPU ops only.
"""
from __future__ import annotations

import numpy as np

_BIG = 20_000_000   # elements above which the torch CPU LAPACK is used


def qr(Z):
    Z = np.asarray(Z, dtype=np.float64)
    if Z.size < _BIG:
        return np.linalg.qr(Z)
    import torch
    q, r = torch.linalg.qr(torch.from_numpy(np.ascontiguousarray(Z)), mode="reduced")
    return q.numpy(), r.numpy()
