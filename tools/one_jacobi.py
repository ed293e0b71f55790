"""One K9 call (n = 384 random core) for an ncu capture of jacobi_cluster_kernel."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_09703_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 384
K = np.random.default_rng(n).standard_normal((n, n))
dK = torch.from_numpy(np.asfortranarray(K).ravel(order="F")).cuda()
kk = int(sys.argv[2]) if len(sys.argv) > 2 else min(128, n)
th = torch.zeros(n, dtype=torch.float64, device="cuda")
F = torch.empty(kk * n, dtype=torch.float64, device="cuda")
G = torch.empty(kk * n, dtype=torch.float64, device="cuda")
print("sweeps", P.k_jacobi_svd(dK, n, n, kk, th, F, G))
