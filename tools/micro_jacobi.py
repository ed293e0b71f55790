"""Timing of the core one-sided Jacobi (K7 <= 128, K9 cluster 128 < n <= 512, K8 otherwise /
TSVD_K9=0) through tsvd_k_jacobi_svd on random and weight-update-like cores.

    python tools/micro_jacobi.py            # prints one JSON line per case
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_09703_b200 as P  # noqa: E402


def core(kind, n, rng):
    if kind == "random":
        return rng.standard_normal((n, n))
    k = n // 3   # weight-update-like: dominant diagonal + low rank + small tail
    S = np.concatenate([np.linspace(1000, 100, k), np.zeros(n - k)])
    return np.diag(S) + rng.standard_normal((n, 8)) @ rng.standard_normal((8, n)) * 3.0


def core_svd(K, kk):
    n = K.shape[0]
    dK = torch.from_numpy(np.asfortranarray(K).ravel(order="F")).cuda()
    th = torch.zeros(kk + 1, dtype=torch.float64, device="cuda")
    F = torch.empty(kk * n, dtype=torch.float64, device="cuda")
    G = torch.empty(kk * n, dtype=torch.float64, device="cuda")
    info = P.k_core_svd(dK, n, n, kk, th, F, G)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    info = P.k_core_svd(dK, n, n, kk, th, F, G)
    e1.record()
    torch.cuda.synchronize()
    ref = np.linalg.svd(K, compute_uv=False)
    err = float(np.max(np.abs(th.cpu().numpy() - ref[:kk + 1]) / ref[:kk + 1]))
    print(json.dumps(dict(kind="core_svd_weights", n=n, kk=kk, ms=e0.elapsed_time(e1), info=info, sigma_err=err)),
          flush=True)


for n, kk in ((384, 128), (512, 256)):
    rng = np.random.default_rng(n)
    S = np.concatenate([np.linspace(1000, 100, kk), np.zeros(n - kk)])
    K = np.diag(S) + rng.standard_normal((n, 6)) @ rng.standard_normal((6, n)) \
        + rng.standard_normal((n, n)) * np.logspace(0, -3, n)[None, :] * 0.5
    core_svd(K, kk)

for kind in ("random", "weights"):
    for n in (64, 96, 128, 160, 256, 384, 512):
        rng = np.random.default_rng(n)
        K = core(kind, n, rng)
        dK = torch.from_numpy(np.asfortranarray(K).ravel(order="F")).cuda()
        kk = min(n, 128)
        th = torch.zeros(n, dtype=torch.float64, device="cuda")
        F = torch.empty(kk * n, dtype=torch.float64, device="cuda")
        G = torch.empty(kk * n, dtype=torch.float64, device="cuda")
        P.k_jacobi_svd(dK, n, n, kk, th, F, G)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sw = P.k_jacobi_svd(dK, n, n, kk, th, F, G)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ref = np.linalg.svd(K, compute_uv=False)
        err = float(np.max(np.abs(th.cpu().numpy() - ref) / np.maximum(ref, 1e-3 * ref[0])))
        print(json.dumps(dict(kind=kind, n=n, ms=ms, sweeps=sw, us_per_round=1e3 * ms / max(sw * (n - 1), 1),
                              sigma_err=err, k9=os.environ.get("TSVD_K9", "1"),
                              k9_small=os.environ.get("TSVD_K9_SMALL", "0"))), flush=True)
