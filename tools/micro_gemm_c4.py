"""Micro-timing of the configs[3] (C4) split-K GEMM shapes: libtsvd DMMA vs cuBLAS (torch).
Environment knobs of gemm.cu (TSVD_SPLIT_SLOTS, TSVD_SPLIT_BIG) select the split for tuning."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_09703_b200 as P  # noqa: E402


def t_ms(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


s = 110_000
shapes = [  # (name, M, N, K, tA, tB, uplo)
    ("gram l=256 (uplo)", 256, 256, s, 1, 0, 1),
    ("C' = C0 P (k x l x s)", 128, 256, s, 1, 0, 0),
    ("core BD BE^T 384^2", 384, 384, s, 0, 1, 0),
    ("apply X T (s x l x l)", s, 256, 256, 0, 0, 0),
    ("P -= C0^T C' (s x l x k)", s, 256, 128, 0, 0, 0),
    ("square 4096", 4096, 4096, 4096, 0, 0, 0),
]
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("TSVD_")}}
for name, M, N, K, tA, tB, uplo in shapes:
    A = torch.randn(K, M, dtype=torch.float64, device="cuda") if tA else torch.randn(M, K, dtype=torch.float64, device="cuda")
    B = torch.randn(N, K, dtype=torch.float64, device="cuda") if tB else torch.randn(K, N, dtype=torch.float64, device="cuda")
    Cm = torch.zeros(M, N, dtype=torch.float64, device="cuda")
    lda, ldb = A.shape[1], B.shape[1]
    ours = t_ms(lambda: P.k_dgemm(tA, tB, M, N, K, 1.0, A, lda, B, ldb, 0.0, Cm, N, uplo))
    Ao = A.t() if tA else A
    Bo = B.t() if tB else B
    cub = t_ms(lambda: torch.matmul(Ao, Bo))
    fl = 2.0 * M * N * K / (2 if uplo else 1)
    out[name] = dict(ours_us=ours * 1e3, ours_tf=fl / ours / 1e9, cublas_us=cub * 1e3, cublas_tf=2.0 * M * N * K / cub / 1e9)
print(json.dumps(out))
