"""Micro-timing: libtsvd DMMA GEMM (k_dgemm, row-major API) vs cuBLAS DGEMM (torch) on the
shapes of the C2 core reduction."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_09703_b200 as P

def t_ms(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

shapes = [  # (name, M, N, K, tA, tB, uplo)
    ("K Y   (col-major K)", 4185, 128, 3345, 1, 0, 0),
    ("K^T Z", 3345, 128, 4185, 0, 0, 0),
    ("Y T  (n x b x b)", 3345, 128, 128, 0, 0, 0),
    ("Y^T Y (uplo)", 128, 128, 3345, 1, 0, 1),
    ("SYRK s x s x 64", 3800, 3800, 64, 1, 0, 1),
    ("square 4096", 4096, 4096, 4096, 0, 0, 0),
]
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
    print(f"{name:22s} M{M} N{N} K{K}: ours {ours*1e3:8.1f} us ({fl/ours/1e9:6.2f} TF/s)   cuBLAS {cub*1e3:8.1f} us ({2.0*M*N*K/cub/1e9:6.2f} TF/s)")
