"""Micro-timing of the Cholesky-QR passes of the core reduction (rows x 128)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_09703_b200 as P
rows, l = int(sys.argv[1]) if len(sys.argv) > 1 else 3345, int(sys.argv[2]) if len(sys.argv) > 2 else 128
X = torch.randn(rows, l, dtype=torch.float64, device="cuda")
for passes in (1, 2):
    for _ in range(3):
        P.k_cholqr(X.clone(), rows, l, passes)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    Xs = [X.clone() for _ in range(20)]
    torch.cuda.synchronize()
    e0.record()
    for Y in Xs:
        P.k_cholqr(Y, rows, l, passes)
    e1.record()
    torch.cuda.synchronize()
    print(f"rows {rows} l {l} passes {passes}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per call")
