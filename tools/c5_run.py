"""configs[4] (C5) at full size on one GPU: GPU generation, the GPU initial SVD (F1,
tsvd_init_sparse), then a few appended-row batches with per-batch timing and statistics, and
the full-size properties the oracle cannot check one by one (orthonormality of U and V on the
device, Σ descending).  Prints JSON lines.

    python tools/c5_run.py [n_batches]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_09703_b200 as P  # noqa: E402
from synth.scaleout import scaleout_rowappend  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 3
gb = lambda: torch.cuda.memory_allocated() / 2**30  # noqa: E731
t0 = time.time()
so = scaleout_rowappend(device="cuda")
torch.cuda.synchronize()
print(json.dumps(dict(step="generate", s=time.time() - t0, nnz=so.meta["nnz"], init_nnz=so.init.nnz,
                      batch_nnz=[b.nnz for b in so.batches[:nb]], torch_gb=gb())), flush=True)
free, total = torch.cuda.mem_get_info()
t = P.TSVD(so.k, m_capacity=so.m, n_capacity=so.n)
c = so.init
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t.init_sparse(P.Sparse(c.rows, c.cols, c.row_ptr, c.col_idx, c.val), oversample=16, power_iters=2, seed=5)
e1.record()
torch.cuda.synchronize()
S0 = t.get_S()
print(json.dumps(dict(step="init_sparse", ms=e0.elapsed_time(e1), free_gb_before=free / 2**30,
                      sigma_head=S0[:4].tolist(), sigma_tail=S0[-3:].tolist())), flush=True)
del so.init, c
torch.cuda.empty_cache()
t.reserve(8 << 30)
for bi, b in enumerate(so.batches[:nb]):
    E = P.Sparse(b.rows, b.cols, b.row_ptr, b.col_idx, b.val)
    o = P.make_opts(mode=P.RPI, l=256, t=3, seed=1000 + bi)
    torch.cuda.synchronize()
    e0.record()
    t.update_rows(E, o)
    e1.record()
    torch.cuda.synchronize()
    st = t.stats()
    print(json.dumps(dict(step="batch", batch=bi, s=b.rows, nnz=b.nnz, ms=e0.elapsed_time(e1),
                          touched=st["touched"], core=[st["core_rows"], st["core_cols"], st["core_path"]],
                          sweeps=st["jacobi_sweeps"], cond=st["cond"], reset=st["reset"],
                          theta_next=st["theta_next"])), flush=True)
# full-size properties on the device (U: 18M + appended rows x 256)
m, n, k = t.dims()
U = torch.empty((m, k), dtype=torch.float64, device="cuda")
t.get_U(U)
eu = (U.T @ U - torch.eye(k, dtype=torch.float64, device="cuda")).abs().max().item()
del U
V = torch.empty((n, k), dtype=torch.float64, device="cuda")
t.get_V(V)
ev = (V.T @ V - torch.eye(k, dtype=torch.float64, device="cuda")).abs().max().item()
S = t.get_S()
print(json.dumps(dict(step="properties", m=m, n=n, orth_U=eu, orth_V=ev, sigma_descending=bool((S[:-1] >= S[1:]).all()),
                      sigma_head=S[:4].tolist(), peak_gb=torch.cuda.max_memory_allocated() / 2**30)), flush=True)
