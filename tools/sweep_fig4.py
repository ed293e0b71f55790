"""F3: the paper's synthetic sparsity sweep (Fig 4):
100k x 100k random sparse matrices with 1e6 .. 1e9 nonzeros, a truncated SVD of the first 50 %
of the columns (here on the GPU, tsvd_init_sparse), then the other 50 % appended as column
batches of s columns; per (nnz, s, method) the device time per batch (CUDA events, first batch
untimed) and the throughput.  Methods: exact (Alg 3 with SV-LCOV), GKL and RPI (l = 10, t = 3 —
the paper's defaults).  Writes JSON lines (and a table with --table).

    python tools/sweep_fig4.py [--nnz 1e6,1e7,1e8] [--s 1000,10000] [--k 64] [--batches 3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_09703_b200 as P  # noqa: E402
from synth.scaleout import uniform_sparse_colappend  # noqa: E402


def sub_rows(b, r0, r1):
    p0, p1 = int(b.row_ptr[r0]), int(b.row_ptr[r1])
    return P.Sparse(r1 - r0, b.cols, (b.row_ptr[r0:r1 + 1] - p0).contiguous(), b.col_idx[p0:p1], b.val[p0:p1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nnz", default="1e6,1e7,1e8")
    ap.add_argument("--s", default="1000,10000")
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--batches", type=int, default=3)
    ap.add_argument("--modes", default="exact,gkl,rpi")
    args = ap.parse_args()
    n = 100_000
    for nnz in [int(float(x)) for x in args.nnz.split(",")]:
        init, app = uniform_sparse_colappend(n, n, nnz, seed=6)
        for s in [int(x) for x in args.s.split(",")]:
            for mode in args.modes.split(","):
                t = P.TSVD(args.k, m_capacity=n, n_capacity=n)
                t0 = time.time()
                t.init_sparse(P.Sparse(init.rows, init.cols, init.row_ptr, init.col_idx, init.val), oversample=32,
                              power_iters=1, seed=1)
                torch.cuda.synchronize()
                t_init = time.time() - t0
                t.reserve(4 << 30)
                opts = {"exact": P.make_opts(), "gkl": P.make_opts(mode=P.GKL, l=10, seed=3),
                        "rpi": P.make_opts(mode=P.RPI, l=10, t=3, seed=3)}[mode]
                times, nz = [], 0
                for bi in range(args.batches + 1):
                    E = sub_rows(app, bi * s, (bi + 1) * s)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    e0.record()
                    t.update_cols(E, opts)
                    e1.record()
                    torch.cuda.synchronize()
                    if bi:
                        times.append(e0.elapsed_time(e1))
                        nz += E.nnz
                ms = sum(times) / len(times)
                st = t.stats()
                print(json.dumps(dict(nnz=nnz, density=nnz / n / n, s=s, phi=(n // 2) // s, mode=mode, k=args.k,
                                      ms_per_batch=ms, cols_per_s=s / (ms * 1e-3), nnz_per_s=nz / (sum(times) * 1e-3),
                                      est_total_s=(n // 2) // s * ms * 1e-3, init_s=t_init,
                                      core=[st["core_rows"], st["core_cols"], st["core_path"]],
                                      rank=st["rank"], resets=st["total_resets"])), flush=True)
                t.close()
                del t
        del init, app
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
