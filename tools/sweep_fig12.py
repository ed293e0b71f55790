"""F3: the paper's k and φ sweeps on an adjacency matrix (Fig 1 "k values of
16,32,64,128,256", Fig 2 "φ values of 10^1 .. 10^4"; protocol P:486-488: a
truncated SVD of the first half of the nodes, then φ batch updates each adding n/φ rows and
columns; streaming = one node per update, the limit of Table 3's "streaming update" P:561).
The graph is the synthetic stand-in of configs[1] (Chung-Lu, N = 100k, mean degree 10, β = 2.1;
the paper's Slashdot / Flickr / Epinions are absent); the initial SVD_k of A[:N/2, :N/2] is the
GPU randomized SVD (tsvd_init_sparse).  A node batch = a row update A[c:c+b, :c] then a column
update A[:c+b, c:c+b] through the C-ABI (inputs already on the device), device-timed with CUDA
events after one untimed warm-up batch; at most --max-batches batches are timed per point and
the total for all N/2 nodes is extrapolated from their mean (marked `est`).  Accuracy: the
relative Frobenius residual ||A_c - U Σ V^T||_F / ||A_c||_F on the matrix seen so far
(tsvd_residual_fro), beside the same for the initial factors.  Methods: exact (Alg 3 with
SV-LCOV), GKL and RPI (l = 10, t = 3, the paper's defaults).  JSON lines.

    python tools/sweep_fig12.py --sweep k   [--ks 16,32,64,128,256] [--phi 10]
    python tools/sweep_fig12.py --sweep phi [--phis 10,100,1000,10000,stream] [--k 64]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_09703_b200 as P  # noqa: E402
from synth.generators import chung_lu  # noqa: E402


def run_point(A, n0, k, batch, mode, max_batches, dev):
    nb_total = n0 // batch
    t = P.TSVD(k, m_capacity=2 * n0, n_capacity=2 * n0)
    t.init_sparse(P.Sparse.from_scipy(A[:n0, :n0], device=dev), oversample=32, power_iters=2, seed=1)
    t.reserve(2 << 30)
    r0 = t.residual_fro(P.Sparse.from_scipy(A[:n0, :n0], device=dev))
    opts = {"exact": P.make_opts(), "gkl": P.make_opts(mode=P.GKL, l=10, seed=3),
            "rpi": P.make_opts(mode=P.RPI, l=10, t=3, seed=3)}[mode]
    nb = min(nb_total, max_batches + 1)
    dev_b = []
    for b in range(nb):
        c = n0 + b * batch
        dev_b.append((P.Sparse.from_scipy(A[c:c + batch, :c], device=dev),
                      P.Sparse.from_scipy(A[c:c + batch, :c + batch], device=dev)))
    times = []
    for b, (Er, EcT) in enumerate(dev_b):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        t.update_rows(Er, opts)
        t.update_cols(EcT, opts)
        e1.record()
        torch.cuda.synchronize()
        if b:
            times.append(e0.elapsed_time(e1))
    c = n0 + nb * batch
    r1 = t.residual_fro(P.Sparse.from_scipy(A[:c, :c], device=dev))
    st = t.stats()
    ms = sum(times) / max(len(times), 1)
    rec = dict(k=k, phi=nb_total, nodes_per_batch=batch, mode=mode, timed_batches=len(times),
               ms_per_batch=ms, nodes_per_s=batch / (ms * 1e-3) if ms else None,
               total_s=nb_total * ms * 1e-3, total_is_estimate=len(times) < nb_total,
               resid_rel_init=r0[0] / max(r0[2], 1e-300) ** 0.5, resid_rel=r1[0] / max(r1[2], 1e-300) ** 0.5,
               nodes_seen=c, core=[st["core_rows"], st["core_cols"], st["core_path"]],
               resets=st["total_resets"])
    t.close()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep", choices=("k", "phi"), default="k")
    ap.add_argument("--ks", default="16,32,64,128,256")
    ap.add_argument("--phis", default="10,100,1000,10000,stream")
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--phi", type=int, default=10)
    ap.add_argument("--N", type=int, default=100_000)
    ap.add_argument("--modes", default="exact,gkl,rpi")
    ap.add_argument("--max-batches", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    A = chung_lu(args.N, 10.0, 2.1, seed=2).tocsr()
    n0 = args.N // 2
    if args.sweep == "k":
        pts = [(int(k), n0 // args.phi) for k in args.ks.split(",")]
    else:
        pts = [(args.k, 1 if p == "stream" else n0 // int(p)) for p in args.phis.split(",")]
    for k, batch in pts:
        for mode in args.modes.split(","):
            rec = run_point(A, n0, k, batch, mode, args.max_batches, dev)
            rec["sweep"] = args.sweep
            rec["graph"] = f"Chung-Lu N={args.N} mean degree 10 beta 2.1 (configs[1] stand-in)"
            print(json.dumps(rec), flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
