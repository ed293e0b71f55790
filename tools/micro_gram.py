"""K3 sparse Gram micro-benchmark on the bench workloads' first batches (device events).

    python tools/micro_gram.py [c2|c3|all] [reps]

c2: the row / column update of configs[1]'s first node batch (5000 x 50k/55k, ~5 nnz per
vector); c3: configs[2]'s first 3500-user batch (3500 x 10k, ~144 ratings per user).  Prints
the mean ms per call and the upper-triangle product count.  Tuning knobs are the library's
environment variables (TSVD_GRAM_HOT, TSVD_GRAM_COLD_RATE, TSVD_GRAM_SYRK_RATE), read once
per process."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_09703_b200 as P  # noqa: E402
from synth import generators as G  # noqa: E402


def batches(which):
    out = []
    if which in ("c2", "all"):
        A = G.chung_lu(100_000, 10.0, 2.1, 2)
        c, b = 50_000, 5_000
        out.append(("c2-rows", A[c:c + b, :c].tocsr()))
        out.append(("c2-cols", A[c:c + b, :c + b].tocsr()))
    if which in ("c3", "all"):
        A = G.ratings_matrix(70_000, 10_000, 10_000_000, 3)
        out.append(("c3-rows", A[35_000:38_500].tocsr()))
    return out


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    for name, E in batches(which):
        s = E.shape[0]
        d = np.diff(E.tocsc().indptr).astype(np.float64)
        dE = P.Sparse.from_scipy(E, device="cuda")
        Gm = torch.empty((s, s), dtype=torch.float64, device="cuda")
        for _ in range(3):
            P.k_sparse_gram(dE, Gm)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            P.k_sparse_gram(dE, Gm)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        print(f"[micro_gram] {name} s={s} nnz={E.nnz} upper_products={(d * (d + 1) / 2).sum():.3g} "
              f"ms={ms:.4f} env={ {k: v for k, v in os.environ.items() if k.startswith('TSVD_GRAM')} }", flush=True)


if __name__ == "__main__":
    main()
