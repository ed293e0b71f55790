"""Probe: per-update stats of the first batches of a config (Jacobi convergence trace with
TSVD_TRACE=1).  python tools/probe_c2.py [c2|c3] [n_steps]"""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2401_09703_b200 as P
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w, steps, desc = bench.make_workload(cfg)
dev = torch.device("cuda:0")
m, n = w.final_dims()
t = P.TSVD(w.k, m, n)
t.init(*(torch.from_numpy(x).to(dev) for x in (w.U0, w.S0, w.V0)))
for i in range(nsteps):
    for b in steps[i]:
        E = P.Sparse.from_scipy(b.E, device=dev)
        t0 = time.time()
        t.update(b.kind, E)
        st = t.stats()
        keys = ["s", "nnz", "rank", "touched", "cond", "reset", "jacobi_sweeps", "core_rows", "core_cols",
                "ms_pre", "ms_svd", "ms_post", "launches", "top_ms", "top_launches"]
        print(json.dumps({"step": i, "kind": b.kind, "wall_s": round(time.time() - t0, 3),
                          **{k: st[k] for k in keys}}), flush=True)
