"""One warm update of a bench config between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists / captures (ncu times are serialised and
cold-cache; the kernels' SHARE of the update is what compares with bench.py).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        python tools/profile_one.py [c4|c2|c3|c1] [warm_batches]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2401_09703_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
nwarm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w, steps, desc, mode = bench.make_workload(cfg)
dev = torch.device("cuda:0")
m, n = w.final_dims()
t = P.TSVD(w.k, m_capacity=m, n_capacity=n, device=0)
t.reserve(8 << 30)
if hasattr(w, "init_state"):
    w.init_state(P, t)
else:
    t.init(*(torch.from_numpy(x).to(dev) for x in (w.U0, w.S0, w.V0)))


def sp(A):
    return bench._to_sparse(P, A, dev=dev)


todo = [(bi, b.kind, sp(b.E), sp(b.D)) for st in steps[:nwarm + 1] for bi, b in st]
per = len(steps[0])
for bi, kind, E, D in todo[:nwarm * per]:
    t.update(kind, E, D, opts=bench.batch_opts(P, mode, bi))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for bi, kind, E, D in todo[nwarm * per:]:
    t.update(kind, E, D, opts=bench.batch_opts(P, mode, bi))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("[profile_one]", cfg, "launches", t.stats()["launches"])
