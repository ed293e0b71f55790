"""Device timeline of streaming (s = 1) updates: node-at-a-time row + column updates of the
configs[1] graph stand-in (tools/sweep_fig12.py's setup), under torch.profiler: GPU busy vs
wall time, per-kernel and host-call totals per update.  python tools/timeline_stream.py [n]"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_09703_b200 as P  # noqa: E402
from synth.generators import chung_lu  # noqa: E402

n_upd = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dev = torch.device("cuda:0")
A = chung_lu(100_000, 10.0, 2.1, seed=2).tocsr()
n0 = 50_000
t = P.TSVD(64, m_capacity=2 * n0, n_capacity=2 * n0)
t.init_sparse(P.Sparse.from_scipy(A[:n0, :n0], device=dev), oversample=32, power_iters=2, seed=1)
t.reserve(1 << 30)
bs = [(P.Sparse.from_scipy(A[c:c + 1, :c], device=dev), P.Sparse.from_scipy(A[c:c + 1, :c + 1], device=dev))
      for c in range(n0, n0 + n_upd + 3)]
for Er, EcT in bs[:3]:
    t.update_rows(Er)
    t.update_cols(EcT)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for Er, EcT in bs[3:]:
        t.update_rows(Er)
        t.update_cols(EcT)
    torch.cuda.synchronize()
path = "gpurun_out/timeline_stream.json"
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
kern = sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")],
              key=lambda e: e["ts"])
rt = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("cuda_runtime", "cuda_driver")]
t0, t1 = kern[0]["ts"], max(e["ts"] + e["dur"] for e in kern)
busy, ce = 0.0, None
cs = None
for e in kern:
    s, d = e["ts"], e["ts"] + e["dur"]
    if ce is None or s > ce:
        if ce is not None:
            busy += ce - cs
        cs, ce = s, d
    else:
        ce = max(ce, d)
busy += ce - cs
nu = 2 * n_upd
print(f"{nu} updates (s = 1): span {(t1 - t0) / 1e3:.2f} ms = {(t1 - t0) / nu:.1f} us/update, GPU busy {busy / nu:.1f} us/update "
      f"({100 * busy / (t1 - t0):.0f} %), kernels {len(kern) / nu:.1f}/update")
kt = collections.defaultdict(lambda: [0.0, 0])
for e in kern:
    k = e["name"].replace("(anonymous namespace)::", "").replace("void ", "").replace("tsvd::", "").split("(")[0][:60]
    kt[k][0] += e["dur"]
    kt[k][1] += 1
print("\nkernel totals (us/update, launches/update):")
for k, (d, c) in sorted(kt.items(), key=lambda x: -x[1][0])[:25]:
    print(f"{d / nu:8.1f} {c / nu:6.1f}  {k}")
ht = collections.defaultdict(lambda: [0.0, 0])
for e in rt:
    ht[e["name"]][0] += e["dur"]
    ht[e["name"]][1] += 1
print("\nhost runtime calls (us/update, calls/update):")
for k, (d, c) in sorted(ht.items(), key=lambda x: -x[1][0])[:12]:
    print(f"{d / nu:8.1f} {c / nu:6.1f}  {k}")
