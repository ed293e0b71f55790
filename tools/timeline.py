"""Device timeline of the hot path: one (or more) warm configs[1] steps under torch.profiler
(CUPTI activity records via kineto), summarised as GPU busy time vs step time, the largest
idle gaps and what precedes them, and per-kernel totals with concurrency.

    python tools/timeline.py [c4|c2|c3] [n_steps] > gpurun_out/timeline.txt
"""
import json
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2401_09703_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
nprof = int(sys.argv[2]) if len(sys.argv) > 2 else 2
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


dev_batches = [[(bi, b.kind, sp(b.E), sp(b.D)) for bi, b in st] for st in steps]
nwarm = 3
for i in range(nwarm):
    for bi, kind, E, D in dev_batches[i]:
        t.update(kind, E, D, opts=bench.batch_opts(P, mode, bi))
torch.cuda.synchronize()

from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for i in range(nwarm, nwarm + nprof):
        for bi, kind, E, D in dev_batches[i]:
            t.update(kind, E, D, opts=bench.batch_opts(P, mode, bi))
    torch.cuda.synchronize()

path = "gpurun_out/timeline_trace.json"
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(path)
tr = json.load(open(path))
ev = tr["traceEvents"] if isinstance(tr, dict) else tr
kern = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
rt = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("cuda_runtime", "cuda_driver")]
kern.sort(key=lambda e: e["ts"])
t0 = kern[0]["ts"]
t1 = max(e["ts"] + e["dur"] for e in kern)
# busy union
busy = 0.0
cur_s, cur_e = None, None
gaps = []
prev_name = None
for e in kern:
    s, d = e["ts"], e["ts"] + e["dur"]
    if cur_e is None:
        cur_s, cur_e = s, d
    elif s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, cur_e, prev_name, e["name"]))
        cur_s, cur_e = s, d
    else:
        cur_e = max(cur_e, d)
    if d >= cur_e:
        prev_name = e["name"]
busy += cur_e - cur_s
span = t1 - t0
print(f"{cfg}: {nprof} steps, span {span/1e3:.2f} ms ({span/1e3/nprof:.2f} ms/step), GPU busy (union) "
      f"{busy/1e3:.2f} ms = {100*busy/span:.1f}%, kernels {len(kern)}")
gsum = sum(g[0] for g in gaps)
print(f"idle gaps: {len(gaps)} totalling {gsum/1e3:.2f} ms; >10us: {sum(1 for g in gaps if g[0] > 10)} "
      f"totalling {sum(g[0] for g in gaps if g[0] > 10)/1e3:.2f} ms")


def short(nm):
    nm = nm.replace("(anonymous namespace)::", "").replace("tsvd::", "")
    return nm.split("(")[0][:60]


# what host call is running during each large gap
rt.sort(key=lambda e: e["ts"])
print("\nlargest gaps (us, after -> before, host calls overlapping the gap):")
for g in sorted(gaps, reverse=True)[:40]:
    dur, at, a, b = g
    hosts = defaultdict(float)
    for r in rt:
        if r["ts"] + r["dur"] < at or r["ts"] > at + dur:
            continue
        hosts[r["name"]] += min(r["ts"] + r["dur"], at + dur) - max(r["ts"], at)
    hs = ", ".join(f"{k}:{v:.0f}" for k, v in sorted(hosts.items(), key=lambda x: -x[1])[:3])
    print(f"{dur:8.1f}  {short(a)} -> {short(b)}   [{hs}]")
# gap classes
cls = defaultdict(lambda: [0, 0.0])
for dur, at, a, b in gaps:
    k = (short(a), short(b))
    cls[k][0] += 1
    cls[k][1] += dur
print("\ngap totals by (after, before) pair (top 25):")
for k, (c, tot) in sorted(cls.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{tot/1e3:8.3f} ms {c:5d}x  {k[0]} -> {k[1]}")
tot = defaultdict(lambda: [0, 0.0])
for e in kern:
    tot[short(e["name"])][0] += 1
    tot[short(e["name"])][1] += e["dur"]
print("\nkernel totals (device time, ms/step):")
for k, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{d/1e3/nprof:8.3f} {c/nprof:7.1f}/step {d/c:9.1f} us  {k}")
host = defaultdict(lambda: [0, 0.0])
for r in rt:
    host[r["name"]][0] += 1
    host[r["name"]][1] += r["dur"]
print("\nhost runtime calls (ms/step):")
for k, (c, d) in sorted(host.items(), key=lambda x: -x[1][1])[:15]:
    print(f"{d/1e3/nprof:8.3f} {c/nprof:7.1f}/step  {k}")
