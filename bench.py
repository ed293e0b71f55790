"""bench.py — throughput of the sparse-aware truncated-SVD update (arXiv 2401.09703) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Metric (BASELINE.json "metric"): tSVD update throughput in fp64, rows/s (appended
nodes per second; nnz/s alongside), plus the roofline of the dominant kernel.

Workload: BASELINE.json configs[1] — symmetric Chung-Lu power-law
graph, 100k nodes, mean degree 10, exponent 2.1, 0/1 values fp64, k = 64, SVD_64 of the
first 50k nodes, then batches of 5k nodes appended as a row update followed by a column
update (synth.graph_nodeappend).  One step = one batch (both halves).  Inputs are
synthetic and seeded; the batches sit in HBM before the timed region; L2 is flushed
(a 512 MB write) before every timed step, outside its CUDA events.

--impl reference times the CPU fp64 oracle (oracle.zha_simon, dense Householder QR +
LAPACK SVD) on a bounded sample of the same workload: the first S nodes of each batch
(row half A[c:c+S, :c], column half A[:c+S, c:c+S]), S = --ref-nodes (default 1000).

N > 1 (torchrun): the C2 path is replicas-only in this round:
every rank runs the whole stream on its own GPU; value = nodes all ranks processed ÷
the max over ranks of the timed device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# FP64 has no entry in MEASURED_PEAKS.json: bench.py measures the FP64 contraction peak
# live (cuBLAS DGEMM via torch.matmul, 8192^3, best of 5, CUDA events) on the same GPU.
# If that fails it falls back to (measured bf16 peak) x (guide nominal ratio 45/2250).
FP64_OVER_BF16 = 45.0 / 2250.0
# kernel classes of tsvd_stats.kern_* (include/tsvd.h) and the roof that bounds each
KCLASS = ("gather_spmm", "sparse_gram", "dgemm_dmma", "chol_panel", "small_chol", "core_jacobi",
          "scatter_add", "approx_sparse")
KBOUND = ("hbm", "hbm", "tensor", "tensor", "tensor", "tensor", "hbm", "hbm")  # "tensor": the FP64 roof
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def measure_dgemm_tflops(dev):
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def peaks():
    try:
        p = json.load(open(PEAKS_PATH))
        p["_src"] = "measured"
    except Exception:
        p = dict(FALLBACK)
        p["_src"] = "fallback"
    return p


# ----------------------------------------------------------------------------- workload
def make_workload(cfg: str):
    import synth
    if cfg == "c2":
        w = synth.graph_nodeappend()          # configs[1], full size
        steps = [(w.batches[2 * i], w.batches[2 * i + 1]) for i in range(len(w.batches) // 2)]
        desc = dict(workload="configs[1] graph node-append: Chung-Lu N=100000 avg_deg=10 beta=2.1, 0/1 fp64; "
                             "SVD_64 of first 50k nodes; batches of 5000 nodes = row update + column update",
                    N=100000, k=w.k, nodes_per_step=5000, mode="exact", l2="flushed before every step (512 MB write)")
        return w, steps, desc
    if cfg == "c1":
        w = synth.tiny_rowappend()
        steps = [(b,) for b in w.batches]
        desc = dict(workload="configs[0] tiny row-append 2000x1000, k=16, batches of 100 rows", k=w.k,
                    nodes_per_step=100, mode="exact", l2="flushed before every step (512 MB write)")
        return w, steps, desc
    if cfg == "c3":
        w = synth.ratings_rowappend()
        steps = [(b,) for b in w.batches]
        desc = dict(workload="configs[2] ratings row-append 70k x 10k, 10M ratings, k=64, batches of 3500 users",
                    k=w.k, nodes_per_step=3500, mode="exact", l2="flushed before every step (512 MB write)")
        return w, steps, desc
    raise SystemExit(f"unknown config {cfg}")


def step_rows(step):
    return step[0].s


def step_nnz(step):
    return sum(b.nnz for b in step)


# ----------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2401_09703_b200 as P
    dev = torch.device(f"cuda:{local_rank}")
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    w, steps, desc = make_workload(args.config)
    nst = len(steps)
    m_fin, n_fin = w.final_dims()
    stream = torch.cuda.current_stream()

    def to_dev(step):
        return [(b.kind, P.Sparse.from_scipy(b.E, device=dev)) for b in step]

    def to_host(step):
        return [(b.kind, P.Sparse.from_scipy(b.E, pin=True)) for b in step]

    dsteps = [to_dev(s) for s in steps]
    hsteps = [to_host(s) for s in steps]
    U0, S0, V0 = (torch.from_numpy(x).to(dev) for x in (w.U0, w.S0, w.V0))
    t = P.TSVD(w.k, m_capacity=m_fin, n_capacity=n_fin, device=local_rank)
    t.reserve(4 << 30)   # scratch pool sized up front (a service would keep it warm)
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=dev)
    opts = P.make_opts()
    opts_prof = P.make_opts(flags=2)   # per-kernel-class events (roofline pass)

    state = {"pos": nst}   # batch index the context is at (nst forces a re-init)

    def ensure_at(i):
        """Bring the context to 'batch i is next' (re-init + replay, untimed)."""
        if state["pos"] != i:
            t.init(U0, S0, V0)
            for j in range(i):
                for kind, E in dsteps[j]:
                    t.update(kind, E, opts=opts)
            state["pos"] = i

    def apply(i, host=False, prof=False):
        launches = 0
        kern = [[0.0, 0, 0.0, 0.0] for _ in KCLASS]   # ms, launches, flops, bytes per class
        for kind, E in (hsteps if host else dsteps)[i]:
            t.update(kind, E, opts=opts_prof if prof else opts)
            st = t.stats(wait=prof)   # counters only: no sync inside the timed region
            launches += st["launches"]
            for c in range(len(KCLASS)):
                kern[c][0] += st["kern_ms"][c]
                kern[c][1] += st["kern_launches"][c]
                kern[c][2] += st["kern_flops"][c]
                kern[c][3] += st["kern_bytes"][c]
        state["pos"] = i + 1
        return launches, kern

    order = [(args.warmup + j) % nst for j in range(args.steps)]
    # ---- warm-up: W untimed steps (the first W batches of the stream, then the stream is
    # replayed up to the timed batches)
    for j in range(args.warmup):
        ensure_at(j % nst)
        apply(j % nst)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in order]
    tot_launch, kern = 0, [[0.0, 0, 0.0, 0.0] for _ in KCLASS]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local_rank) as ck:
        for j, i in enumerate(order):
            ensure_at(i)
            flush.zero_()
            ev[j][0].record(stream)
            nl, kp = apply(i)
            ev[j][1].record(stream)
            tot_launch += nl
            kern = [[a + b for a, b in zip(x, y)] for x, y in zip(kern, kp)]
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    rows = sum(step_rows(steps[i]) for i in order)

    # ---- roofline pass: the same K steps again with per-kernel-class CUDA events (the
    # events cost host time, so the headline value above comes from the uninstrumented pass)
    kern = [[0.0, 0, 0.0, 0.0] for _ in KCLASS]
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in order]
    for j, i in enumerate(order):
        ensure_at(i)
        flush.zero_()
        ev2[j][0].record(stream)
        _, kp = apply(i, prof=True)
        ev2[j][1].record(stream)
        kern = [[a + b for a, b in zip(x, y)] for x, y in zip(kern, kp)]
    torch.cuda.synchronize()
    ms_prof = sum(a.elapsed_time(b) for a, b in ev2)
    nnz = sum(step_nnz(steps[i]) for i in order)

    # ---- end to end: host CSR in, Σ out, through the C-ABI (library stages the copies)
    h2d = 0
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in order]
    S_host = torch.empty(w.k, dtype=torch.float64).pin_memory()
    for j, i in enumerate(order):
        ensure_at(i)
        flush.zero_()
        e2e_ev[j][0].record(stream)
        apply(i, host=True)
        t.get_S(S_host)
        e2e_ev[j][1].record(stream)
        for _, E in hsteps[i]:
            h2d += E.row_ptr.numel() * 8 + E.col_idx.numel() * 4 + E.val.numel() * 8
    torch.cuda.synchronize()
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)

    top = max(range(len(KCLASS)), key=lambda c: kern[c][0])
    vals = torch.tensor([ms, e2e_ms, kern[top][0]], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, e2e_ms, top_ms = vals.tolist()
    if rank == 0:
        pk = peaks()
        try:
            fp64_peak = measure_dgemm_tflops(dev)
            fp64_src = "FP64 DGEMM measured live in bench.py (cuBLAS via torch.matmul 8192^3, best of 5)"
        except Exception as ex:  # pragma: no cover
            fp64_peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) * FP64_OVER_BF16
            fp64_src = f"{pk['_src']} bf16 sustained x 45/2250 (guide nominal ratio); dgemm probe failed: {ex}"
        bound = KBOUND[top]
        tk = kern[top]
        if bound == "hbm":
            achieved, peak, unit = tk[3] / (top_ms * 1e-3) / 1e9, pk["hbm_gbs"], "GB/s"
            psrc = f"hbm_gbs, {pk['_src']} (MEASURED_PEAKS.json)"
        else:
            achieved, peak, unit = tk[2] / (top_ms * 1e-3) / 1e12, fp64_peak, "TFLOP/s"
            psrc = fp64_src
        traffic, traffic_src = class_traffic(KCLASS[top])
        kern_tab = {KCLASS[c]: {"ms_per_step": kern[c][0] / args.steps, "launches_per_step": kern[c][1] / args.steps,
                                "tflops": (kern[c][2] / (kern[c][0] * 1e-3) / 1e12) if kern[c][0] else None,
                                "gbs": (kern[c][3] / (kern[c][0] * 1e-3) / 1e9) if kern[c][0] else None}
                    for c in range(len(KCLASS)) if kern[c][0] > 0}
        cpu = None if (world > 1 or args.no_cpu_baseline) else cpu_baseline(args, w, steps)
        out = {
            "metric": "tSVD update throughput (rows/s appended nodes; nnz/s alongside), fp64",
            "value": world * rows / (ms * 1e-3),
            "unit": "rows/s",
            "nnz_per_s": world * nnz / (ms * 1e-3),
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded Chung-Lu graph, synth.graph_nodeappend)",
            "config": dict(desc, parallelism=("replicas" if world > 1 else "single")),
            "roofline": {"kernel": KCLASS[top], "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                         "frac": achieved / peak if peak else None, "traffic": traffic, "traffic_src": traffic_src,
                         "launches": tk[1], "avg_launch_us": 1e3 * top_ms / max(tk[1], 1),
                         "share_of_step": top_ms / ms_prof if ms_prof else None,
                         "measured_in": "a second pass over the same K steps with per-kernel-class CUDA events "
                                        f"({ms_prof / args.steps:.1f} ms/step instrumented)",
                         "algorithmic_flops_per_launch": tk[2] / max(tk[1], 1),
                         "algorithmic_bytes_per_launch": tk[3] / max(tk[1], 1), "peak_src": psrc},
            "kernels": kern_tab,
            "fp64_dgemm_tflops_measured": fp64_peak,
            "e2e": {"value": world * rows / (e2e_ms * 1e-3), "unit": "rows/s",
                    "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": w.k * 8},
            "gpu_launches": tot_launch,
            "clocks": ck.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


# DRAM bytes per launch of a class's kernels, from the committed ncu --set full captures
# (profiles/r1_traffic.json, written by tools/ncu_traffic.py); the class's kernels launch
# equally often per update, so their per-launch traffic is averaged
CLASS_KERNELS = {"chol_panel": ["chol_dag_kernel", "trsm_dag_kernel"], "dgemm_dmma": ["dgemm_v2_kernel"],
                 "core_jacobi": ["jacobi_cta_kernel"], "small_chol": ["chol_inv_small_kernel"],
                 "sparse_gram": ["sparse_gram_kernel"], "gather_spmm": ["gather_spmm_kernel"],
                 "scatter_add": ["scatter_add_kernel"]}


def class_traffic(cls):
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_traffic.json")
    try:
        tab = json.load(open(path))
    except (OSError, ValueError):
        return None, None
    ks = [k for k in CLASS_KERNELS.get(cls, []) if k in tab]
    if not ks:
        return None, None
    return (sum(tab[k]["dram_bytes"] for k in ks) / len(ks),
            f"profiles/r1_traffic.json: mean over {', '.join(ks)} (ncu --set full, one capture each)")


# ----------------------------------------------------------------------------- oracle arm
def sample_step(w, steps, i, S):
    """First S nodes of batch i: rows A[c:c+S, :c], cols A[:c+S, c:c+S]."""
    import synth
    c = w.m0 + sum(st[0].s for st in steps[:i])
    out = [synth.Batch("rows", steps[i][0].E[:S])]
    if len(steps[i]) > 1:
        out.append(synth.Batch("cols", steps[i][1].E[:S, :c + S].tocsr()))
    return out


def time_oracle_steps(w, steps, idxs, S):
    """Oracle time on the sampled steps idxs.  The oracle's cost depends on m, n, k and s,
    not on how its state got there, so each sampled step starts from the init factors
    zero-padded to the batch's dimensions (still orthonormal) instead of replaying the
    stream on the CPU."""
    from oracle import zha_simon
    tot, rows, nnz = 0.0, 0, 0
    for i in idxs:
        c = w.m0 + sum(st[0].s for st in steps[:i])
        U, Sg, V = _pad_rows(w.U0, c), w.S0.copy(), _pad_rows(w.V0, w.n0 + (c - w.m0) * (len(steps[i]) - 1))
        bs = sample_step(w, steps, i, S)
        t0 = time.perf_counter()
        for b in bs:
            U, Sg, V, _ = zha_simon.apply_batch(U, Sg, V, b)
        tot += time.perf_counter() - t0
        rows += bs[0].s
        nnz += sum(b.nnz for b in bs)
    return tot, rows, nnz


def _pad_rows(X, rows):
    import numpy as np
    out = np.zeros((rows, X.shape[1]))
    out[:X.shape[0]] = X
    return out


def _threads():
    try:
        from threadpoolctl import threadpool_info
        return max(int(i.get("num_threads", 1)) for i in threadpool_info()) or os.cpu_count()
    except Exception:
        return os.cpu_count()


def cpu_baseline(args, w, steps):
    idx = [0]
    tot, rows, nnz = time_oracle_steps(w, steps, idx, args.ref_nodes)
    return {"value": rows / tot, "unit": "rows/s", "nnz_per_s": nnz / tot, "cores": _threads(), "kind": "oracle",
            "sample": f"oracle (dense Householder QR + LAPACK gesdd, fp64) on the first {args.ref_nodes} of the "
                      f"{step_rows(steps[0])} nodes of batch 0 (row half + column half); its cost grows "
                      f"superlinearly in s, so this overstates its full-batch throughput; {tot:.1f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    w, steps, desc = make_workload(args.config)
    nst = len(steps)
    for j in range(args.warmup):
        time_oracle_steps(w, steps, [j % nst], args.ref_nodes)
    idxs = [(args.warmup + j) % nst for j in range(args.steps)]
    tot, rows, nnz = time_oracle_steps(w, steps, idxs, args.ref_nodes)
    v = rows / tot
    out = {"impl": "reference", "metric": "tSVD update throughput (rows/s appended nodes; nnz/s alongside), fp64",
           "value": v, "unit": "rows/s", "nnz_per_s": nnz / tot, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": dict(desc, sample_nodes=args.ref_nodes),
           "cpu_baseline": {"value": v, "unit": "rows/s", "cores": _threads(), "kind": "oracle",
                            "sample": f"first {args.ref_nodes} nodes of each batch (row + column half)"},
           "e2e": {"value": v, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3"])
    ap.add_argument("--ref-nodes", type=int, default=1000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
