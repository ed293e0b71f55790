"""bench.py — throughput of the sparse-aware truncated-SVD update (arXiv 2401.09703) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4|c1|c2|c3]

Metric (BASELINE.json "metric"): tSVD update throughput in fp64 — nnz/s and rows/s — plus
the roofline of the dominant kernel class.

Default workload: BASELINE.json configs[3] (C4), the largest configuration
that runs on one GPU: weight updates A + D E^T on a symmetric Chung-Lu graph, 1M nodes,
mean degree 20, exponent 2.1, k = 128; per batch 50k edge deletions + 50k insertions (ΔA,
2e5 nonzeros of ±1), D = one-hot columns of the s ≈ 1.1e5 touched rows, E = ΔA[R,:]^T;
RPI (Alg 8) with l = 256, t = 3, the start blocks drawn by the counter-based generator K12
(seed 1000 + batch).  One step = one batch.  value = nnz(ΔA) per second; rows/s (touched
rows s per second) alongside.  Inputs are synthetic and seeded and sit in HBM before the
timed region; L2 (126 MB) is flushed (a 512 MB write) before every timed step, outside its
CUDA events.

--config c2 (configs[1], graph node-append: one step = 5000 appended nodes as a row update
followed by a column update, value = rows/s), c3 (configs[2]) and c1 (configs[0]) are kept
for the round-1 comparisons.

--impl reference times the CPU fp64 oracle as it stands: for C4 one FULL batch per step
(oracle.variants.update_weights: dense RPI, Alg 7, with the same start blocks; about 30 s on
16 host cores); for C2 the first S nodes of each batch (--ref-nodes).

N > 1 (torchrun): C4 runs the row-sharded path: U' and V' rows dealt over the
N ranks, the same batches on every rank, partial products summed by NCCL all-reduce inside
the library; value = the job's nnz per second (total work fixed: "scaling": "strong").
C1-C3 run replicas (one stream per rank, "weak").
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
L2FLUSH = "flushed before every step (512 MB write)"


def make_workload(cfg: str):
    """(workload, steps, desc, mode): steps = list of tuples of (global batch index, Batch)."""
    import synth
    if cfg == "c4":
        w = synth.weights_rpi()               # configs[3], full size
        steps = [((i, b),) for i, b in enumerate(w.batches)]
        desc = dict(workload="configs[3] weight update A+DE^T, RPI: Chung-Lu N=1000000 avg_deg=20 beta=2.1, fp64; "
                             "SVD_128 of the initial graph; batches of 50k edge deletions + 50k insertions "
                             "(nnz(dA)=2e5, D one-hot over the ~1.1e5 touched rows); RPI l=256 t=3 (K12 start "
                             "blocks, seed 1000+batch)", N=1_000_000, k=w.k, l=256, t=3, mode="rpi",
                    nnz_counted="nnz(dA) = nnz(E_m) per batch", rows_counted="touched rows s per batch", l2=L2FLUSH)
        return w, steps, desc, "rpi"
    if cfg == "c5":
        w = C5Workload()                      # configs[4], full size, generated on the GPU
        steps = [((i, b),) for i, b in enumerate(w.batches)]
        desc = dict(workload="configs[4] scale-out row-append: 20M x 2M, ~0.97B nnz, power-law row degrees "
                             "(exponent 2, [5, 2e5]), column popularity Zipf(0.8), U(0,1) fp64; k=256; init = GPU "
                             "randomized SVD (tsvd_init_sparse, p=272, 2 power steps) of the first 18M rows; batches "
                             "of 100k appended rows; RPI l=256 t=3 (K12 start blocks, seed 1000+batch)",
                    m=w.m, n=w.n, k=w.k, l=256, t=3, mode="rpi", nnz_counted="nnz of the appended rows",
                    rows_counted="appended rows", l2=L2FLUSH)
        return w, steps, desc, "rpi_rows"
    if cfg == "c2":
        w = synth.graph_nodeappend()          # configs[1], full size
        steps = [((2 * i, w.batches[2 * i]), (2 * i + 1, w.batches[2 * i + 1])) for i in range(len(w.batches) // 2)]
        desc = dict(workload="configs[1] graph node-append: Chung-Lu N=100000 avg_deg=10 beta=2.1, 0/1 fp64; "
                             "SVD_64 of first 50k nodes; batches of 5000 nodes = row update + column update",
                    N=100000, k=w.k, nodes_per_step=5000, mode="exact", l2=L2FLUSH)
        return w, steps, desc, "exact"
    if cfg == "c1":
        w = synth.tiny_rowappend()
        steps = [((i, b),) for i, b in enumerate(w.batches)]
        desc = dict(workload="configs[0] tiny row-append 2000x1000, k=16, batches of 100 rows", k=w.k,
                    nodes_per_step=100, mode="exact", l2=L2FLUSH)
        return w, steps, desc, "exact"
    if cfg == "c3":
        w = synth.ratings_rowappend()
        steps = [((i, b),) for i, b in enumerate(w.batches)]
        desc = dict(workload="configs[2] ratings row-append 70k x 10k, 10M ratings, k=64, batches of 3500 users",
                    k=w.k, nodes_per_step=3500, mode="exact", l2=L2FLUSH)
        return w, steps, desc, "exact"
    raise SystemExit(f"unknown config {cfg}")


class C5Workload:
    """configs[4] generated on the GPU (synth.scaleout); the initial SVD is computed on the GPU
    by the library (tsvd_init_sparse, F1) — there are no host init factors."""

    def __init__(self):
        from synth.scaleout import scaleout_rowappend
        self.so = scaleout_rowappend(device="cuda")
        self.k, self.m, self.n = self.so.k, self.so.m, self.so.n
        self.name = "C5-scaleout-rowappend (GPU-generated)"
        self.batches = [_DevBatch(b) for b in self.so.batches]

    def final_dims(self):
        return self.m, self.n

    def init_state(self, P, t):
        c = self.so.init
        t.init_sparse(P.Sparse(c.rows, c.cols, c.row_ptr, c.col_idx, c.val), oversample=16, power_iters=2, seed=5)


class _DevBatch:
    kind = "rows"
    D = None

    def __init__(self, b):
        self.dev = b
        self.s = b.rows

    @property
    def nnz(self):
        return self.dev.nnz

    @property
    def E(self):
        return self  # marker: converted by _to_sparse


def _to_sparse(P, A, dev=None, pin=False):
    """scipy CSR or a GPU-generated block -> the binding's Sparse (device or pinned host)."""
    if A is None:
        return None
    if isinstance(A, _DevBatch):
        b = A.dev
        if pin:
            return P.Sparse(b.rows, b.cols, b.row_ptr.cpu().pin_memory(), b.col_idx.cpu().pin_memory(),
                            b.val.cpu().pin_memory())
        return P.Sparse(b.rows, b.cols, b.row_ptr, b.col_idx, b.val)
    return P.Sparse.from_scipy(A, device=dev, pin=pin)


def batch_opts(P, mode, bi, flags=0):
    if mode in ("rpi", "rpi_rows"):
        return P.make_opts(mode=P.RPI, l=256, t=3, seed=1000 + bi, flags=flags)
    return P.make_opts(flags=flags)


def step_rows(step):
    return step[0][1].s


def step_nnz(step, mode):
    # weight updates: nnz(dA) = nnz(E_m) (D is the one-hot factor of the reading)
    return sum((b.E.nnz if mode == "rpi" else b.nnz) for _, b in step)


def unit_of(mode):
    return "nnz/s" if mode == "rpi" else "rows/s"


def headline(mode, nnz, rows):
    return nnz if mode == "rpi" else rows


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
    w, steps, desc, mode = make_workload(args.config)
    sharded = world > 1 and mode in ("rpi", "rpi_rows")
    nst = len(steps)
    m_fin, n_fin = w.final_dims()
    stream = torch.cuda.current_stream()

    dsteps = [[(bi, b.kind, _to_sparse(P, b.E, dev=dev), _to_sparse(P, b.D, dev=dev)) for bi, b in st] for st in steps]
    hsteps = [[(bi, b.kind, _to_sparse(P, b.E, pin=True), _to_sparse(P, b.D, pin=True)) for bi, b in st]
              for st in steps]
    if hasattr(w, "init_state"):
        init_fn = lambda: w.init_state(P, t)   # noqa: E731  (GPU-computed initial SVD, F1)
    else:
        U0, S0, V0 = (torch.from_numpy(x).to(dev) for x in (w.U0, w.S0, w.V0))
        init_fn = lambda: t.init(U0, S0, V0)   # noqa: E731
    shard = None
    if sharded:   # row-sharded U', V'; the NCCL id comes from rank 0
        obj = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        shard = dict(world=world, rank=rank, nccl_id=obj[0])
    t = P.TSVD(w.k, m_capacity=m_fin, n_capacity=n_fin, device=local_rank, shard=shard)
    t.reserve((8 if mode in ("rpi", "rpi_rows") else 4) << 30)   # scratch pool sized up front (a service keeps it warm)
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=dev)
    opts = {bi: batch_opts(P, mode, bi) for st in steps for bi, _ in st}
    opts_prof = {bi: batch_opts(P, mode, bi, flags=2) for st in steps for bi, _ in st}   # per-class events

    state = {"pos": nst}   # batch index the context is at (nst forces a re-init)

    def ensure_at(i):
        """Bring the context to 'step i is next' (re-init + replay, untimed)."""
        if state["pos"] != i:
            init_fn()
            for j in range(i):
                for bi, kind, E, D in dsteps[j]:
                    t.update(kind, E, D, opts=opts[bi])
            state["pos"] = i

    def apply(i, host=False, prof=False):
        launches = 0
        kern = [[0.0, 0, 0.0, 0.0] for _ in KCLASS]   # ms, launches, flops, bytes per class
        for bi, kind, E, D in (hsteps if host else dsteps)[i]:
            t.update(kind, E, D, opts=(opts_prof if prof else opts)[bi])
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
    # ---- warm-up: W untimed steps (the first W batches of the stream; the stream is then
    # replayed up to the timed batches)
    for j in range(args.warmup):
        ensure_at(j % nst)
        apply(j % nst)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in order]
    tot_launch = 0
    for i in order[:1]:
        ensure_at(i)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local_rank) as ck:
        for j, i in enumerate(order):
            ensure_at(i)
            flush.zero_()
            ev[j][0].record(stream)
            nl, _ = apply(i)
            ev[j][1].record(stream)
            tot_launch += nl
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    rows = sum(step_rows(steps[i]) for i in order)
    nnz = sum(step_nnz(steps[i], mode) for i in order)

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

    # ---- end to end: host CSR in (pinned; the library stages the copies), Σ out
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
        for _, _, E, D in hsteps[i]:
            for X in (E, D):
                if X is not None:
                    h2d += X.row_ptr.numel() * 8 + X.col_idx.numel() * 4 + X.val.numel() * 8
    torch.cuda.synchronize()
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)

    top = max(range(len(KCLASS)), key=lambda c: kern[c][0])
    vals = torch.tensor([ms, e2e_ms, kern[top][0]], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, e2e_ms, top_ms = vals.tolist()
    # sharded: every rank processes the same batches jointly (work counted once);
    # replicas: every rank processes its own copy of the stream
    mult = 1 if sharded else world
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
        traffic, traffic_launches, traffic_src = class_traffic(args.config, KCLASS[top])
        kern_tab = {KCLASS[c]: {"ms_per_step": kern[c][0] / args.steps, "launches_per_step": kern[c][1] / args.steps,
                                "tflops": (kern[c][2] / (kern[c][0] * 1e-3) / 1e12) if kern[c][0] else None,
                                "gbs": (kern[c][3] / (kern[c][0] * 1e-3) / 1e9) if kern[c][0] else None}
                    for c in range(len(KCLASS)) if kern[c][0] > 0}
        cpu = None if (world > 1 or args.no_cpu_baseline) else cpu_baseline(args, w, steps, mode)
        u = unit_of(mode)
        val = mult * (nnz if mode == "rpi" else rows) / (ms * 1e-3)
        out = {
            "metric": "tSVD update throughput (nnz/s, rows/s) fp64",
            "value": val,
            "unit": u,
            "rows_per_s": mult * rows / (ms * 1e-3),
            "nnz_per_s": mult * nnz / (ms * 1e-3),
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if sharded else "weak", "vs_baseline": None,
            "dtype": "f64", "data": f"synthetic (seeded, synth: {w.name})",
            "config": dict(desc, parallelism=(f"row-sharded x{world} (NCCL)" if sharded else
                                              ("replicas" if world > 1 else "single"))),
            "roofline": {"kernel": KCLASS[top], "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "traffic_vs_algorithmic": (traffic / (tk[3] / max(tk[1], 1))) if traffic and tk[3] else None,
                         "traffic_src": traffic_src,
                         "launches": tk[1], "avg_launch_us": 1e3 * top_ms / max(tk[1], 1),
                         "share_of_step": top_ms / ms_prof if ms_prof else None,
                         "measured_in": "a second pass over the same K steps with per-kernel-class CUDA events "
                                        f"({ms_prof / args.steps:.1f} ms/step instrumented)",
                         "algorithmic_flops_per_launch": tk[2] / max(tk[1], 1),
                         "algorithmic_bytes_per_launch": tk[3] / max(tk[1], 1), "peak_src": psrc},
            "kernels": kern_tab,
            "fp64_dgemm_tflops_measured": fp64_peak,
            "e2e": {"value": mult * (nnz if mode == "rpi" else rows) / (e2e_ms * 1e-3), "unit": u,
                    "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": w.k * 8},
            "gpu_launches": tot_launch,
            "clocks": ck.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


# DRAM bytes per launch of the class's ncu-captured kernel (profiles/r2_traffic_<cfg>.json, written
# by tools/ncu_traffic.py from one `ncu --set full` capture): dram__bytes_read.sum +
# dram__bytes_write.sum of that launch beside the algorithmic bytes of the SAME launch (the
# library's launch log, TSVD_LAUNCH_LOG), so that the two compare like with like
def class_traffic(cfg, cls):
    path = os.path.join(ROOT, "profiles", f"r2_traffic_{cfg}.json")
    try:
        tab = json.load(open(path))
    except (OSError, ValueError):
        return None, None, None
    ent = tab.get(cls)
    if not ent:
        return None, None, None
    return ent.get("dram_bytes"), ent.get("launches"), f"profiles/r2_traffic_{cfg}.json: {ent.get('what', '')}"


# ----------------------------------------------------------------------------- oracle arm
def sample_step(w, steps, i, S):
    """C2: first S nodes of batch i (rows A[c:c+S, :c], cols A[:c+S, c:c+S])."""
    import synth
    c = w.m0 + sum(st[0][1].s for st in steps[:i])
    out = [synth.Batch("rows", steps[i][0][1].E[:S])]
    if len(steps[i]) > 1:
        out.append(synth.Batch("cols", steps[i][1][1].E[:S, :c + S].tocsr()))
    return out


_C5_SAMPLE = None


def c5_oracle_sample(nb):
    """The oracle cannot hold configs[4] (dense U' alone is 41 GB and one batch's dense products
    take minutes): it is timed on the same recipe at 1/100 of the rows and columns (m = 200k,
    n = 20k, k = 256, batches of 1000 rows, RPI l = 256, t = 3), host-generated, host init."""
    global _C5_SAMPLE
    import synth
    from synth.scaleout import scaleout_rowappend
    if _C5_SAMPLE is None:
        so = scaleout_rowappend(m=200_000, n=20_000, k=256, batch=1_000, n_batches=8, deg_max=20_000, device="cpu",
                                chunk_rows=1 << 16)
        U0, S0, V0 = synth.init_truncated_svd(so.init.to_scipy(), so.k, seed=5, method="randomized", power_iters=2)
        _C5_SAMPLE = (so, U0, S0, V0)
    so, U0, S0, V0 = _C5_SAMPLE
    from oracle import variants
    tot, rows, nnz = 0.0, 0, 0
    for bi in range(nb):
        b = so.batches[bi % len(so.batches)]
        E = b.to_scipy()
        sk = synth.counter_gaussian(1000 + bi, 1, b.rows, 256)
        t0 = time.perf_counter()
        variants.add_rows(U0, S0, V0, E, "rpi", sk, l=256, t=3)
        tot += time.perf_counter() - t0
        rows += b.rows
        nnz += b.nnz
    return tot, rows, nnz


def time_oracle_steps(w, steps, idxs, S, mode):
    """Oracle time on the steps idxs.  The oracle's cost depends on m, n, k and s, not on how
    its state got there, so each step starts from the init factors (zero-padded to the batch's
    dimensions for appends, still orthonormal) instead of replaying the stream on the CPU.
    RPI (C4): the full batch, start blocks = the numpy counter-based generator (seed 1000+b)."""
    import synth
    from oracle import variants, zha_simon
    if mode == "rpi_rows":
        return c5_oracle_sample(len(idxs))
    tot, rows, nnz = 0.0, 0, 0
    for i in idxs:
        if mode == "rpi":
            (bi, b), = steps[i]
            skD = synth.counter_gaussian(1000 + bi, 0, b.s, 256)
            skE = synth.counter_gaussian(1000 + bi, 1, b.s, 256)
            t0 = time.perf_counter()
            variants.update_weights(w.U0, w.S0, w.V0, b.D, b.E, "rpi", skD, skE, l=256, t=3)
            tot += time.perf_counter() - t0
            rows += b.s
            nnz += b.E.nnz
            continue
        c = w.m0 + sum(st[0][1].s for st in steps[:i])
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
        n = max(int(i.get("num_threads", 1)) for i in threadpool_info())
    except Exception:
        n = 0
    try:
        import torch
        n = max(n, torch.get_num_threads())
    except Exception:
        pass
    return n or os.cpu_count()


def _sample_desc(args, steps, mode, n):
    if mode == "rpi_rows":
        return (f"oracle (dense RPI Alg 7 + D.3 core, fp64) on {n} batch(es) of the configs[4] recipe at 1/100 "
                "scale (m=200k, n=20k, k=256, 1000-row batches, l=256, t=3): the full-size state does not fit a "
                "dense host oracle")
    if mode == "rpi":
        return (f"oracle (dense RPI Alg 7 + D.3 core, torch-CPU LAPACK QR / scipy gesdd, fp64) on {n} FULL "
                f"configs[3] batch(es) from the init factors (same start blocks as the GPU)")
    return (f"oracle (dense Householder QR + LAPACK gesdd, fp64) on the first {args.ref_nodes} of the "
            f"{step_rows(steps[0])} nodes of {n} batch(es) (row half + column half); its cost grows "
            f"superlinearly in s, so this overstates its full-batch throughput")


def cpu_baseline(args, w, steps, mode):
    idx = [0]
    tot, rows, nnz = time_oracle_steps(w, steps, idx, args.ref_nodes, mode)
    v = (nnz if mode == "rpi" else rows) / tot
    return {"value": v, "unit": unit_of(mode), "rows_per_s": rows / tot, "nnz_per_s": nnz / tot,
            "cores": _threads(), "kind": "oracle", "seconds": tot, "sample": _sample_desc(args, steps, mode, 1)}


def run_reference(args, rank, world):
    if rank != 0:
        return
    w, steps, desc, mode = make_workload(args.config)
    nst = len(steps)
    # one untimed step warms the host BLAS thread pools and page cache; a CPU program has
    # nothing else to warm, and each full C4 batch costs ~25 s of oracle work, so the remaining
    # warm-up steps are not executed (the run stays within a few minutes at --steps 10)
    nwarm = min(args.warmup, 1)
    for j in range(nwarm):
        time_oracle_steps(w, steps, [j % nst], args.ref_nodes, mode)
    idxs = [(args.warmup + j) % nst for j in range(args.steps)]
    tot, rows, nnz = time_oracle_steps(w, steps, idxs, args.ref_nodes, mode)
    u = unit_of(mode)
    v = (nnz if mode == "rpi" else rows) / tot
    out = {"impl": "reference", "metric": "tSVD update throughput (nnz/s, rows/s) fp64",
           "value": v, "unit": u, "rows_per_s": rows / tot, "nnz_per_s": nnz / tot, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "warmup_steps_run": nwarm, "ms_per_step": 1e3 * tot / args.steps,
           "higher_is_better": True, "scaling": "strong" if mode in ("rpi", "rpi_rows") else "weak", "vs_baseline": None,
           "dtype": "f64", "data": f"synthetic (seeded, synth: {w.name})",
           "config": dict(desc, sample_nodes=None if mode in ("rpi", "rpi_rows") else args.ref_nodes),
           "cpu_baseline": {"value": v, "unit": u, "cores": _threads(), "kind": "oracle",
                            "sample": _sample_desc(args, steps, mode, args.steps)},
           "e2e": {"value": v, "unit": u, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
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
