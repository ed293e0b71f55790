"""One-off probe: measured FP64 GEMM throughput (cuBLAS DGEMM via torch) and host facts.
The number is the FP64 roofline denominator reference for DESIGN.md (MEASURED_PEAKS has none)."""
import os, json, time, torch
r = {"cpu_count": os.cpu_count(), "sched_affinity": len(os.sched_getaffinity(0))}
d = torch.device("cuda:0")
p = torch.cuda.get_device_properties(d)
r["sm_count"] = p.multi_processor_count; r["l2"] = getattr(p, "L2_cache_size", None)
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=d); b = torch.randn(n, n, dtype=torch.float64, device=d)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    r[f"dgemm_{n}_tflops"] = 2 * n**3 / (best * 1e-3) / 1e12
x = torch.empty(2**28, dtype=torch.float64, device=d); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); best = 1e9
for _ in range(10):
    e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
r["copy_gbs"] = 2 * x.numel() * 8 / (best * 1e-3) / 1e9
print(json.dumps(r))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(r, open("gpurun_out/probe_fp64.json", "w"))
