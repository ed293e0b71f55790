"""Micro: device time of the k x k Gauss-Jordan inverse kernel via the profiler."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2401_09703_b200 as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 64
M = torch.tensor(np.random.default_rng(1).standard_normal((k, k)) + 2 * np.eye(k), device='cuda')
Minv = torch.empty_like(M); cond = torch.empty(1, dtype=torch.float64, device='cuda')
for _ in range(10): P.k_inverse(M, k, Minv, cond)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(20): P.k_inverse(M, k, Minv, cond)
    torch.cuda.synchronize()
for e in prof.key_averages():
    if 'gj' in e.key:
        t = e.device_time_total if hasattr(e, 'device_time_total') else e.cuda_time_total
        print(e.key[:40], 'device us avg', t / e.count)
err = np.abs(Minv.cpu().numpy() @ M.cpu().numpy() - np.eye(k)).max()
print('max |Minv M - I|', err)
