"""Micro: the latency-bound small dense kernels of an RPI update — the l x l Cholesky + R^+
(chol_rinv, 22 per configs[3] update at l = 256) and the k x k multiplier inverse (inverse_gj,
2 per update at k = 128) — through the kernel-test C-ABI, CUDA-event timed (median of 20),
with their residuals.  Device time per call = the sum of the call's kernel durations from
CUDA events over a back-to-back burst (host launch cost hidden while the device is busy).  python tools/micro_small.py [l ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, reps=50):
    """per-call device time in us: CUDA events around reps back-to-back calls after a warm-up
    burst (the device stays busy, so its clocks stay up: isolated calls with a synchronize
    each measured 2-3x slower on an otherwise idle GPU)"""
    import torch
    for _ in range(reps):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps, []


def main(sizes):
    import torch
    import paper_2401_09703_b200 as P
    dev = torch.device("cuda:0")
    for l in sizes:
        g = torch.Generator(device="cuda").manual_seed(l)
        X = torch.randn(4 * l, l, device=dev, dtype=torch.float64, generator=g)
        G0 = X.T @ X
        G = G0.clone()
        T = torch.empty_like(G0)
        keep = torch.empty(l, dtype=torch.int32, device=dev)
        P.k_chol_rinv(G, l, None, 1e-14, keep, T)
        torch.cuda.synchronize()
        R = torch.triu(G)
        eR = ((R.T @ R - G0).abs().max() / G0.abs().max()).item()
        eT = (T @ R - torch.eye(l, device=dev, dtype=torch.float64)).abs().max().item()

        def run():
            G.copy_(G0)
            P.k_chol_rinv(G, l, None, 1e-14, keep, T)
        tc, nc = timed(run)
        tc -= timed(lambda: G.copy_(G0))[0]
        M = torch.randn(l, l, device=dev, dtype=torch.float64, generator=g) + 4 * torch.eye(l, device=dev,
                                                                                            dtype=torch.float64)
        Mi = torch.empty_like(M)
        cond = torch.empty(1, device=dev, dtype=torch.float64)
        P.k_inverse(M, l, Mi, cond)
        torch.cuda.synchronize()
        eI = (M @ Mi - torch.eye(l, device=dev, dtype=torch.float64)).abs().max().item()
        ti, ni = timed(lambda: P.k_inverse(M, l, Mi, cond))
        print(f"l={l:4d}  chol_rinv {tc:8.1f} us (|R'R-G|/|G| {eR:.1e}, |TR-I| {eT:.1e})   "
              f"inverse_gj {ti:8.1f} us (|M Minv - I| {eI:.1e})  {nc} {ni}", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [64, 96, 128, 192, 256])
