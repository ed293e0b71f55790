"""Micro: the s x s Cholesky with deflation (K5) through the C-ABI step, tile-DAG path vs the
launch-per-panel path (TSVD_CHOL=panel in a child process).  python tools/micro_chol.py [s ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(sizes):
    import torch
    import paper_2401_09703_b200 as P
    for s in sizes:
        g = torch.Generator(device="cuda").manual_seed(s)
        E = torch.randn(s, 2 * s, device="cuda", dtype=torch.float64, generator=g)
        G0 = E @ E.T
        en = torch.diagonal(G0).clone()
        keep = torch.empty(s, dtype=torch.int32, device="cuda")
        G = G0.clone()
        P.k_chol_deflate(G, s, en, 1e-12, keep)
        torch.cuda.synchronize()
        R = torch.triu(G)
        err = ((R.T @ R - G0).abs().max() / G0.abs().max()).item()
        ts = []
        for _ in range(5):
            G.copy_(G0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            P.k_chol_deflate(G, s, en, 1e-12, keep)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"{os.environ.get('TSVD_CHOL', 'dag'):5s} s {s:6d}  {min(ts):8.3f} ms  err {err:.1e}  "
              f"{s**3 / 3 / min(ts) / 1e9:.2f} TF/s", flush=True)


if __name__ == "__main__":
    sizes = [int(x) for x in sys.argv[1:]] or [1000, 2500, 4500, 8000]
    if os.environ.get("MICRO_CHILD"):
        run(sizes)
    else:
        for mode in ("panel", "dag"):
            env = dict(os.environ, MICRO_CHILD="1", TSVD_CHOL=mode)
            subprocess.run([sys.executable, __file__] + [str(s) for s in sizes], env=env)
