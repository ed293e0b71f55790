"""Build libtsvd.so in-tree with nvcc for sm_100a (no GPU needed: nvcc cross-compiles).

    python -m paper_2401_09703_b200.build        # or __graft_entry__.build()

Objects go to paper_2401_09703_b200/build/, the shared library to
paper_2401_09703_b200/libtsvd.so (git-ignored; travels to the GPU box with gpurun).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libtsvd.so")
SOURCES = ["gemm.cu", "sparse.cu", "dense.cu", "dag.cu", "jacobi.cu", "jacobi_cluster.cu", "init_svd.cu", "eval.cu", "variants.cu", "shard.cu", "api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xptxas", "-v"]


def _needs(obj: str, deps) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers += [os.path.join(HERE, "..", "include", h) for h in ("tsvd.h", "tsvd_kernels.h")]
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]

    def one(src):
        obj = os.path.join(OUT, src.replace(".cu", ".o"))
        if force or _needs(obj, [os.path.join(CSRC, src)] + headers):
            cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            with open(obj + ".log", "w") as f:
                f.write(r.stdout + r.stderr)
            if r.returncode != 0:
                err = "\n".join(l for l in r.stderr.splitlines()
                                if not l.startswith("ptxas info") and "bytes stack frame" not in l)
                raise RuntimeError(f"nvcc failed on {src}:\n{err[-4000:]}")
            if verbose:
                print(f"[build] {src}")
        return obj

    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(one, srcs))
    if force or _needs(LIB, objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
        if verbose:
            print(f"[build] linked {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
