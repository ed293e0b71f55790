"""CPU-side checks of the boundary (-m "not gpu"): libtsvd.so loads and exports every
symbol include/*.h declares; the binding's struct layouts match the header."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("tsvd.h", "tsvd_kernels.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(tsvd_\w+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    import paper_2401_09703_b200 as P
    lib = ctypes.CDLL(P.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 20
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding wraps every one of them
    assert set(P.EXPORTED) == declared


def test_version_string():
    import paper_2401_09703_b200 as P
    assert "sm_100a" in P.version()


def test_struct_sizes_match_header():
    """Compile a tiny C program against the header and compare sizeof/offsetof."""
    import subprocess
    import tempfile
    from paper_2401_09703_b200 import tsvd as T
    code = r'''
#include <stdio.h>
#include <stddef.h>
#include "tsvd.h"
int main(){printf("%zu %zu %zu %zu %zu %zu\n", sizeof(tsvd_opts), sizeof(tsvd_sparse), sizeof(tsvd_stats),
 offsetof(tsvd_stats, ms_pre), offsetof(tsvd_stats, launches), offsetof(tsvd_stats, top_flops));return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "s.c")
        open(src, "w").write(code)
        exe = os.path.join(d, "s")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    got = [ctypes.sizeof(T.tsvd_opts), ctypes.sizeof(T.tsvd_sparse), ctypes.sizeof(T.tsvd_stats),
           T.tsvd_stats.ms_pre.offset, T.tsvd_stats.launches.offset, T.tsvd_stats.top_flops.offset]
    assert [int(x) for x in out] == got


def test_no_gpu_call_fails_loudly_without_device():
    """On a box without a GPU the library must return an error, never compute on CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2401_09703_b200 as P
    with pytest.raises(P.TsvdError):
        P.TSVD(k=4, m_capacity=10, n_capacity=10)
