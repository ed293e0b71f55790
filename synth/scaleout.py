"""BASELINE.json configs[4] (C5) scale-out row-append generator, vectorised and device-capable.

SURVEY §8(d) C5 recipe (and App A #26/#27): m = 20M rows, n = 2M columns; row degrees i.i.d.
from the discrete power law P(d) ∝ d^-2 on [5, 200000] (mean ≈ 48 -> ≈ 0.97B nonzeros);
the columns of a row drawn ∝ Zipf(0.8) over a seeded random permutation of the columns;
values U(0,1); the first m - 20 x 100k rows are the initial matrix, the last 2M rows arrive as
20 batches of 100k appended rows.

Reading of "columns per row without replacement": each row's d draws are taken with
replacement from the Zipf law and repeated columns merged (a row keeps its distinct columns,
slightly fewer than d for the heaviest rows) — the same sparsity structure, drawable in one
vectorised pass (the r1 generator drew n Gumbel keys per row: 4e13 draws at full size).

No arithmetic of the method: inverse-CDF sampling, sorting and deduplication only.  Runs on
torch's CUDA device for the full size (the host path is for the reduced test instances);
deterministic in (seed, device, torch version)."""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np


@dataclass
class DevCSR:
    """CSR on a torch device: int64 row_ptr, int32 col_idx, float64 val."""
    rows: int
    cols: int
    row_ptr: object
    col_idx: object
    val: object

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val.cpu().numpy(), self.col_idx.cpu().numpy().astype(np.int64),
                              self.row_ptr.cpu().numpy()), shape=(self.rows, self.cols))


@dataclass
class ScaleOut:
    k: int
    m: int
    n: int
    m_init: int
    init: DevCSR               # first m_init rows
    batches: List[DevCSR]      # appended row blocks
    meta: dict


def scaleout_rowappend(seed: int = 5, m: int = 20_000_000, n: int = 2_000_000, k: int = 256, batch: int = 100_000,
                       n_batches: int = 20, deg_min: int = 5, deg_max: int = 200_000, deg_exp: float = 2.0,
                       zipf: float = 0.8, device: str = "cuda", chunk_rows: int = 1 << 20) -> ScaleOut:
    import torch
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    dmax = min(deg_max, n)
    ds = torch.arange(deg_min, dmax + 1, dtype=torch.float64, device=dev)
    cdf_d = torch.cumsum(ds ** (-deg_exp), 0)
    cdf_d /= cdf_d[-1].clone()
    deg = torch.searchsorted(cdf_d, torch.rand(m, generator=g, dtype=torch.float64, device=dev)) + deg_min
    deg = torch.clamp(deg, max=dmax)
    perm = torch.randperm(n, generator=g, device=dev)
    cdf_c = torch.cumsum(torch.arange(1, n + 1, dtype=torch.float64, device=dev) ** (-zipf), 0)
    cdf_c /= cdf_c[-1].clone()
    m_init = m - n_batches * batch
    bounds = [0, m_init] + [m_init + (b + 1) * batch for b in range(n_batches)]
    parts_rp, parts_ci = [], []
    for r0 in range(0, m, chunk_rows):
        r1 = min(m, r0 + chunk_rows)
        d = deg[r0:r1]
        rowid = torch.repeat_interleave(torch.arange(r1 - r0, device=dev), d)
        u = torch.rand(int(rowid.numel()), generator=g, dtype=torch.float64, device=dev)
        col = perm[torch.clamp(torch.searchsorted(cdf_c, u), max=n - 1)]
        key = torch.unique(rowid * n + col)            # sorted: rows ascending, columns ascending
        row = key // n
        parts_ci.append((key - row * n).to(torch.int32))
        parts_rp.append(torch.bincount(row, minlength=r1 - r0))
        del rowid, u, col, key, row
    counts = torch.cat(parts_rp)
    ci = torch.cat(parts_ci)
    del parts_rp, parts_ci
    rp = torch.zeros(m + 1, dtype=torch.int64, device=dev)
    rp[1:] = torch.cumsum(counts, 0)
    val = torch.rand(int(ci.numel()), generator=g, dtype=torch.float64, device=dev)

    def block(a, b):
        p0, p1 = int(rp[a]), int(rp[b])
        return DevCSR(b - a, n, (rp[a:b + 1] - p0).contiguous(), ci[p0:p1].contiguous(), val[p0:p1].contiguous())

    init = block(bounds[0], bounds[1])
    batches = [block(bounds[i], bounds[i + 1]) for i in range(1, len(bounds) - 1)]
    del rp, ci, val
    if dev.type == "cuda":
        torch.cuda.empty_cache()
    return ScaleOut(k, m, n, m_init, init, batches,
                    meta=dict(seed=seed, nnz=init.nnz + sum(b.nnz for b in batches), deg_exp=deg_exp, zipf=zipf,
                              recipe="SURVEY §8(d) C5; draws with replacement, repeats merged"))


def uniform_sparse_colappend(n_rows: int = 100_000, n_cols: int = 100_000, nnz: int = 10_000_000, seed: int = 6,
                             device: str = "cuda"):
    """PAPER.md:1014-1021 (Fig 4): a random sparse n_rows x n_cols matrix with ~nnz nonzeros at
    uniform positions, U(0,1) values; returns (init, appended): init = the first half of the
    columns as an n_rows x n_cols/2 CSR, appended = the other half as CSR rows of E_c^T (one row
    per appended column, length n_rows).  Positions drawn with replacement, repeats merged."""
    import torch
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    half = n_cols // 2

    def block(rows, cols, cnt):
        key = torch.randint(0, rows * cols, (cnt,), generator=g, device=dev, dtype=torch.int64)
        key = torch.unique(key)
        r = key // cols
        c = (key - r * cols).to(torch.int32)
        rp = torch.zeros(rows + 1, dtype=torch.int64, device=dev)
        rp[1:] = torch.cumsum(torch.bincount(r, minlength=rows), 0)
        val = torch.rand(int(key.numel()), generator=g, dtype=torch.float64, device=dev)
        return DevCSR(rows, cols, rp, c.contiguous(), val)

    init = block(n_rows, half, nnz // 2)                 # A[:, :half] (rows x half)
    app = block(n_cols - half, n_rows, nnz - nnz // 2)   # E_c^T: appended columns as rows
    return init, app
