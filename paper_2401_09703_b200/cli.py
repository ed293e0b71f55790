"""Command-line front end (SPEC.md cli_io): build an initial
factorisation from a dataset file, stream update batches into a saved state, query rows.

    python -m paper_2401_09703_b200.cli init   --matrix A.mtx --k 16 [--fraction 0.5] --state s.tsvd
    python -m paper_2401_09703_b200.cli update --state s.tsvd --kind rows --E batch.mtx [--variant rpi --l 10 --t 3]
    python -m paper_2401_09703_b200.cli update --state s.tsvd --kind weights --D D.mtx --E E.mtx
    python -m paper_2401_09703_b200.cli query  --state s.tsvd --side u --index 0
    python -m paper_2401_09703_b200.cli info   --state s.tsvd

Every command prints one JSON line (the machine-readable record) and exits 0; usage errors
exit 2 (argparse), library errors 1 with {"error": ...}; `--verify` makes the exit status also
depend on the factors' orthonormality (||X^T X - I||_max <= 1e-8 on both sides).

Subcommands map one-to-one onto the C-ABI (Theorem 1's operations): init =
tsvd_init_sparse (the GPU randomized initial SVD, F1) on the leading fraction of the rows,
update = tsvd_update_rows / _cols / _weights, query = tsvd_query_row.  State files are the
tsvd_save container (include/tsvd.h "State persistence"): updates load, apply and save with an
atomic replace, holding an advisory lock on `<state>.lock`.  Dataset formats (SPEC.md
DatasetSpec): MatrixMarket (verbatim), an edge-list TSV (`--edges`, symmetric 0/1 with
`--undirected`: "all graphs are undirected"), a ratings CSV userId,movieId,rating
(contiguous re-indexing).  Batch files are MatrixMarket: rows / cols batches hold the s new
rows (s x n) / the s new columns (m x s); a weights batch A + D E^T holds D (m x s) and E
(n x s).  A first comment line `%tsvd-batch <kind>` names the kind when --kind is omitted.
"""
from __future__ import annotations

import argparse
import fcntl
import json
import os
import sys

import numpy as np
import scipy.sparse as sp

MODES = {"exact": 0, "gkl": 1, "rpi": 2}


# ----------------------------------------------------------------------------- dataset I/O
def load_edges(path: str, undirected: bool = True) -> sp.csr_matrix:
    """Edge list, one `u<TAB>v[<TAB>w]` per line ('#' comments); nodes are integer ids taken
    as indices.  Undirected: symmetric; duplicate edges keep the maximum value."""
    us, vs, ws = [], [], []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            line = line.strip()
            if not line or line.startswith("#") or line.startswith("%"):
                continue
            parts = line.split()
            if len(parts) < 2:
                raise ValueError(f"{path}:{ln}: malformed edge line")
            try:
                u, v = int(parts[0]), int(parts[1])
                w = float(parts[2]) if len(parts) > 2 else 1.0
            except ValueError as e:
                raise ValueError(f"{path}:{ln}: malformed edge line") from e
            if u < 0 or v < 0:
                raise ValueError(f"{path}:{ln}: negative node id")
            us.append(u)
            vs.append(v)
            ws.append(w)
    n = (max(max(us), max(vs)) + 1) if us else 0
    u, v, w = np.array(us, dtype=np.int64), np.array(vs, dtype=np.int64), np.array(ws)
    if undirected:
        u, v, w = np.concatenate([u, v]), np.concatenate([v, u]), np.concatenate([w, w])
    B = sp.coo_matrix((w, (u, v)), shape=(n, n))
    key = B.row * max(n, 1) + B.col
    order = np.lexsort((-B.data, key))
    first = np.ones(len(order), dtype=bool)
    first[1:] = key[order][1:] != key[order][:-1]
    sel = order[first]
    return sp.csr_matrix((B.data[sel], (B.row[sel], B.col[sel])), shape=(n, n))


def load_ratings(path: str) -> sp.csr_matrix:
    """userId,movieId,rating CSV (a header line allowed) -> user x item matrix, ids re-indexed
    contiguously in order of first appearance; duplicate pairs keep the maximum."""
    users, items, vals = {}, {}, {}
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            line = line.strip()
            if not line:
                continue
            parts = line.split(",")
            if len(parts) < 3:
                raise ValueError(f"{path}:{ln}: malformed ratings line")
            try:
                r = float(parts[2])
            except ValueError as e:
                if ln == 1:
                    continue  # header
                raise ValueError(f"{path}:{ln}: malformed ratings line") from e
            u = users.setdefault(parts[0], len(users))
            i = items.setdefault(parts[1], len(items))
            vals[(u, i)] = max(vals.get((u, i), -np.inf), r)
    if not vals:
        return sp.csr_matrix((len(users), len(items)))
    keys = np.array(list(vals.keys()), dtype=np.int64)
    return sp.csr_matrix((np.array(list(vals.values())), (keys[:, 0], keys[:, 1])), shape=(len(users), len(items)))


def load_matrix(args) -> sp.csr_matrix:
    if args.matrix:
        import scipy.io
        return sp.csr_matrix(scipy.io.mmread(args.matrix, spmatrix=False))
    if args.edges:
        return load_edges(args.edges, undirected=not args.directed)
    return load_ratings(args.ratings)


def read_batch_mtx(path: str):
    """(matrix, kind or None) of a MatrixMarket batch file with an optional `%tsvd-batch` line."""
    import scipy.io
    kind = None
    with open(path) as f:
        for line in f:
            if line.startswith("%tsvd-batch"):
                kind = line.split()[1].strip()
                break
            if not line.startswith("%"):
                break
    return sp.csr_matrix(scipy.io.mmread(path, spmatrix=False)), kind


# ----------------------------------------------------------------------------- commands
def _emit(rec: dict) -> None:
    print(json.dumps(rec), flush=True)


def _verify(t) -> float:
    import torch
    worst = 0.0
    for X in (t.get_U(), t.get_V()):
        Xd = X if isinstance(X, torch.Tensor) else torch.from_numpy(X)
        Xd = Xd.to(torch.device("cuda", t.device)) if torch.cuda.is_available() else Xd
        G = Xd.T @ Xd
        worst = max(worst, (G - torch.eye(G.shape[0], dtype=G.dtype, device=G.device)).abs().max().item())
    return worst


def cmd_init(args) -> int:
    from . import tsvd as T
    A = load_matrix(args)
    m = int(round(A.shape[0] * args.fraction))
    A0 = A[:m, : int(round(A.shape[1] * args.fraction))] if args.square else A[:m, :]
    t = T.TSVD(args.k, m_capacity=A0.shape[0], n_capacity=A0.shape[1], device=args.device)
    t.init_sparse(T.Sparse.from_scipy(A0), oversample=args.oversample, power_iters=args.power_iters, seed=args.seed)
    t.save(args.state)
    rec = {"cmd": "init", "state": args.state, "k": args.k, "m": A0.shape[0], "n": A0.shape[1], "nnz": int(A0.nnz),
           "sigma": [float(x) for x in t.get_S()]}
    ok = True
    if args.verify:
        rec["orth_err"] = _verify(t)
        ok = rec["orth_err"] <= 1e-8
    _emit(rec)
    return 0 if ok else 1


def cmd_update(args) -> int:
    from . import tsvd as T
    kind = args.kind
    E, k_file = read_batch_mtx(args.E)
    kind = kind or k_file
    if kind not in ("rows", "cols", "weights"):
        print("update: --kind rows|cols|weights (or a %tsvd-batch line) is required", file=sys.stderr)
        return 2
    if (kind == "weights") != bool(args.D):
        print("update: --D is required with (and only with) --kind weights", file=sys.stderr)
        return 2
    # one writer per state file: an advisory lock on a sidecar (the state file itself is
    # replaced by rename on save, so a lock on its inode would not exclude the next writer)
    fd = os.open(args.state + ".lock", os.O_RDWR | os.O_CREAT, 0o644)
    try:
        fcntl.flock(fd, fcntl.LOCK_EX)
        k, m, n = T.state_info(args.state)
        s = E.shape[0] if kind == "rows" else E.shape[1]
        t = T.TSVD.from_file(args.state, device=args.device, m_capacity=m + (s if kind == "rows" else 0),
                             n_capacity=n + (s if kind == "cols" else 0))
        opts = T.make_opts(mode=MODES[args.variant], l=args.l, t=args.t, seed=args.seed, reset_cond=args.reset_threshold)
        if kind == "rows":
            t.update_rows(T.Sparse.from_scipy(E), opts)
        elif kind == "cols":
            t.update_cols(T.Sparse.from_scipy(E.T.tocsr()), opts)
        else:
            D, _ = read_batch_mtx(args.D)
            t.update_weights(T.Sparse.from_scipy(D.T.tocsr()), T.Sparse.from_scipy(E.T.tocsr()), opts)
        st = t.stats()
        t.save(args.state)
        m2, n2, _ = t.dims()
        rec = {"cmd": "update", "kind": kind, "variant": args.variant, "s": int(s), "m": m2, "n": n2,
               "theta_next": st.get("theta_next"), "resets": st.get("reset"),
               "sigma": [float(x) for x in t.get_S()]}
        ok = True
        if args.verify:
            rec["orth_err"] = _verify(t)
            ok = rec["orth_err"] <= 1e-8
        _emit(rec)
        return 0 if ok else 1
    finally:
        os.close(fd)


def cmd_query(args) -> int:
    from . import tsvd as T
    t = T.TSVD.from_file(args.state, device=args.device)
    side = 0 if args.side == "u" else 1
    row = t.query_row(side, args.index)
    _emit({"cmd": "query", "side": args.side, "index": args.index, "row": [float(x) for x in np.asarray(row)],
           "sigma": [float(x) for x in t.get_S()]})
    return 0


def cmd_info(args) -> int:
    from . import tsvd as T
    k, m, n = T.state_info(args.state)
    _emit({"cmd": "info", "state": args.state, "k": k, "m": m, "n": n, "bytes": os.path.getsize(args.state)})
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="tsvd", description="sparse-aware truncated-SVD updates on a B200")
    ap.add_argument("--device", type=int, default=0)
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("init", help="initial truncated SVD of a dataset (GPU randomized SVD)")
    src = p.add_mutually_exclusive_group(required=True)
    src.add_argument("--matrix", help="MatrixMarket file")
    src.add_argument("--edges", help="edge-list TSV (undirected unless --directed)")
    src.add_argument("--ratings", help="userId,movieId,rating CSV")
    p.add_argument("--directed", action="store_true")
    p.add_argument("--k", type=int, required=True)
    p.add_argument("--fraction", type=float, default=0.5, help="leading fraction of the rows (P:486: 50%%)")
    p.add_argument("--square", action="store_true", help="take the leading fraction of the columns too (graphs)")
    p.add_argument("--oversample", type=int, default=32)
    p.add_argument("--power-iters", type=int, default=2)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--state", required=True)
    p.add_argument("--verify", action="store_true")
    p.set_defaults(fn=cmd_init)
    p = sub.add_parser("update", help="apply one batch to a saved state (atomic replace)")
    p.add_argument("--state", required=True)
    p.add_argument("--kind", choices=("rows", "cols", "weights"))
    p.add_argument("--E", required=True, help="MatrixMarket: new rows (s x n) / new columns (m x s) / E (n x s)")
    p.add_argument("--D", help="MatrixMarket D (m x s) of a weights update A + D E^T")
    p.add_argument("--variant", choices=tuple(MODES), default="exact")
    p.add_argument("--l", type=int, default=10, help="GKL / RPI width (P:479)")
    p.add_argument("--t", type=int, default=3, help="RPI power iterations (P:480)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--reset-threshold", type=float, default=1e4)
    p.add_argument("--verify", action="store_true")
    p.set_defaults(fn=cmd_update)
    p = sub.add_parser("query", help="row i of U or V (O(k^2), Query(i) P:418) and sigma")
    p.add_argument("--state", required=True)
    p.add_argument("--side", choices=("u", "v"), required=True)
    p.add_argument("--index", type=int, required=True)
    p.set_defaults(fn=cmd_query)
    p = sub.add_parser("info", help="a state file's header")
    p.add_argument("--state", required=True)
    p.set_defaults(fn=cmd_info)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except Exception as e:  # library / file errors: one JSON error record, exit 1
        _emit({"cmd": args.cmd, "error": f"{type(e).__name__}: {e}"})
        return 1


if __name__ == "__main__":
    sys.exit(main())
