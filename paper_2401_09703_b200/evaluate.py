"""F2: the downstream metrics of the paper's experiments, computed on the host
from scores the library returns (tsvd_score_pairs, tsvd_residual_fro).

* link prediction: score a candidate edge (i, j) by U[i] Σ V[j]^T, rank the
  held-out edges against sampled non-edges, report average precision (AP);
* collaborative filtering: predict rating (u, i) by U[u] Σ V[i]^T, report the
  mean squared error (MSE) on held-out ratings;
* the Frobenius residual ||A - Ã||_F comes from TSVD.residual_fro.

Evaluation, not the update path: plain numpy on a few million scores."""
from __future__ import annotations

import numpy as np


def average_precision(scores, labels) -> float:
    """AP = mean over the positives of the precision at each positive's rank (scores sorted
    descending; ties broken by input order, a stable sort)."""
    s = np.asarray(scores, dtype=np.float64)
    y = np.asarray(labels).astype(bool)
    if not y.any():
        return 0.0
    order = np.argsort(-s, kind="stable")
    hit = y[order]
    prec = np.cumsum(hit) / np.arange(1, len(hit) + 1)
    return float(prec[hit].mean())


def mse(pred, truth) -> float:
    p = np.asarray(pred, dtype=np.float64)
    t = np.asarray(truth, dtype=np.float64)
    return float(np.mean((p - t) ** 2)) if p.size else 0.0


def link_prediction_ap(t, pos_pairs, neg_pairs) -> float:
    """AP of held-out edges (pos) against non-edges (neg) scored by the context `t`."""
    pos, neg = np.asarray(pos_pairs, np.int64), np.asarray(neg_pairs, np.int64)
    pairs = np.concatenate([pos, neg])
    sc = t.score_pairs(pairs[:, 0], pairs[:, 1])
    return average_precision(sc, np.r_[np.ones(len(pos)), np.zeros(len(neg))])
