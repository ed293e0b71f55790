"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the paper's method (arXiv 2401.09703): it only
draws sparse matrices / update batches with the shapes and value distributions of
BASELINE.json's configs, the initial truncated SVD the stream
starts from (harness work, SURVEY Appendix A #21 — Def 2, makes
the result independent of how the init was obtained) and Gaussian sketches
("random unitary columns", passed explicitly to both sides).

The recipes are stated in DESIGN.md §"Input recipe".
"""
from .generators import (  # noqa: F401
    Workload, Batch, tiny_rowappend, graph_nodeappend, ratings_rowappend,
    weights_rpi, synthetic_colappend, scaleout_rowappend, random_sparse, gaussian_sketch, unit_vector,
    init_truncated_svd, random_orthonormal,
)
from .counter_rng import counter_gaussian  # noqa: F401
