/*
 * tsvd_kernels.h — step-level C-ABI of libtsvd.so.
 *
 * Each entry point runs ONE step of the update path on the device, so that the
 * parity tests can check every kernel against the CPU oracle's plain definition of
 * that step (oracle/steps.py).  The update entry points in tsvd.h are composed of
 * exactly these kernels.
 *
 * Conventions: all pointers are DEVICE pointers on the current CUDA device, fp64
 * values, dense matrices ROW-MAJOR unless stated, `stream` is a cudaStream_t as void*.
 * Scratch memory is allocated stream-ordered inside the call and freed before return.
 * The calls are asynchronous unless stated; errors are returned as tsvd_status
 * (TSVD_E_CUDA on a launch failure, TSVD_E_INVALID on bad sizes).
 */
#ifndef TSVD_KERNELS_H_
#define TSVD_KERNELS_H_

#include "tsvd.h"

#ifdef __cplusplus
extern "C" {
#endif

/* K4: C = alpha op(A) op(B) + beta C, row-major with leading dimensions, FP64 DMMA
 * (mma.sync m8n8k4 f64).  op(X) = X^T when trans* != 0.  uplo = 1 computes only the
 * tiles that intersect the upper triangle (i <= j) and writes only i <= j (SYRK use). */
tsvd_status tsvd_k_dgemm(int32_t transA, int32_t transB, int64_t M, int64_t N, int64_t K,
                         double alpha, const double* A, int64_t lda, const double* B,
                         int64_t ldb, double beta, double* C, int64_t ldc, int32_t uplo,
                         void* stream);

/* K2, Lemma 1: W = E X  (E: s x d CSR, X: d x k, W: s x k). */
tsvd_status tsvd_k_gather_spmm(const tsvd_sparse* E, const double* X, int32_t k, double* W,
                               void* stream);

/* K3, Lemma 2 inner products of the sparse parts: G = E E^T (s x s,
 * row-major); only the upper triangle (i <= j, what K5 and the SYRK read) is defined, the
 * strictly lower triangle is left unspecified.  Deterministic (no float atomics).  May
 * synchronise the stream once (the hot/cold column split of batches with >= 16 nonzeros
 * per vector). */
tsvd_status tsvd_k_sparse_gram(const tsvd_sparse* E, double* G, void* stream);

/* K5, Alg 2 as Cholesky-QR with deflation (R8/R9):
 * in place, the upper triangle of G (s x s) becomes R with G = R^T R; pivot i is
 * deflated (row i of R = 0, keep[i] = 0) when its Schur diagonal <= tau * enorm2[i]
 * or enorm2[i] == 0.  The strictly lower triangle is zeroed.  *rank (host) = #kept;
 * this call synchronises the stream. */
tsvd_status tsvd_k_chol_deflate(double* G, int64_t s, const double* enorm2, double tau,
                                int32_t* keep, int64_t* rank, void* stream);

/* K6: X <- R^{-1} X restricted to kept pivots (R upper s x s from tsvd_k_chol_deflate,
 * X s x k); rows of deflated pivots are set to 0. */
tsvd_status tsvd_k_trsm_upper(const double* R, int64_t s, const int32_t* keep, double* X,
                              int32_t k, void* stream);

/* K7/K8: one-sided (block) Jacobi SVD of K (m x n COLUMN-MAJOR, m >= n), SVD_kk
 * (PAPER.md:81).  theta: all n singular values descending; F: m x kk and G: n x kk
 * COLUMN-MAJOR (left / right singular vectors).  *sweeps (host) = sweeps used;
 * returns TSVD_E_SVD_FAIL on non-convergence.  Synchronises the stream. */
tsvd_status tsvd_k_jacobi_svd(const double* K, int64_t m, int64_t n, int32_t kk, double* theta,
                              double* F, double* G, int32_t* sweeps, void* stream);

/* K15: Minv = M^{-1} (k x k) by Gauss-Jordan with partial pivoting; cond (device, 1
 * double) = ||M||_1 ||M^{-1}||_1 (the MII test, R18); +inf if singular. */
tsvd_status tsvd_k_inverse(const double* M, int32_t k, double* Minv, double* cond, void* stream);

/* The MII decision's cond_2 estimate (reading R18): *out (device) = an
 * estimate of ||M||_2 of the k x k row-major device matrix M by 40 power iterations on M^T M
 * (a lower estimate, exact to the top singular-value cluster).  Synchronises the stream. */
tsvd_status tsvd_k_norm2_est(const double* M, int32_t k, double* out, void* stream);

/* K10, the sparse matrix addition of PAPER.md:307 / Alg 9 line 7:
 * X[j, :] += sum_i E[i, j] Z[i, :]  (E: s x d CSR, Z: s x k, X: d x k). */
tsvd_status tsvd_k_scatter_add(const tsvd_sparse* E, const double* Z, int32_t k, double* X,
                               void* stream);

/* K11, reset / materialisation: X <- X M in place (X: rows x k, M: k x k). */
tsvd_status tsvd_k_materialize(double* X, int64_t rows, int32_t k, const double* M, void* stream);

/* A5, the core SVD as the update calls run it (DESIGN.md §6 "core SVD"): SVD_kk of K
 * (m x n COLUMN-MAJOR, m >= n, kk <= n).  theta: the kk+1 leading singular values
 * (min(n, kk+1) of them) descending; F: m x kk, G: n x kk COLUMN-MAJOR.  info (host, 4
 * doubles, may be NULL): {path (0 full Jacobi, 1 Cholesky-QR2 + Jacobi on R^T, 2 Rayleigh-
 * Ritz reduction by subspace iteration on K^T K), subspace iterations, Jacobi sweeps,
 * ||K||_F^2}.  Returns TSVD_E_SVD_FAIL on non-convergence.  Synchronises the stream. */
tsvd_status tsvd_k_core_svd(const double* K, int64_t m, int64_t n, int32_t kk, double* theta, double* F, double* G,
                            double* info, void* stream);

/* Cholesky-QR with deflation (the dense analogue of Alg 2; reading R8) of a
 * block X (rows x l, row-major, device) in place, `passes` passes (1 or 2): X <- X R^+ with
 * X_in = X_out R up to the deflated directions (a pivot whose Schur diagonal is <= tau times
 * its column's squared norm gets a zero row in R and a zero column in X).  R (l x l upper
 * row-major, device, may be NULL) receives the product of the passes' factors. */
tsvd_status tsvd_k_cholqr(double* X, int64_t rows, int64_t l, int32_t passes, double tau, double* R, void* stream);

/* The small-Gram step of every Cholesky-QR pass (reading R8/R30): in place, the upper
 * triangle of G (l x l row-major, device) becomes R with G = R^T R up to the deflated pivots
 * (pivot i deflated when its Schur diagonal <= tau * en[i], en = NULL: G's diagonal;
 * keep[i] = 0 and row i of R = 0), and T (l x l row-major, device) = R^+ (the inverse on the
 * kept pivots, zero rows / columns at deflated ones).  Does not synchronise. */
tsvd_status tsvd_k_chol_rinv(double* G, int64_t l, const double* en, double tau, int32_t* keep, double* T,
                             void* stream);

/* K12: out (s x l row-major, device) = the counter-based standard-normal block of
 * DESIGN.md §2.1 for (seed, side) — the RPI start block Ω / GKL p1
 * the update calls draw when tsvd_opts.sketch is NULL. */
tsvd_status tsvd_k_gaussian(uint64_t seed, int32_t side, int64_t s, int64_t l, double* out, void* stream);

/* RPI / GKL basis of one lift side (Alg 8 PAPER.md:904-920 / Alg 6) for the
 * s update vectors E (s x d CSR) against X (d x k row-major, orthonormal columns):
 * B' = E P on the touched rows J (returned densely as BJfull, d x l row-major, zero off J),
 * C' (k x l), P (s x l), all row-major device buffers, with Q = B' - X C' orthonormal
 * (deflated columns zero) and Q^T Z = P^T, Z = (I - X X^T) E^T.  opts: mode, l, t, sketch /
 * seed as in tsvd_update_*; side selects the K12 stream.  Synchronises the stream. */
tsvd_status tsvd_k_approx_basis(const tsvd_sparse* E, const double* X, int32_t k, const tsvd_opts* opts,
                                int32_t side, double* BJfull, double* Cp, double* P, void* stream);

/* Task order of the persistent tile-DAG kernels that realise K5 (kind 0: Cholesky with deflation,
 * Alg 2 PAPER.md:251-272 as DESIGN.md R8) and K6 (kind 1: back substitution, Eq (5)
 * PAPER.md:326) on nt = ceil(s/64) tiles and nkb = ceil(k/64) column blocks: the host reference
 * list, written as int32 quadruples {type, q, i, c} (type 0 chain, 1 S, 2 U, 4 V; DESIGN.md
 * §5) into out (host, up to cap quadruples; NULL: count only).  Returns the number of tasks, or
 * -1 for invalid arguments.  Host only (no device work): the tests check on the CPU that every
 * task's dependencies precede it. */
int64_t tsvd_dag_order(int32_t kind, int32_t nt, int32_t nkb, int32_t* out, int64_t cap);

/* Generates the same order on the device (the generator the kernels use) and returns the
 * number of entries that differ from tsvd_dag_order's (0 expected), -1 on error.  Synchronises. */
int64_t tsvd_dag_check(int32_t kind, int32_t nt, int32_t nkb);

#ifdef __cplusplus
}
#endif
#endif /* TSVD_KERNELS_H_ */
