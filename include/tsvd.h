/*
 * tsvd.h — C-ABI of the B200-native sparse-aware truncated-SVD update library
 * (libtsvd.so), a from-scratch implementation of arXiv 2401.09703.
 *
 * The library maintains an approximate rank-k truncated SVD  A ≈ U_k Σ_k V_k^T
 * (Def 2) under the three operations of Theorem 1
 * (PAPER.md:406-421): add rows, add columns, update weights (A + D E_m^T), plus the
 * O(k²) query.  The state is the five-factor extended decomposition of Eq (4)
 * (PAPER.md:313-321):  U = U'·U'',  V = V'·V'',  A ≈ U' U'' Σ V''^T V'^T.
 *
 * Every step runs in this library's sm_100a CUDA kernels; there is no CPU path.
 *
 * Conventions (all functions):
 *  - Floating point is fp64 throughout; indices are int32 except CSR row pointers (int64).
 *  - Dense matrices are ROW-MAJOR (one row = one entity = k contiguous doubles).
 *  - A pointer argument may be device memory (of the context's device) or host
 *    memory (pageable or pinned); the library detects which with
 *    cudaPointerGetAttributes and stages host data through its own device workspace
 *    inside the call.  Output pointers follow the same rule.
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).  Calls
 *    enqueue on it and block the host only where noted (status / rank / convergence
 *    read-backs in the middle of an update).  An update returns once its last kernels
 *    are ENQUEUED, without synchronising the stream at its end: work enqueued later on
 *    the same stream (queries, the next update, a D2H copy of a result) sees the updated
 *    state; host code reading device memory directly must synchronise the stream first.
 *    Status is final at return (every failure is detected before the commit kernels).
 *  - Ownership: the context allocates and owns all state and workspace; input
 *    buffers are borrowed for the duration of the call; outputs are caller-owned.
 *  - Errors: every function returns a tsvd_status; on any error of an update the
 *    maintained state is unchanged (transactional) unless the error
 *    is TSVD_E_CUDA raised during the final commit, which leaves the context
 *    unusable.  tsvd_last_error() gives a one-line description.
 *  - Concurrency: single writer.  Queries may run concurrently with each other, not
 *    with an update.
 */
#ifndef TSVD_H_
#define TSVD_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tsvd_ctx tsvd_ctx;

typedef enum {
  TSVD_OK = 0,
  TSVD_E_SHAPE = 1,            /* dimension mismatch */
  TSVD_E_NOT_ORTHONORMAL = 2,  /* init: ||X^T X - I||_max > 1e-10 */
  TSVD_E_BAD_SIGMA = 3,        /* init: Σ not descending or negative */
  TSVD_E_NUMERIC = 4,          /* non-finite input value */
  TSVD_E_SVD_FAIL = 5,         /* core Jacobi SVD did not converge */
  TSVD_E_OOB = 6,              /* query index out of range */
  TSVD_E_INVALID = 7,          /* bad CSR: index out of range / unsorted / duplicate, bad opts */
  TSVD_E_OOM = 8,
  TSVD_E_CUDA = 9,
  TSVD_E_NCCL = 10,
  TSVD_E_UNSUPPORTED = 11,     /* option combination not implemented */
  TSVD_E_NOT_LOCAL = 12,       /* tsvd_query_row_local: the row lives on another process's shard */
  TSVD_E_STATE_VERSION = 13,   /* tsvd_load: a state file of another format version ("state_version") */
  TSVD_E_IO = 14               /* tsvd_save / tsvd_load: file error, bad magic, truncated file or checksum mismatch */
} tsvd_status;

/* How the augmented space of an update is orthogonalised. */
typedef enum {
  TSVD_EXACT = 0,  /* Alg 2 realised as Cholesky-QR with deflation */
  TSVD_GKL = 1,    /* Alg 6 */
  TSVD_RPI = 2     /* Alg 8 */
} tsvd_mode;

typedef struct {
  int32_t mode;          /* tsvd_mode */
  int32_t l;             /* GKL / RPI width (paper default 10) */
  int32_t t;             /* RPI power iterations (paper default 3) */
  int32_t flags;         /* bit 0: skip CSR validation (caller guarantees it);
                            bit 1: per-kernel-class device-time accounting (tsvd_stats.kern_*):
                            CUDA events around every kernel class, off by default (the event
                            records cost host time on launch-bound steps) */
  const double* sketch;  /* RPI: s x l row-major start block Ω; GKL: s-vector p1 (normalised
                            by the library).  update_weights: the D-side block followed by the
                            E-side block.  Host or device memory.  NULL: drawn on the device by
                            the counter-based generator K12 from `seed` (R13, §2.1;
                            side id 0 = U side, 1 = V side). */
  uint64_t seed;         /* K12 seed, used when sketch == NULL */
  double reset_cond;     /* MII threshold τ_reset on the 2-norm condition number of a new
                            multiplier (reading R18): no reset while its
                            cond_1 <= τ; above, cond_2 is estimated by power iterations (one
                            extra synchronisation) and decides; <= 0 -> 1e4 */
  double defl_tol;       /* Cholesky-QR deflation τ (reading R8); <= 0 -> 1e-12 */
} tsvd_opts;

/* s sparse update vectors of length `dim`, stored as CSR rows (row i = vector i).
 *   rows    : E_r            (s x n)
 *   columns : E_c^T          (s x m)   (column j of E_c is row j here)
 *   weights : D^T (s x m) and E_m^T (s x n)
 * Column indices must be in [0, dim), strictly increasing within a row. */
typedef struct {
  int64_t s;
  int64_t dim;
  int64_t nnz;
  const int64_t* row_ptr;  /* s+1 */
  const int32_t* col_idx;  /* nnz */
  const double* val;       /* nnz */
} tsvd_sparse;

typedef struct {
  int64_t s, nnz;           /* last update's size */
  int64_t s_eff;            /* update vectors left after dropping empty ones (exact mode) */
  int64_t rank[2];          /* numerical rank r kept by the orthogonaliser, [lift U side, lift V side] (-1: side not lifted) */
  int64_t touched[2];       /* |J| distinct base-factor rows touched, [U side, V side] */
  double theta_next;        /* θ_{k+1} of the core (0 if the core has only k values); on the Rayleigh-Ritz
                               core path the (k+1)-th Ritz value (second-order accurate, ~1e-10 rel.) */
  double energy;            /* Σ_i θ_i² over the full core spectrum */
  double cond[2];           /* cond_1 of the new U'', V'' (before any reset) */
  int32_t reset[2];         /* 1 if that side was materialised (MII reset) this update */
  int32_t jacobi_sweeps;    /* sweeps of the core one-sided Jacobi (summed over its calls) */
  int32_t core_iters;       /* subspace iterations of the core reduction (0: not used) */
  int32_t core_path;        /* 0 full Jacobi, 1 Cholesky-QR2 + Jacobi on R^T, 2 Rayleigh-Ritz reduction */
  int32_t core_rows, core_cols;
  int32_t total_resets;
  float ms_pre;             /* lift + orthogonalisation + core formation (PAPER.md:980 step 1) */
  float ms_svd;             /* core SVD (step 2) */
  float ms_post;            /* multiplier updates, append, sparse add, resets (step 3) */
  float ms_total;
  int32_t launches;         /* kernels this library launched during the update */
  /* Device time per kernel class, from CUDA events the library records on the update's
   * stream around each class's back-to-back launches (no host gaps inside), with the
   * algorithmic FP64 flops and bytes of those launches and their launch
   * count.  Kernel classes (non-overlapping: every launch belongs to one): 0 gather-SpMM
   * (K2), 1 sparse Gram (K3), 2 DMMA GEMM (K4: all dgemm calls of every step), 3 Cholesky
   * panels (K5 panel factor + K6 warp triangular solves), 4 fused small Cholesky + inverse,
   * 5 core Jacobi (K7/K8), 6 sparse row update (K10), 7 RPI / GKL sparse kernels.  top_*
   * repeat the class with the largest time (bench.py's roofline). */
  float kern_ms[8];
  double kern_flops[8];
  double kern_bytes[8];
  int32_t kern_launches[8];
  int32_t top_class;
  int32_t top_launches;
  float top_ms;
  double top_flops;
  double top_bytes;
} tsvd_stats;

/* Create a context on CUDA device `device` for rank k (k fixed); the
 * capacities are hints for U' and V' rows (grown by reallocation when exceeded). */
tsvd_status tsvd_create(tsvd_ctx** out, int32_t device, int64_t m_capacity,
                        int64_t n_capacity, int32_t k);
void tsvd_destroy(tsvd_ctx* ctx);
const char* tsvd_last_error(const tsvd_ctx* ctx);
const char* tsvd_version(void);

/* Row sharding of U' and V' over GPUs.  Global row i lives
 * on shard (i / block) % world (block-cyclic, so appended rows spread over the shards).
 * Every shard receives the same (replicated) inputs of every call; the partial products
 * over local rows are summed by ncclAllReduce (NCCL mode: one process per GPU,
 * virtual_shards = 1, this process owns shard `rank`; the 128-byte ncclUniqueId comes from
 * tsvd_nccl_unique_id on rank 0, shared by the caller) or on the device (virtual mode:
 * virtual_shards = world, all shards held by this context on one GPU — the partitioned
 * path exercised on a single GPU).  k x k, s x s and core work is replicated.  GKL is not
 * available on a sharded context (TSVD_E_UNSUPPORTED). */
typedef struct {
  int32_t world;           /* shards W >= 1 */
  int32_t rank;            /* NCCL mode: this process's shard in [0, W) */
  int32_t virtual_shards;  /* 1: NCCL mode; W: virtual mode */
  int32_t block;           /* rows per block of the block-cyclic deal (<= 0: 1024) */
  const void* nccl_id;     /* NCCL mode with W > 1: 128-byte ncclUniqueId (host memory) */
} tsvd_shard_opts;

tsvd_status tsvd_create_sharded(tsvd_ctx** out, int32_t device, const tsvd_shard_opts* opts, int64_t m_capacity,
                                int64_t n_capacity, int32_t k);
/* ncclGetUniqueId into out128 (128 bytes, host); NCCL is loaded with dlopen on first use. */
tsvd_status tsvd_nccl_unique_id(void* out128);

/* Host-only helpers of the block-cyclic deal (no GPU needed): the owner shard and local
 * row of global row i; the CSR of the columns of E (host arrays, dim = global rows of the
 * lift side) owned by `shard`, with local column indices — pass NULL outputs to get *nnz
 * first.  The device path (shard.cu) computes the same split. */
tsvd_status tsvd_shard_owner(int64_t i, int32_t world, int32_t block, int32_t* shard, int64_t* local);
tsvd_status tsvd_shard_split_host(const tsvd_sparse* E, int32_t world, int32_t block, int32_t shard,
                                  int64_t* row_ptr, int32_t* col_idx, double* val, int64_t* nnz);

/* Initialise from a truncated SVD: U (m x k), S (k), V (n x k).  U' = U, V' = V,
 * U'' = V'' = I.  Validates orthonormality and Σ. */
tsvd_status tsvd_init(tsvd_ctx* ctx, int64_t m, int64_t n, const double* U,
                      const double* S, const double* V, void* stream);

/* The initial truncated SVD on the GPU (the step before the update path: the paper initialises
 * on the first half of the data, with randomized numerical linear algebra,
 * PAPER.md:19): randomized subspace iteration with p = k + oversample columns (rounded up to
 * 16, at most 512), `power_iters` power steps (A^T A), start block from the counter-based
 * generator (seed, side 3), Cholesky-QR2 orthonormalisation, and the core Jacobi of the
 * projected p x p matrix; then tsvd_init on the result (U' = U, V' = V).  A: m rows of length
 * n (CSR, host or device, validated as an update block).  For rank(A) <= p the result is A's
 * exact rank-k truncated SVD to rounding; otherwise the randomized approximation.  Columns A
 * never touches get zero rows in V.  TSVD_E_SHAPE when m or the touched columns < p. */
tsvd_status tsvd_init_sparse(tsvd_ctx* ctx, const tsvd_sparse* A, int32_t oversample, int32_t power_iters,
                             uint64_t seed, void* stream);

/* Theorem 1 'Add rows' (Alg 9, core block read as
 * E_r V_k and the inverse of the NEW V'', R1/R7):
 * [Ã; E_r] -> SVD_k.  m grows by s; V' gets a sparse row update; U' gets s new rows. */
tsvd_status tsvd_update_rows(tsvd_ctx* ctx, const tsvd_sparse* Er, const tsvd_opts* opts,
                             void* stream);

/* Theorem 1 'Add columns' (Alg 3): [Ã, E_c] -> SVD_k.
 * EcT holds the s new columns as sparse rows (dim = m).  n grows by s. */
tsvd_status tsvd_update_cols(tsvd_ctx* ctx, const tsvd_sparse* EcT, const tsvd_opts* opts,
                             void* stream);

/* Theorem 1 'Update weights' (Alg 4 PAPER.md:375-397 with V''^{-1} on
 * line 8, R2): Ã + D E_m^T -> SVD_k.  DT: s x m, EmT: s x n. */
tsvd_status tsvd_update_weights(tsvd_ctx* ctx, const tsvd_sparse* DT, const tsvd_sparse* EmT,
                                const tsvd_opts* opts, void* stream);

/* Materialised factors: out = U' U'' (m x k) / V' V'' (n x k), row-major.  The represented
 * factor is not changed, but a deferred MII reset of the side (reading R18: an append-only
 * side keeps pending row blocks U = X' P U'') is materialised into X' first (one m x k x k
 * GEMM per pending block, on `stream`).  S: the k singular values, descending. */
tsvd_status tsvd_get_U(tsvd_ctx* ctx, double* out, void* stream);
tsvd_status tsvd_get_V(tsvd_ctx* ctx, double* out, void* stream);
tsvd_status tsvd_get_S(tsvd_ctx* ctx, double* out, void* stream);

/* Theorem 1 'Query(i)': row i of U (side 0) or V (side 1) in O(k²):
 * out (k doubles) = X'[i, :] X'' (inside a pending reset block: X'[i, :] P X'', O(k³)). */
tsvd_status tsvd_query_row(tsvd_ctx* ctx, int32_t side, int64_t i, double* out, void* stream);

/* Sharded contexts (tsvd_create_sharded).  get_U / get_V assemble the whole factor on every
 * process (NCCL mode: each process materialises its own rows, one ncclAllGather of the
 * per-shard blocks, a device row permutation); query_row is collective in NCCL mode (the
 * owning process computes the row in O(k^2) and broadcasts it). */

/* Row i of U (side 0) or V (side 1) computed by this process alone, O(k^2), without
 * any collective: TSVD_E_NOT_LOCAL when the row belongs to another process's shard (owner =
 * (i / block) % world, tsvd_shard_owner).  Unsharded contexts own every row. */
tsvd_status tsvd_query_row_local(tsvd_ctx* ctx, int32_t side, int64_t i, double* out, void* stream);

/* The rows of U (resp. V) held by local shard `local_shard` (0 in NCCL mode; 0..world-1 in
 * virtual mode), materialised X'_g X'' into out (nrows x k row-major, host or device; NULL:
 * sizes only), with their global row indices in global_rows (host, nrows entries; may be NULL):
 * local row j of shard g is global row ((j / block) world + g) block + j % block.  No
 * collective; *nrows receives the count (call with out = global_rows = NULL to size them). */
tsvd_status tsvd_get_U_shard(tsvd_ctx* ctx, int32_t local_shard, double* out, int64_t* global_rows, int64_t* nrows,
                             void* stream);
tsvd_status tsvd_get_V_shard(tsvd_ctx* ctx, int32_t local_shard, double* out, int64_t* global_rows, int64_t* nrows,
                             void* stream);

/* F2 — downstream evaluation on the maintained approximation Ã = U Σ V^T (PAPER.md:490-512:
 * link prediction scores the pair (i, j) by U[i] Σ V[j]^T, collaborative filtering predicts the
 * rating by it; AP / MSE are computed from these scores by the caller).
 * tsvd_score_pairs: out[p] = Ã[rows[p], cols[p]] for p < n (rows, cols int64, host or device;
 * out host or device), O(k^2) per pair, chunked; TSVD_E_OOB on an index out of range.
 * tsvd_residual_fro: for a sparse A (m rows of length n, CSR, host or device),
 * out3 (host) = { ||A - Ã||_F, <A, Ã>, ||A||_F^2 } with ||A - Ã||_F^2 = ||A||^2 - 2<A, Ã> + ||Σ||^2
 * (U, V orthonormal; Ã is never formed; the subtraction loses ~eps ||A||_F^2 absolute).
 * Unsharded contexts only (TSVD_E_UNSUPPORTED otherwise). */
tsvd_status tsvd_score_pairs(tsvd_ctx* ctx, int64_t n, const int64_t* rows, const int64_t* cols, double* out,
                             void* stream);
tsvd_status tsvd_residual_fro(tsvd_ctx* ctx, const tsvd_sparse* A, double* out3, void* stream);

/* Reset of PAPER.md:349-351: X' <- X' X'' on both sides (FP64 DMMA GEMM), X'' <- I. */
tsvd_status tsvd_materialize(tsvd_ctx* ctx, void* stream);

tsvd_status tsvd_dims(const tsvd_ctx* ctx, int64_t* m, int64_t* n, int32_t* k);

/* Reserve `bytes` of device memory in the stream-ordered pool the updates' scratch comes
 * from (allocated and freed once; the pool keeps it), so that the first updates of a stream
 * do not pay for growing the pool. */
tsvd_status tsvd_reserve(tsvd_ctx* ctx, int64_t bytes, void* stream);

/* State persistence ("a versioned binary container holding dims, k,
 * the five factors in little-endian 64-bit floats, plus a header checksum; a lossless round
 * trip is required (save→load→save byte-identical)").  File = a 64-byte header {char magic[8]
 * = "TSVDSTAT"; uint32 version = 1; int32 k; int64 m; int64 n; int64 total_resets; uint64
 * FNV-1a-64 of the payload; uint64 FNV-1a-64 of the header's first 48 bytes; 0 pad} followed by
 * the payload U' (m x k row-major), U'' (k x k), Σ (k), V' (n x k), V'' (k x k), all f64.
 * tsvd_save first materialises any deferred MII reset (the state it writes is the one get_U/V
 * would read, U = U' U''), writes `path`.tmp, flushes it and renames it over `path` (atomic
 * replace: a reader never sees a partial file).  tsvd_load replaces the context's state with
 * the file's (the context's k must equal the file's; its capacities grow as needed): a later
 * tsvd_save writes the same bytes.  Both synchronise the stream.  Unsharded contexts only
 * (TSVD_E_UNSUPPORTED otherwise).  Errors: TSVD_E_IO (open/read/write/rename failure, bad
 * magic, truncated file, checksum mismatch), TSVD_E_STATE_VERSION, TSVD_E_SHAPE (k differs).
 * tsvd_state_info reads only the header (k, m, n; any pointer may be NULL): no context needed. */
tsvd_status tsvd_save(tsvd_ctx* ctx, const char* path, void* stream);
tsvd_status tsvd_load(tsvd_ctx* ctx, const char* path, void* stream);
tsvd_status tsvd_state_info(const char* path, int32_t* k, int64_t* m, int64_t* n);

tsvd_status tsvd_last_stats(const tsvd_ctx* ctx, tsvd_stats* out);

/* The same without waiting for the device: the phase times ms_pre / ms_svd / ms_post /
 * ms_total of the last update are those of an earlier update if it has not completed yet
 * (everything else is current).  Updates return without synchronising at their end; this call
 * lets a caller read counters (launches, ranks, iterations) without forcing a sync. */
tsvd_status tsvd_last_stats_nowait(const tsvd_ctx* ctx, tsvd_stats* out);

#ifdef __cplusplus
}
#endif
#endif /* TSVD_H_ */
