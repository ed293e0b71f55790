// ops.h — host-side launchers of the libtsvd kernels (internal; C++ linkage).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace tsvd {

// Number of kernels this library launched on the calling thread (reported in
// tsvd_stats.launches and by bench.py as gpu_launches).
extern thread_local long long g_launches;

// Device-resident CSR of s update vectors of length dim.
struct DevCSR {
  int64_t s = 0, dim = 0, nnz = 0;
  const int64_t* row_ptr = nullptr;
  const int32_t* col_idx = nullptr;
  const double* val = nullptr;
};

// Device CSC (the transpose) restricted to the touched columns J.
struct DevCSC {
  int64_t nJ = 0;           // |J| (host copy)
  int64_t* colptr = nullptr;  // dim+1 (over all columns)
  int32_t* J = nullptr;       // touched columns, ascending, nJ entries (device)
  int32_t* row = nullptr;     // nnz: row (update-vector) index
  double* val = nullptr;      // nnz
  int64_t* jpos = nullptr;    // dim+1: compact index of column j in J (valid where touched)
};

// Simple stream-ordered scratch arena: every allocation made between mark() and
// release() is freed by release().
// Stream-ordered scratch of one update.  Requests up to 16 MB are carved (256-byte aligned)
// out of 64 MB chunks, larger ones get their own block; everything is returned to the pool at
// release — a few cudaFreeAsync calls at the end of an update instead of one per request
// (~50: ~100 us of host time during which the GPU waited for the next update's first launch).
struct Scratch {
  static constexpr size_t kChunk = size_t(64) << 20, kSmall = size_t(16) << 20;
  cudaStream_t st;
  void* ptrs[128];
  int n = 0;
  cudaError_t err = cudaSuccess;
  char* cur = nullptr;
  size_t left = 0;
  explicit Scratch(cudaStream_t s) : st(s) {}
  void* raw(size_t bytes) {
    void* p = nullptr;
    cudaError_t e = n < 128 ? cudaMallocAsync(&p, bytes, st) : cudaErrorMemoryAllocation;
    if (e != cudaSuccess) { err = e; return nullptr; }
    ptrs[n++] = p;
    return p;
  }
  template <class T>
  T* alloc(size_t count) {
    if (count == 0) count = 1;
    const size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    if (bytes > kSmall) return static_cast<T*>(raw(bytes));
    if (bytes > left) {
      cur = static_cast<char*>(raw(kChunk));
      if (!cur) { left = 0; return nullptr; }
      left = kChunk;
    }
    void* p = cur;
    cur += bytes;
    left -= bytes;
    return static_cast<T*>(p);
  }
  // mark / rewind: allocations made after a mark are returned by rewind (stream-ordered, so
  // kernels already enqueued on st that use them are unaffected); loops that allocate per
  // iteration (the core subspace iteration's Cholesky-QR workspaces) rewind every pass
  struct Mark {
    int n;
    char* cur;
    size_t left;
  };
  Mark mark() const { return Mark{n, cur, left}; }
  void rewind(const Mark& m) {
    for (int i = m.n; i < n; ++i) cudaFreeAsync(ptrs[i], st);
    n = m.n;
    cur = m.cur;
    left = m.left;
  }
  void release() {
    for (int i = 0; i < n; ++i) cudaFreeAsync(ptrs[i], st);
    n = 0;
    cur = nullptr;
    left = 0;
  }
  ~Scratch() { release(); }
};

// ---- gemm.cu
// kr (optional): per 64-row block of C, the range [x, y) of K outside which that block's rows
// of op(A) are structurally zero (the products skip it); kfrac = nonzero fraction (accounting)
// b_upper: B is upper triangular (B[k][n] = 0 for k > n; e.g. T = R^+ of a Cholesky factor): each
// N tile reads only the K rows its columns can use (half the flops of the full product)
cudaError_t dgemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, CMat A, CMat B,
                  double beta, Mat C, int uplo, const int2* kr = nullptr, double kfrac = 1.0, bool b_upper = false);
// C (M x N) = A (M x K) B (K x N upper triangular), row-major, no transposes
cudaError_t dgemm_rm_btri(cudaStream_t st, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                          const double* B, int64_t ldb, double* C, int64_t ldc);
// call after writing new contents into a kr array (invalidates the cached split plans)
void kr_plan_epoch_bump();
// row-major convenience: C(MxN, ldc) = alpha op(A) op(B) + beta C
cudaError_t dgemm_rm(cudaStream_t st, bool tA, bool tB, int64_t M, int64_t N, int64_t K, double alpha,
                     const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                     int64_t ldc, int uplo = 0);

// ---- sparse.cu
// Selection of the update vectors that are nonempty (and, for weight updates, whose
// partner in B is nonempty too): an empty e_i contributes a zero row to the Gram, the core
// and the augmented matrix, so dropping it leaves the update unchanged.
struct RowSel {
  int64_t s = 0, s_eff = 0;
  int64_t* flag = nullptr;  // s+1
  int64_t* pos = nullptr;   // s+1: compact index
  int64_t* map = nullptr;   // (select_unique) s: compact index of the row's representative, -1 empty
  double* scl = nullptr;    // (select_unique) s: 1 / sqrt(multiplicity of the row's group)
};
// empty rows dropped and identical rows merged into one row scaled by sqrt(multiplicity)
cudaError_t select_unique(cudaStream_t st, const DevCSR& A, DevCSR& Aout, RowSel& sel, Scratch& ws,
                          int64_t* h_scratch);
cudaError_t select_nonempty(cudaStream_t st, const DevCSR& A, const DevCSR* B, DevCSR& Aout, DevCSR* Bout,
                            RowSel& sel, Scratch& ws, int64_t* h_scratch);
// dst (sel.s x k) = the compact rows of src (sel.s_eff x k) at their positions, zeros elsewhere
cudaError_t expand_selected(cudaStream_t st, const RowSel& sel, const double* src, int k, double* dst);
cudaError_t scan_exclusive_i64(cudaStream_t st, const int64_t* in, int64_t* out, int64_t n, Scratch& ws);
cudaError_t validate_csr(cudaStream_t st, const DevCSR& E, int* d_flag);
cudaError_t build_csc(cudaStream_t st, const DevCSR& E, DevCSC& out, Scratch& ws, int64_t* h_nJ);
cudaError_t gather_spmm(cudaStream_t st, const DevCSR& E, const double* X, int k, double* W);
// W (s x width, ldw) = E X (dim x width, ldx); width a multiple of 16 (panels of the fast widths)
cudaError_t gather_spmm_ld(cudaStream_t st, const DevCSR& E, const double* X, int64_t ldx, int width, double* W,
                           int64_t ldw);
cudaError_t sparse_gram(cudaStream_t st, const DevCSR& E, const DevCSC& C, double* G, Scratch& ws);
// the flat sparse enumeration of the products of the columns with at most `hot` entries
cudaError_t sparse_gram_cold(cudaStream_t st, const DevCSR& E, const DevCSC& C, double* G, Scratch& ws, int64_t hot);
// number of scalar products of sparse_gram (synchronises: accounting of the profiling pass only)
double sparse_gram_products(cudaStream_t st, const DevCSR& E, const DevCSC& C);
cudaError_t pad_even_rows(cudaStream_t st, DevCSR& E, Scratch& ws);
cudaError_t scatter_add(cudaStream_t st, const DevCSC& C, int64_t nnz, const double* Z, int k, double* X);
cudaError_t row_sqnorms(cudaStream_t st, const DevCSR& E, double* out);

// ---- dense.cu
// Tb (optional, nt = ceil(s/64) blocks of 64 x 64): receives T_qq = R_qq^+ of every diagonal
// tile, which trsm_upper uses when given (the tile-DAG path of dag.cu); null = scratch.  With Tb
// given the strict lower triangle of G is left as it was (the lift's consumers read R's upper
// part only); without, it is zeroed (R returned as a full upper-triangular matrix).
cudaError_t chol_deflate(cudaStream_t st, double* G, int64_t s, const double* enorm2, double tau,
                         int32_t* keep, double* Tb = nullptr);
cudaError_t trsm_upper(cudaStream_t st, const double* R, int64_t s, const int32_t* keep, double* X, int k,
                       const double* Tb = nullptr);
// ---- dag.cu (persistent tile-DAG kernels; enorm2 required)
cudaError_t chol_dag(cudaStream_t st, double* G, int64_t s, const double* enorm2, double tau, int32_t* keep,
                     double* Tb, bool zero_lower);
cudaError_t trsm_dag(cudaStream_t st, const double* R, int64_t s, const double* Tb, double* X, int k);
bool dag_enabled();
// l <= 128: G (l x l Gram, upper part) -> R in place (chol_deflate semantics; enorm2 null =
// use G's diagonal) and T = R^+ (l x l upper, the inverse on the kept pivots), one CTA
cudaError_t chol_inv_small(cudaStream_t st, double* G, int l, const double* enorm2, double tau, int32_t* keep,
                           double* T);
cudaError_t inverse_gj(cudaStream_t st, const double* M, int k, double* Minv, double* cond, Scratch& ws);
// ||A||_2 estimates (40 power iterations on A^T A) of nm <= 4 k x k row-major matrices -> d_out[i]
cudaError_t norm2_estimates(cudaStream_t st, const double* const* mats, int nm, int k, double* d_out);
cudaError_t materialize_rows(cudaStream_t st, double* X, int64_t rows, int k, const double* M);
cudaError_t set_identity(cudaStream_t st, double* M, int k);
cudaError_t compact_keep(cudaStream_t st, const int32_t* keep, int64_t s, int32_t* kidx, int64_t* d_r,
                         Scratch& ws);
cudaError_t copy_diag(cudaStream_t st, const double* G, int64_t s, double* d);
cudaError_t build_core_rows(cudaStream_t st, int k, int64_t s, int64_t r, const double* Sigma,
                            const double* P0, const double* R, const int32_t* kidx, double* K);
cudaError_t build_lift_block(cudaStream_t st, int k, int64_t s, int64_t r, const double* P0,
                             const double* R, const int32_t* kidx, double* L);
cudaError_t add_diag_sigma(cudaStream_t st, double* K, int64_t ldk, int k, const double* Sigma,
                           bool colmajor);
cudaError_t expand_rows(cudaStream_t st, const double* Gc, int64_t ldg, int k, int64_t s, const int32_t* kidx,
                        double* Gfull);
cudaError_t colmajor_to_rowmajor(cudaStream_t st, const double* A, int64_t lda, int64_t rows, int64_t cols,
                                 double* out, int64_t ldo);
cudaError_t check_init(cudaStream_t st, const double* X, int64_t rows, int k, double* d_maxdev, Scratch& ws);
cudaError_t find_nonfinite(cudaStream_t st, const double* v, int64_t n, int* d_flag);
// C(i,j) = beta C(i,j) + alpha A(i,j) over rows x cols (strided views)
cudaError_t mat_axpby(cudaStream_t st, int64_t rows, int64_t cols, double alpha, CMat A, double beta, Mat C);

// ---- per-kernel device-time accounting (tsvd_stats.kern_*, bench.py roofline)
// Kernel classes, non-overlapping (each launch belongs to one; include/tsvd.h): 0 gather-SpMM
// (K2), 1 sparse Gram (K3), 2 DMMA GEMM (K4, every dgemm call), 3 Cholesky panels (K5 panel
// factor + K6 warp triangular solves), 4 fused small Cholesky + inverse, 5 core Jacobi
// (K7/K8), 6 sparse row update (K10), 7 RPI / GKL sparse kernels (K13/K14).
constexpr int KC_GATHER = 0, KC_SGRAM = 1, KC_GEMM = 2, KC_PANEL = 3, KC_SMALLCHOL = 4, KC_JACOBI = 5,
              KC_SCATTER = 6, KC_APPROX = 7, KC_N = 8;
struct KProfiler {
  struct Rec {
    int cls;
    cudaEvent_t a, b;
    double flops, bytes;
    long long l0, l1;
    cudaStream_t s;
  };
  cudaStream_t st = nullptr;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t get();
  int begin(int cls, double flops, double bytes, cudaStream_t on = nullptr);
  void end(int idx);
  void set(int idx, double flops, double bytes) {
    if (idx >= 0) { recs[idx].flops = flops; recs[idx].bytes = bytes; }
  }
  // sum per class (synchronises on the last event)
  void resolve(float* ms, double* flops, double* bytes, int* launches);
  void reset(cudaStream_t s) { st = s; recs.clear(); used = 0; }
  ~KProfiler();
};
extern thread_local KProfiler* g_prof;
struct KScope {
  int idx = -1;
  KScope(int cls, double flops = 0.0, double bytes = 0.0) {
    if (g_prof) idx = g_prof->begin(cls, flops, bytes);
  }
  void set(double flops, double bytes) {
    if (g_prof) g_prof->set(idx, flops, bytes);
  }
  ~KScope() {
    if (g_prof && idx >= 0) g_prof->end(idx);
  }
};

// Device-time account of one kernel class (bench.py roofline, tsvd_stats.top_*).
struct KProf {
  float ms = 0.f;
  int launches = 0;
  double flops = 0.0, bytes = 0.0;
};

// ---- init_svd.cu (F1: randomized truncated SVD of a sparse A on the GPU)
cudaError_t randomized_svd(cudaStream_t st, const DevCSR& A, int k, int p, int q, uint64_t seed, double* U, double* S,
                           double* V, Scratch& ws, int* sweeps, bool* converged);

// ---- eval.cu (F2: scores U[i] Σ V[j]^T and <A, Ã> for the downstream evaluation)
cudaError_t score_pairs(cudaStream_t st, const double* Xu, const double* Mu, const double* Xv, const double* Mv,
                        const double* S, int k, int64_t n, const int64_t* rows, const int64_t* cols, double* out,
                        Scratch& ws);
cudaError_t sparse_inner(cudaStream_t st, const double* Xu, const double* Mu, const double* Xv, const double* Mv,
                         const double* S, int k, const DevCSR& A, double* h_out, Scratch& ws);
cudaError_t pairs_in_range(cudaStream_t st, int64_t n, const int64_t* r, const int64_t* c, int64_t m, int64_t nn,
                           int* d_flag, bool* ok);

// ---- jacobi_cluster.cu (K9: one-sided Jacobi resident in one CTA cluster, 128 < n <= 512)
bool k9_supported(int64_t m, int64_t n);
// kt > 0: only the kt largest triplets are needed (the tail's internal rotations may be skipped;
// theta beyond kt then holds column norms, not singular values)
cudaError_t jacobi_cluster(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, int kk, double tol,
                           double* theta, double* F, int64_t ldf, int* info, double* tiny, int kt = 0);

// ---- variants.cu (approximate augmented space: RPI Alg 8, GKL Alg 6) and helpers
// index maps that let the two RPI sparse products run as K2 gather-SpMMs (hub rows on CTAs):
// rpJ (nJ+1) the CSC's row pointer compacted to J, ciJ (nnz) E's column indices mapped to J
struct GatherMaps {
  int64_t* rpJ = nullptr;
  int32_t* ciJ = nullptr;
};
cudaError_t gather_maps(cudaStream_t st, const DevCSR& E, const DevCSC& C, GatherMaps& out, Scratch& ws);
// BJ[jj, :] = sum_q val_q P[row_q, :] over CSC column J[jj] (B' = E P on the support J)
cudaError_t csc_spmm(cudaStream_t st, const DevCSC& C, const GatherMaps* gm, int64_t nnz, const double* P, int w,
                     double* BJ);
// out[i, :] = sum_p v_p BJ[jpos[col_p], :]   (E^T B' for B' held on J)
cudaError_t csr_gather_compact(cudaStream_t st, const DevCSR& E, const int64_t* jpos, const GatherMaps* gm,
                               const double* BJ, int w, double* out);
// X <- X R^{-1} (R upper l x l row-major, kept pivots; deflated columns of X set to 0), X rows x l row-major
cudaError_t trsm_right_upper(cudaStream_t st, const double* R, int64_t l, const int32_t* keep, double* X,
                             int64_t rows);
// X[J[jj], :] += Z[jj, :]
cudaError_t index_add_rows(cudaStream_t st, const int32_t* J, int64_t nJ, const double* Z, int k, double* X);
// K12: Omega (s x l row-major) standard normal from the counter-based generator
cudaError_t counter_gaussian(cudaStream_t st, uint64_t seed, int side, int64_t s, int64_t l, double* Omega);
// K (col-major (k+s) x (k+l)) = [[diag Σ, 0], [P0, P]]
cudaError_t build_core_approx(cudaStream_t st, int k, int64_t s, int64_t l, const double* Sigma, const double* P0,
                              const double* P, double* K);
// L (row-major (k+l) x s) = [P0^T; P^T]
cudaError_t build_lift_block_approx(cudaStream_t st, int k, int64_t s, int64_t l, const double* P0, const double* P,
                                    double* L);
// GKL (Alg 6) on the tuples: outputs BJ (nJ x l), Cp (k x l), P (s x l), all row-major
cudaError_t gkl_basis(cudaStream_t st, const DevCSR& E, const DevCSC& C, const double* P0, int k, const double* p1,
                      int l, double tau, double* BJ, double* Cp, double* P, Scratch& ws);
// CholQR2 with deflation of a dense block (rows x l row-major) in place
cudaError_t cholqr2_dense(cudaStream_t st, double* X, int64_t rows, int64_t l, double tau, Scratch& ws);
// Cholesky with deflation of the l x l Gram in G -> R (in G) and T = R^+ (l x l row-major)
cudaError_t chol_rinv(cudaStream_t st, double* G, int64_t l, const double* en, double tau, int32_t* keep, double* T,
                      Scratch& ws, bool zero_lower);
// `passes` of Cholesky-QR with deflation (1: orthogonality ~ eps cond^2; 2: ~ eps), R optional
cudaError_t cholqr_dense(cudaStream_t st, double* X, int64_t rows, int64_t l, double tau, int passes, double* R,
                         Scratch& ws, double* Xout = nullptr);
// X <- X R^{-1} over kept pivots via the explicit triangular inverse and one GEMM
cudaError_t apply_rinv(cudaStream_t st, const double* R, int64_t l, const int32_t* keep, double* X, int64_t rows,
                       Scratch& ws);
// CholQR2 with deflation of the SV-LCOV tuple (BJ nJ x l, Cp k x l) in place (Alg 2 on tuples)
cudaError_t cholqr2_tuple(cudaStream_t st, double* BJ, int64_t nJ, double* Cp, int k, int64_t l, double tau,
                          Scratch& ws);

// CholQR2 with deflation of a dense block (rows x l row-major) in place, returning the
// triangular factor R (l x l row-major upper, R = R2 R1) with X_in = X_out R
cudaError_t cholqr2_r(cudaStream_t st, double* X, int64_t rows, int64_t l, double tau, double* R, Scratch& ws);

// ---- shard.cu (row sharding)
struct NcclUniqueIdBytes {
  char b[128];
};
int64_t shard_rows(int64_t rows, int g, int world, int block);
// E (s x d, replicated) -> the block of the columns owned by shard g, local column indices
cudaError_t shard_split(cudaStream_t st, const DevCSR& E, int g, int world, int block, int64_t dim_local, DevCSR& out,
                        Scratch& ws, int64_t* h_scratch);
cudaError_t shard_gather_owned(cudaStream_t st, const double* full, int64_t rows, int k, int g, int world, int block,
                               double* Xg);
cudaError_t shard_put_rows(cudaStream_t st, const double* R, int64_t s, int k, int64_t row0, int g, int world,
                           int block, double* Xg);
cudaError_t shard_scatter_owned(cudaStream_t st, const double* Xl, int64_t rows, int k, int g, int world, int block,
                                double* out);
cudaError_t add_into(cudaStream_t st, double* acc, const double* x, int64_t n);
int nccl_unique_id(void* out128);
int nccl_comm_init(void** comm, int world, const void* id128, int rank);
int nccl_allreduce_sum_f64(void* comm, double* buf, int64_t count, cudaStream_t st);
int nccl_allgather_f64(void* comm, const double* send, double* recv, int64_t count, cudaStream_t st);
int nccl_broadcast_f64(void* comm, const double* send, double* recv, int64_t count, int root, cudaStream_t st);
// rows of an all-gather of per-shard blocks (maxl rows each) to their global positions
cudaError_t shard_unshuffle(cudaStream_t st, const double* G, int64_t rows, int64_t maxl, int k, int world, int block,
                            double* out);
int64_t shard_global_row(int64_t j, int g, int world, int block);
void nccl_comm_destroy(void* comm);
const char* nccl_error(int rc);

// ---- jacobi.cu
struct CoreInfo {
  int path = 0;       // 0 full Jacobi of the core, 1 Cholesky-QR2 preconditioned, 2 subspace Rayleigh-Ritz
  int iters = 0;      // subspace iterations
  int sweeps = 0;     // Jacobi sweeps (summed)
  bool converged = false;
  double energy = 0;  // ||K||_F^2 = sum of all theta^2
  double theta_next = 0;  // theta_{kk+1}
  int hint = 0;       // in: iteration of the first Rayleigh-Ritz check (0: default 8), e.g. the count the
                      // previous update of the same stream needed
  double growth = 0;  // in/out: (theta_1 / theta_b)^2 per power step (0: unknown), carried across updates
  double thb2 = 0;    // in/out: theta_b^2 of the last Rayleigh-Ritz check (Chebyshev interval; 0: unknown)
  int hint_next = 0;  // out: suggested first-check iteration for the next update of the stream (0: none)
  int b_hint = 0;     // in: subspace width suggested by the previous update of the stream (0: default)
  int b_next = 0;     // out: the narrowest width (kk + 16 j) whose Ritz ratio (theta_b / theta_kk)^2 at
                      // this update's converged check was below 1e-3 (0: keep the default)
  bool defer_theta_next = false;           // in: the caller synchronises later and reads theta_next
  double* theta_next_dst = nullptr;        // in (deferred): caller-owned pinned host word for theta_next
  const double* theta_next_host = nullptr;  // out (deferred): = theta_next_dst, valid after the caller's sync
};
// SVD_kk of the core A (m x n col-major, m >= n): theta (kk+1 values, descending; fewer
// if n <= kk), F (m x kk, ldf) and G (n x kk, ldg) col-major.  Large cores are reduced by
// Rayleigh-Ritz on a subspace iteration of A^T A and finished by the one-sided Jacobi.
// shape (optional): A is the exact-mode core [Σ, 0; C0^T, R_kept^T] (k + s) x (k + r) with
// the kept pivots klist (ascending, device), so column k + c is zero above row k + klist[c]:
// the subspace products skip the structurally zero part (about half of A).
struct CoreShape {
  int k;
  int64_t s, r;
  const int32_t* klist;
};
cudaError_t core_svd(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, int kk, double* theta,
                     double* F, int64_t ldf, double* G, int64_t ldg, CoreInfo* info, Scratch& ws,
                     KProf* prof = nullptr, const CoreShape* shape = nullptr);
// One-sided block Jacobi SVD of A (m x n col-major, lda), top kk triplets.
// theta(n) all values descending; F (m x kk, ldf) and G (n x kk, ldg) col-major.
cudaError_t jacobi_svd(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, int kk,
                       double* theta, double* F, int64_t ldf, double* G, int64_t ldg, int* sweeps,
                       bool* converged, Scratch& ws, KProf* prof = nullptr);

}  // namespace tsvd
