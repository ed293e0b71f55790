// init_svd.cu — F1: the initial truncated SVD on the GPU (the step before the
// path: "the SVD is initialised on the first 50% of the rows/columns", by the
// randomized numerical linear algebra the paper's introduction names).
//
// Randomized subspace iteration (range finder with q power steps) on a sparse A (m x n, CSR):
//   Y = A Ω  (Ω: n x p Gaussian, K12 side 3),  Y <- orth(Y)
//   q times:  Z = A^T Y, Z <- orth(Z);  Y = A Z, Y <- orth(Y)
//   A^T Y = Q_b R_b  (Cholesky-QR2);  R_b^T = U_r Σ V_r^T  (one-sided Jacobi, K7 / K9)
//   A ≈ Y Y^T A = Y R_b^T Q_b^T = (Y U_r) Σ (Q_b V_r)^T  ->  U = Y U_r[:, :k], V = Q_b V_r[:, :k]
// p = k + oversampling.  Every step runs in this library's kernels: the CSR and CSC gathers of
// K2 (A Ω, A Z, A^T Y — the CSC from K1, the columns A never touches are zero rows of Z and V),
// Cholesky-QR2 on DMMA, the core Jacobi, DMMA GEMMs.  For an A of rank <= p the result is
// A's exact truncated SVD (to rounding); otherwise the usual randomized-SVD approximation,
// sharpened by the power steps.  The factors then go through tsvd_init's validation.
#include <algorithm>

#include "ops.h"

namespace tsvd {

namespace {
__global__ void scatter_rows_kernel(const int32_t* __restrict__ J, int64_t nJ, const double* __restrict__ src, int k,
                                    double* __restrict__ dst) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nJ * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jj = e / k;
    dst[(int64_t)J[jj] * k + e % k] = src[e];
  }
}
inline unsigned gsi(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16)); }
}  // namespace

cudaError_t randomized_svd(cudaStream_t st, const DevCSR& A, int k, int p, int q, uint64_t seed, double* U, double* S,
                           double* V, Scratch& ws, int* sweeps, bool* converged) {
  const int64_t m = A.s, n = A.dim;
  cudaError_t e;
  // CSC of A over the columns it touches (K1) and the compact index maps
  DevCSC C;
  int64_t nJ = 0;
  if ((e = build_csc(st, A, C, ws, &nJ))) return e;
  if (nJ < p || m < p) return cudaErrorInvalidValue;
  GatherMaps gm;
  if ((e = gather_maps(st, A, C, gm, ws))) return e;
  DevCSR AT;  // A^T restricted to J, as a CSR with nJ rows (row jj = column J[jj] of A)
  AT.s = nJ;
  AT.dim = m;
  AT.nnz = A.nnz;
  AT.row_ptr = gm.rpJ;
  AT.col_idx = C.row;
  AT.val = C.val;
  DevCSR AJ = A;  // A with its column indices mapped to J positions (reads compact Z)
  AJ.col_idx = gm.ciJ;
  double* Y = ws.alloc<double>((size_t)m * p);
  double* Z = ws.alloc<double>((size_t)nJ * p);
  double* Om = ws.alloc<double>((size_t)nJ * p);
  double* Rb = ws.alloc<double>((size_t)p * p);
  double* th = ws.alloc<double>(p);
  double* Fr = ws.alloc<double>((size_t)p * k);
  double* Gr = ws.alloc<double>((size_t)p * k);
  double* VJ = ws.alloc<double>((size_t)nJ * k);
  if (ws.err) return ws.err;
  const double tau = 1e-14;
  // Ω on the touched columns only (an untouched column multiplies zeros)
  if ((e = counter_gaussian(st, seed, 3, nJ, p, Om))) return e;
  if ((e = gather_spmm_ld(st, AJ, Om, p, p, Y, p))) return e;        // Y = A Ω
  if ((e = cholqr_dense(st, Y, m, p, tau, 2, nullptr, ws))) return e;
  for (int it = 0; it < q; ++it) {
    if ((e = gather_spmm_ld(st, AT, Y, p, p, Z, p))) return e;       // Z = A^T Y (on J)
    if ((e = cholqr_dense(st, Z, nJ, p, tau, 2, nullptr, ws))) return e;
    if ((e = gather_spmm_ld(st, AJ, Z, p, p, Y, p))) return e;       // Y = A Z
    if ((e = cholqr_dense(st, Y, m, p, tau, 2, nullptr, ws))) return e;
  }
  if ((e = gather_spmm_ld(st, AT, Y, p, p, Z, p))) return e;         // A^T Y = Q_b R_b
  if ((e = cudaMemsetAsync(Rb, 0, (size_t)p * p * sizeof(double), st))) return e;
  if ((e = cholqr2_r(st, Z, nJ, p, tau, Rb, ws))) return e;
  // R_b^T: R_b row-major is R_b^T column-major (lda p); left vectors U_r, right V_r
  if ((e = jacobi_svd(st, Rb, p, p, p, k, th, Fr, p, Gr, p, sweeps, converged, ws, nullptr))) return e;
  if (!*converged) return cudaSuccess;
  // U = Y U_r[:, :k] (m x k row-major), V[J] = Q_b V_r[:, :k], V elsewhere 0
  if ((e = dgemm(st, m, k, p, 1.0, CMat{Y, p, 1}, CMat{Fr, 1, p}, 0.0, Mat{U, k, 1}, 0))) return e;
  if ((e = dgemm(st, nJ, k, p, 1.0, CMat{Z, p, 1}, CMat{Gr, 1, p}, 0.0, Mat{VJ, k, 1}, 0))) return e;
  if ((e = cudaMemsetAsync(V, 0, (size_t)n * k * sizeof(double), st))) return e;
  ++g_launches;
  launch_k(scatter_rows_kernel, gsi(nJ * k), 256, 0, st, C.J, nJ, VJ, k, V);
  return cudaMemcpyAsync(S, th, k * sizeof(double), cudaMemcpyDeviceToDevice, st);
}

}  // namespace tsvd
