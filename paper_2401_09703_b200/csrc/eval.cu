// eval.cu — F2: the downstream evaluation the paper's experiments score with,
// on the maintained approximation Ã = U Σ V^T (Def 2) in its extended form
// U = U'U'', V = V'V'' (Eq 4):
//   * entries of Ã at given (i, j) pairs — the link-prediction / collaborative-filtering score
//     U[i] Σ V[j]^T (AP and MSE are computed from these scores by the caller);
//   * the Frobenius residual ||A - Ã||_F against a sparse A, as
//     ||A||_F^2 - 2 <A, Ã> + ||Σ||^2 (U, V orthonormal), <A, Ã> = sum over A's nonzeros of
//     a_ij Ã_ij — Ã is never formed.
// The pairs are processed in chunks: gathered rows of U', V' (K2-style row gathers), one DMMA
// GEMM each with U''Σ and V'', and a warp-per-pair dot product.
#include <algorithm>
#include <vector>

#include "ops.h"

namespace tsvd {

namespace {
__global__ void gather_rows_kernel(const int64_t* __restrict__ idx, int64_t n, const double* __restrict__ X, int k,
                                   double* __restrict__ out) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / k;
    out[e] = X[idx[p] * k + e % k];
  }
}

// out[p] = a[p, :] . b[p, :]  (warp per pair)
__global__ void rowdot_kernel(int64_t n, int k, const double* __restrict__ a, const double* __restrict__ b,
                              double* __restrict__ out) {
  pdl_begin();
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= n) return;
  double s = 0.0;
  for (int c = lane; c < k; c += 32) s = fma(a[p * k + c], b[p * k + c], s);
  s = warp_sum(s);
  if (lane == 0) out[p] = s;
}

// M (k x k) <- M diag(S)
__global__ void scale_cols_rm_kernel(double* __restrict__ M, int k, const double* __restrict__ S) {
  pdl_begin();
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) M[e] *= S[e % k];
}

// row indices of a CSR's nonzeros
__global__ void csr_rowid_kernel(int64_t s, const int64_t* __restrict__ rp, int64_t* __restrict__ rows) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s) return;
  for (int64_t p = rp[w] + lane; p < rp[w + 1]; p += 32) rows[p] = w;
}

__global__ void widen_cols_kernel(int64_t n, const int32_t* __restrict__ ci, int64_t* __restrict__ cols) {
  pdl_begin();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    cols[p] = ci[p];
}

// acc[0] += sum a_p s_p, acc[1] += sum a_p^2  (deterministic: per-block partials, fixed order)
__global__ void dot_sq_partial_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ s,
                                      double* __restrict__ part) {
  pdl_begin();
  __shared__ double r0[8], r1[8];
  double x = 0.0, y = 0.0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    x = fma(a[p], s[p], x);
    y = fma(a[p], a[p], y);
  }
  x = warp_sum(x);
  y = warp_sum(y);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    r0[w] = x;
    r1[w] = y;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a0 = 0.0, a1 = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      a0 += r0[q];
      a1 += r1[q];
    }
    part[2 * blockIdx.x] = a0;
    part[2 * blockIdx.x + 1] = a1;
  }
}

inline unsigned gse(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16)); }
}  // namespace

// scores[p] = U[rows[p]] Σ V[cols[p]]^T for p < n, U = Xu Mu, V = Xv Mv (row-major k x k);
// rows / cols device int64 arrays; chunks of `chunk` pairs
cudaError_t score_pairs(cudaStream_t st, const double* Xu, const double* Mu, const double* Xv, const double* Mv,
                        const double* S, int k, int64_t n, const int64_t* rows, const int64_t* cols, double* out,
                        Scratch& ws) {
  if (n == 0) return cudaSuccess;
  const int64_t chunk = std::min<int64_t>(n, ((int64_t)32 << 20) / (8 * k));  // 32 MB gather blocks
  double* MuS = ws.alloc<double>((size_t)k * k);
  double* gu = ws.alloc<double>((size_t)chunk * k);
  double* gv = ws.alloc<double>((size_t)chunk * k);
  double* pu = ws.alloc<double>((size_t)chunk * k);
  double* pv = ws.alloc<double>((size_t)chunk * k);
  if (ws.err) return ws.err;
  cudaError_t e;
  if ((e = cudaMemcpyAsync(MuS, Mu, (size_t)k * k * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
  ++g_launches;
  launch_k(scale_cols_rm_kernel, cdiv((int64_t)k * k, 256), 256, 0, st, MuS, k, S);
  for (int64_t p0 = 0; p0 < n; p0 += chunk) {
    const int64_t c = std::min(chunk, n - p0);
    g_launches += 3;
    launch_k(gather_rows_kernel, gse(c * k), 256, 0, st, rows + p0, c, Xu, k, gu);
    launch_k(gather_rows_kernel, gse(c * k), 256, 0, st, cols + p0, c, Xv, k, gv);
    if ((e = dgemm_rm(st, false, false, c, k, k, 1.0, gu, k, MuS, k, 0.0, pu, k))) return e;
    if ((e = dgemm_rm(st, false, false, c, k, k, 1.0, gv, k, Mv, k, 0.0, pv, k))) return e;
    launch_k(rowdot_kernel, cdiv(c * 32, 256), 256, 0, st, c, k, pu, pv, out + p0);
  }
  return cudaGetLastError();
}

// <A, Ã> and ||A||_F^2 over the nonzeros of the m x n CSR A; h_out[0..1] (host, synchronises)
cudaError_t sparse_inner(cudaStream_t st, const double* Xu, const double* Mu, const double* Xv, const double* Mv,
                         const double* S, int k, const DevCSR& A, double* h_out, Scratch& ws) {
  h_out[0] = h_out[1] = 0.0;
  if (A.nnz == 0) return cudaSuccess;
  const int64_t chunk = std::min<int64_t>(A.nnz, (int64_t)1 << 22);
  int64_t* rows = ws.alloc<int64_t>(A.nnz);
  int64_t* cols = ws.alloc<int64_t>(A.nnz);
  double* sc = ws.alloc<double>(chunk);
  const int nb = 148 * 4;
  double* part = ws.alloc<double>((size_t)2 * nb);
  if (ws.err) return ws.err;
  g_launches += 2;
  launch_k(csr_rowid_kernel, cdiv(A.s * 32, 256), 256, 0, st, A.s, A.row_ptr, rows);
  launch_k(widen_cols_kernel, gse(A.nnz), 256, 0, st, A.nnz, A.col_idx, cols);
  std::vector<double> hp(2 * nb);
  double acc0 = 0.0, acc1 = 0.0;
  cudaError_t e;
  const Scratch::Mark mk = ws.mark();
  for (int64_t p0 = 0; p0 < A.nnz; p0 += chunk) {
    const int64_t c = std::min(chunk, A.nnz - p0);
    ws.rewind(mk);  // score_pairs' per-chunk workspaces
    if ((e = score_pairs(st, Xu, Mu, Xv, Mv, S, k, c, rows + p0, cols + p0, sc, ws))) return e;
    ++g_launches;
    launch_k(dot_sq_partial_kernel, nb, 256, 0, st, c, A.val + p0, sc, part);
    if ((e = cudaMemcpyAsync(hp.data(), part, 2 * nb * sizeof(double), cudaMemcpyDeviceToHost, st))) return e;
    if ((e = cudaStreamSynchronize(st))) return e;
    for (int b = 0; b < nb; ++b) {
      acc0 += hp[2 * b];
      acc1 += hp[2 * b + 1];
    }
  }
  h_out[0] = acc0;
  h_out[1] = acc1;
  return cudaSuccess;
}

__global__ void pairs_check_kernel(int64_t n, const int64_t* __restrict__ r, const int64_t* __restrict__ c, int64_t m,
                                   int64_t nn, int* __restrict__ flag) {
  pdl_begin();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    if (r[p] < 0 || r[p] >= m || c[p] < 0 || c[p] >= nn) *flag = 1;
}

cudaError_t pairs_in_range(cudaStream_t st, int64_t n, const int64_t* r, const int64_t* c, int64_t m, int64_t nn,
                           int* d_flag, bool* ok) {
  int h = 0;
  cudaError_t e;
  if ((e = cudaMemsetAsync(d_flag, 0, sizeof(int), st))) return e;
  if (n) {
    ++g_launches;
    launch_k(pairs_check_kernel, gse(n), 256, 0, st, n, r, c, m, nn, d_flag);
  }
  if ((e = cudaMemcpyAsync(&h, d_flag, sizeof(int), cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;
  *ok = h == 0;
  return cudaSuccess;
}

}  // namespace tsvd
