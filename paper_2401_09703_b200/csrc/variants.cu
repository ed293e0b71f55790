// variants.cu — the approximate augmented space of App D on the GPU.
//
//   RPI  (Alg 8; dense Alg 7): t power iterations on the
//        SV-LCOV tuples  Q = B' - X C'  with  B' = E P (held on the support J),
//        C' = C0 P,  Alg 2 (as Cholesky-QR2 with deflation) on the tuples, and
//        P <- E^T B' - C0^T C'.  P is orthonormalised at the top of each iteration
//        (Alg 7 line 4, R14).
//   GKL  (Alg 6): l Lanczos steps on the tuples with full
//        reorthogonalisation of p, H read as l x (l+1) (R11), P = P_{l+1} H^T.
//   K12  counter-based Gaussian start block (R13 / §2.1).
// Both produce (B'_J, C', P) with Q^T Z = P^T; the core and the updates of App D.3
// then run as in the exact path with B' in place of E R^{-1}.
#include <algorithm>
#include <cmath>

#include "ops.h"

namespace tsvd {

namespace {

// ---------------------------------------------------------------- B'_J = E P on the support
// warp per touched column; lanes stride the w output columns (2 at a time when w even)
__global__ void __launch_bounds__(256) csc_spmm_kernel(int64_t nJ, const int32_t* __restrict__ J,
                                                       const int64_t* __restrict__ colptr,
                                                       const int32_t* __restrict__ crow,
                                                       const double* __restrict__ cval, const double* __restrict__ P,
                                                       int w, double* __restrict__ BJ) {
  pdl_begin();
  const int64_t jj = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (jj >= nJ) return;
  const int lane = threadIdx.x & 31;
  const int j = J[jj];
  const int64_t b = colptr[j], e = colptr[j + 1];
  for (int c0 = 0; c0 < w; c0 += 64) {
    const int c = c0 + 2 * lane;
    double a0 = 0.0, a1 = 0.0;
    for (int64_t q = b; q < e; ++q) {
      const double v = cval[q];
      const double* pr = P + (int64_t)crow[q] * w;
      if (c < w) a0 = fma(v, pr[c], a0);
      if (c + 1 < w) a1 = fma(v, pr[c + 1], a1);
    }
    if (c < w) BJ[jj * w + c] = a0;
    if (c + 1 < w) BJ[jj * w + c + 1] = a1;
  }
}

// out[i, :] = sum_p v_p BJ[jpos[col_p], :]; warp per update vector
__global__ void __launch_bounds__(256) csr_gather_compact_kernel(int64_t s, const int64_t* __restrict__ rp,
                                                                 const int32_t* __restrict__ ci,
                                                                 const double* __restrict__ v,
                                                                 const int64_t* __restrict__ jpos,
                                                                 const double* __restrict__ BJ, int w,
                                                                 double* __restrict__ out) {
  pdl_begin();
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= s) return;
  const int lane = threadIdx.x & 31;
  const int64_t b = rp[i], e = rp[i + 1];
  for (int c0 = 0; c0 < w; c0 += 64) {
    const int c = c0 + 2 * lane;
    double a0 = 0.0, a1 = 0.0;
    for (int64_t p = b; p < e; ++p) {
      const double x = v[p];
      const double* br = BJ + jpos[ci[p]] * w;
      if (c < w) a0 = fma(x, br[c], a0);
      if (c + 1 < w) a1 = fma(x, br[c + 1], a1);
    }
    if (c < w) out[i * w + c] = a0;
    if (c + 1 < w) out[i * w + c + 1] = a1;
  }
}

// ---------------------------------------------------------------- X <- X R^{-1} (diagonal block)
constexpr int TB = 32;
// one thread per row of X: forward substitution over the nb x nb diagonal block at (p, p)
__global__ void __launch_bounds__(128) trsm_right_diag_kernel(const double* __restrict__ R, int64_t l, int64_t p,
                                                              int nb, const int32_t* __restrict__ keep, double* X,
                                                              int64_t rows) {
  pdl_begin();
  __shared__ double Rs[TB][TB + 1];
  __shared__ int kp[TB];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    Rs[i][j] = (j >= i) ? R[(p + i) * l + p + j] : 0.0;
  }
  for (int i = threadIdx.x; i < nb; i += blockDim.x) kp[i] = keep[p + i];
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double* x = X + r * l + p;
  double y[TB];
#pragma unroll
  for (int j = 0; j < TB; ++j) {
    if (j < nb) {
      double g = x[j];
#pragma unroll
      for (int i = 0; i < j; ++i) g -= y[i] * Rs[i][j];
      y[j] = kp[j] ? g / Rs[j][j] : 0.0;
      x[j] = y[j];
    }
  }
}

__global__ void index_add_rows_kernel(const int32_t* __restrict__ J, int64_t nJ, const double* __restrict__ Z, int k,
                                      double* __restrict__ X) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nJ * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jj = e / k;
    const int c = (int)(e % k);
    X[(int64_t)J[jj] * k + c] += Z[e];
  }
}

// ---------------------------------------------------------------- K12 counter-based Gaussian
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// rows on a grid-stride loop, columns on the threads (no 64-bit division per element);
// cos(2 pi u2) as cospi(2 u2) (no argument reduction; within an ulp of the spec's cos(2 pi u2))
__global__ void counter_gaussian_kernel(uint64_t seed, int side, int64_t s, int64_t l, double* __restrict__ O) {
  pdl_begin();
  const int64_t tpr = (l + 31) / 32 * 32 < blockDim.x ? (l + 31) / 32 * 32 : blockDim.x;  // threads per row
  const int64_t rpb = blockDim.x / tpr;                                                   // rows per block
  const int64_t jt = threadIdx.x % tpr, r0 = threadIdx.x / tpr;
  if (r0 >= rpb) return;
  for (int64_t i = (int64_t)blockIdx.x * rpb + r0; i < s; i += (int64_t)gridDim.x * rpb) {
    for (int64_t j = jt; j < l; j += tpr) {
      const uint64_t c = ((uint64_t)side << 60) | ((uint64_t)i << 20) | (uint64_t)j;
      const uint64_t z1 = splitmix64(seed ^ (2 * c)), z2 = splitmix64(seed ^ (2 * c + 1));
      const double u1 = ((double)(z1 >> 11) + 0.5) * 0x1.0p-53;
      const double u2 = (double)(z2 >> 11) * 0x1.0p-53;
      O[i * l + j] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
  }
}

// ---------------------------------------------------------------- cores
__global__ void core_approx_kernel(int k, int64_t s, int64_t l, const double* __restrict__ Sigma,
                                   const double* __restrict__ P0, const double* __restrict__ P, double* __restrict__ K) {
  pdl_begin();
  const int64_t mr = k + s;
  const int64_t n = (int64_t)(k + l) * mr;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / mr, i = e % mr;
    double v;
    if (i < k)
      v = (j == i) ? Sigma[i] : 0.0;
    else if (j < k)
      v = P0[(i - k) * k + j];
    else
      v = P[(i - k) * l + (j - k)];
    K[e] = v;
  }
}

__global__ void lift_block_approx_kernel(int k, int64_t s, int64_t l, const double* __restrict__ P0,
                                         const double* __restrict__ P, double* __restrict__ L) {
  pdl_begin();
  const int64_t n = (int64_t)(k + l) * s;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / s, c = e % s;
    L[e] = (i < k) ? P0[c * k + i] : P[c * l + (i - k)];
  }
}

// ---------------------------------------------------------------- GKL step kernels
// b'_i[jj] = sum_q val_q p[row_q] - beta_prev * bprev[jj]   (Alg 6 line 4 on the support)
__global__ void gkl_b_kernel(int64_t nJ, const int32_t* __restrict__ J, const int64_t* __restrict__ colptr,
                             const int32_t* __restrict__ crow, const double* __restrict__ cval,
                             const double* __restrict__ p, const double* __restrict__ beta_prev,
                             const double* __restrict__ bprev, double* __restrict__ b) {
  pdl_begin();
  const int64_t jj = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (jj >= nJ) return;
  const int lane = threadIdx.x & 31;
  const int j = J[jj];
  double a = 0.0;
  for (int64_t q = colptr[j] + lane; q < colptr[j + 1]; q += 32) a = fma(cval[q], p[crow[q]], a);
  a = warp_sum(a);
  if (lane == 0) b[jj] = bprev ? a - (*beta_prev) * bprev[jj] : a;
}

// c'_i[a] = sum_r P0[r, a] p[r] - beta_prev * cprev[a]   (Alg 6 line 5); block per a
__global__ void __launch_bounds__(256) gkl_c_kernel(int64_t s, int k, const double* __restrict__ P0,
                                                    const double* __restrict__ p, const double* __restrict__ beta_prev,
                                                    const double* __restrict__ cprev, double* __restrict__ c) {
  pdl_begin();
  __shared__ double red[8];
  const int a = blockIdx.x;
  double acc = 0.0;
  for (int64_t r = threadIdx.x; r < s; r += blockDim.x) acc = fma(P0[r * k + a], p[r], acc);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    c[a] = cprev ? t - (*beta_prev) * cprev[a] : t;
  }
}

// alpha = sqrt(<b,b> - <c,c>) with deflation (R8/R9), then b, c /= alpha (Alg 6 lines 6-8)
__global__ void __launch_bounds__(1024) gkl_alpha_kernel(int64_t nJ, int k, double* __restrict__ b,
                                                         double* __restrict__ c, double tau,
                                                         double* __restrict__ alpha) {
  pdl_begin();
  __shared__ double r1[32], r2[32];
  __shared__ double sa;
  double bb = 0.0, cc = 0.0;
  for (int64_t i = threadIdx.x; i < nJ; i += blockDim.x) bb = fma(b[i], b[i], bb);
  for (int i = threadIdx.x; i < k; i += blockDim.x) cc = fma(c[i], c[i], cc);
  bb = warp_sum(bb);
  cc = warp_sum(cc);
  if ((threadIdx.x & 31) == 0) { r1[threadIdx.x >> 5] = bb; r2[threadIdx.x >> 5] = cc; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double B = 0.0, Cc = 0.0;
    for (int w = 0; w < 32; ++w) { B += r1[w]; Cc += r2[w]; }
    const double a2 = B - Cc;
    const double a = (B == 0.0 || a2 <= tau * B) ? 0.0 : sqrt(a2);
    *alpha = a;
    sa = a;
  }
  __syncthreads();
  const double inv = sa > 0.0 ? 1.0 / sa : 0.0;
  for (int64_t i = threadIdx.x; i < nJ; i += blockDim.x) b[i] *= inv;
  for (int i = threadIdx.x; i < k; i += blockDim.x) c[i] *= inv;
}

// p_next[i] = sum_p v_p b[jpos[col_p]] - sum_a P0[i, a] c[a] - alpha p[i]   (Alg 6 line 9)
__global__ void gkl_p_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                             const double* __restrict__ v, const int64_t* __restrict__ jpos,
                             const double* __restrict__ b, int k, const double* __restrict__ P0,
                             const double* __restrict__ c, const double* __restrict__ alpha,
                             const double* __restrict__ p, double* __restrict__ pn) {
  pdl_begin();
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= s) return;
  const int lane = threadIdx.x & 31;
  double a = 0.0;
  for (int64_t q = rp[i] + lane; q < rp[i + 1]; q += 32) a = fma(v[q], b[jpos[ci[q]]], a);
  for (int x = lane; x < k; x += 32) a = fma(-P0[i * k + x], c[x], a);
  a = warp_sum(a);
  if (lane == 0) pn[i] = a - (*alpha) * p[i];
}

// h[j] = <Pm[:, j], x> for j < nc (Pm col-major, ld s); block per j
__global__ void __launch_bounds__(256) multi_dot_kernel(int64_t s, const double* __restrict__ Pm,
                                                        const double* __restrict__ x, double* __restrict__ h) {
  pdl_begin();
  __shared__ double red[8];
  const int j = blockIdx.x;
  double acc = 0.0;
  for (int64_t r = threadIdx.x; r < s; r += blockDim.x) acc = fma(Pm[(int64_t)j * s + r], x[r], acc);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    h[j] = t;
  }
}

// x[r] -= sum_j Pm[r, j] h[j]
__global__ void sub_comb_kernel(int64_t s, int nc, const double* __restrict__ Pm, const double* __restrict__ h,
                                double* __restrict__ x) {
  pdl_begin();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= s) return;
  double a = x[r];
  for (int j = 0; j < nc; ++j) a = fma(-Pm[(int64_t)j * s + r], h[j], a);
  x[r] = a;
}

// beta = ||x||; x /= beta (Alg 6 lines 11-12).  Breakdown: beta = 0 and x = 0 when
// ||x||^2 <= rel2 * ref2 (ref2: squared norm before the reorthogonalisation).
__global__ void __launch_bounds__(1024) norm_scale_kernel(int64_t s, double* __restrict__ x, double* __restrict__ beta,
                                                          const double* __restrict__ ref2, double rel2) {
  pdl_begin();
  __shared__ double red[32];
  __shared__ double sb;
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < s; i += blockDim.x) a = fma(x[i], x[i], a);
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += red[w];
    double nb = sqrt(t);
    if (ref2 && !(t > rel2 * (*ref2))) nb = 0.0;
    sb = nb;
    if (beta) *beta = nb;
  }
  __syncthreads();
  const double inv = sb > 0.0 ? 1.0 / sb : 0.0;
  for (int64_t i = threadIdx.x; i < s; i += blockDim.x) x[i] *= inv;
}

// P[:, i] = alpha_i p_i + beta_i p_{i+1}  (P = P_{l+1} H^T, H l x (l+1)); output row-major s x l
__global__ void gkl_combine_kernel(int64_t s, int l, const double* __restrict__ Pm, const double* __restrict__ alpha,
                                   const double* __restrict__ beta, double* __restrict__ P) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < s * l; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / l;
    const int i = (int)(e % l);
    P[e] = alpha[i] * Pm[(int64_t)i * s + r] + beta[i] * Pm[(int64_t)(i + 1) * s + r];
  }
}

__global__ void transpose_cm_to_rm(const double* __restrict__ A, int64_t rows, int64_t cols, double* __restrict__ O) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    O[e] = A[j * rows + i];
  }
}

inline unsigned gs(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16)); }

}  // namespace

namespace {
bool gather_width(int w) { return w == 16 || w == 32 || w == 64 || w == 128 || w == 256; }

// compact row pointer of the CSC over J: rp[jj] = colptr[J[jj]] (untouched columns are empty)
__global__ void csc_rowptr_kernel(int64_t nJ, const int32_t* __restrict__ J, const int64_t* __restrict__ colptr,
                                  int64_t nnz, int64_t* __restrict__ rp) {
  pdl_begin();
  const int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (jj < nJ) rp[jj] = colptr[J[jj]];
  if (jj == nJ) rp[nJ] = nnz;
}
// column indices of E mapped to their compact position in J
__global__ void map_cols_kernel(int64_t nnz, const int32_t* __restrict__ ci, const int64_t* __restrict__ jpos,
                                int32_t* __restrict__ out) {
  pdl_begin();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
    out[p] = (int32_t)jpos[ci[p]];
}
}  // namespace

cudaError_t gather_maps(cudaStream_t st, const DevCSR& E, const DevCSC& C, GatherMaps& out, Scratch& ws) {
  out.rpJ = ws.alloc<int64_t>(C.nJ + 1);
  out.ciJ = ws.alloc<int32_t>(std::max<int64_t>(E.nnz, 1));
  if (ws.err) return ws.err;
  g_launches += 2;
  launch_k(csc_rowptr_kernel, cdiv(C.nJ + 1, 256), 256, 0, st, C.nJ, C.J, C.colptr, E.nnz, out.rpJ);
  if (E.nnz) launch_k(map_cols_kernel, gs(E.nnz), 256, 0, st, E.nnz, E.col_idx, C.jpos, out.ciJ);
  return cudaGetLastError();
}

// B'_J = E P on the support: the CSC over J read as a CSR with nJ rows (K2's gather-SpMM with
// its hub-row handling: a hub column of E — a high-degree vertex, thousands of entries — gets
// a CTA instead of serialising one warp)
cudaError_t csc_spmm(cudaStream_t st, const DevCSC& C, const GatherMaps* gm, int64_t nnz, const double* P, int w,
                     double* BJ) {
  if (C.nJ == 0) return cudaSuccess;
  KScope sc(KC_APPROX, 2.0 * nnz * w, 12.0 * nnz + 8.0 * (double)C.nJ * w);
  if (gm && gather_width(w)) {
    DevCSR T;
    T.s = C.nJ;
    T.nnz = nnz;
    T.row_ptr = gm->rpJ;
    T.col_idx = C.row;
    T.val = C.val;
    return gather_spmm(st, T, P, w, BJ);
  }
  ++g_launches;
  launch_k(csc_spmm_kernel, cdiv(C.nJ * 32, 256), 256, 0, st, C.nJ, C.J, C.colptr, C.row, C.val, P, w, BJ);
  return cudaGetLastError();
}

cudaError_t csr_gather_compact(cudaStream_t st, const DevCSR& E, const int64_t* jpos, const GatherMaps* gm,
                               const double* BJ, int w, double* out) {
  if (E.s == 0) return cudaSuccess;
  KScope sc(KC_APPROX, 2.0 * E.nnz * w, 12.0 * E.nnz + 8.0 * (double)E.s * w);
  if (gm && gather_width(w)) {
    DevCSR T = E;
    T.col_idx = gm->ciJ;
    return gather_spmm(st, T, BJ, w, out);
  }
  ++g_launches;
  launch_k(csr_gather_compact_kernel, cdiv(E.s * 32, 256), 256, 0, st, E.s, E.row_ptr, E.col_idx, E.val, jpos, BJ, w, out);
  return cudaGetLastError();
}

cudaError_t trsm_right_upper(cudaStream_t st, const double* R, int64_t l, const int32_t* keep, double* X,
                             int64_t rows) {
  if (rows == 0 || l == 0) return cudaSuccess;
  for (int64_t p = 0; p < l; p += TB) {
    const int nb = (int)std::min<int64_t>(TB, l - p);
    ++g_launches;
    launch_k(trsm_right_diag_kernel, cdiv(rows, 128), 128, 0, st, R, l, p, nb, keep, X, rows);
    const int64_t rest = l - p - nb;
    if (rest > 0) {
      // X[:, p+nb:] -= X[:, p:p+nb] R[p:p+nb, p+nb:]
      cudaError_t e = dgemm_rm(st, false, false, rows, rest, nb, -1.0, X + p, l, R + p * l + p + nb, l, 1.0,
                               X + p + nb, l);
      if (e) return e;
    }
  }
  return cudaGetLastError();
}

cudaError_t index_add_rows(cudaStream_t st, const int32_t* J, int64_t nJ, const double* Z, int k, double* X) {
  if (nJ == 0) return cudaSuccess;
  ++g_launches;
  launch_k(index_add_rows_kernel, gs(nJ * k), 256, 0, st, J, nJ, Z, k, X);
  return cudaGetLastError();
}

cudaError_t counter_gaussian(cudaStream_t st, uint64_t seed, int side, int64_t s, int64_t l, double* Omega) {
  if (s * l == 0) return cudaSuccess;
  ++g_launches;
  launch_k(counter_gaussian_kernel, gs(s * l), 256, 0, st, seed, side, s, l, Omega);
  return cudaGetLastError();
}

cudaError_t build_core_approx(cudaStream_t st, int k, int64_t s, int64_t l, const double* Sigma, const double* P0,
                              const double* P, double* K) {
  ++g_launches;
  launch_k(core_approx_kernel, gs((int64_t)(k + l) * (k + s)), 256, 0, st, k, s, l, Sigma, P0, P, K);
  return cudaGetLastError();
}

cudaError_t build_lift_block_approx(cudaStream_t st, int k, int64_t s, int64_t l, const double* P0, const double* P,
                                    double* L) {
  if (s == 0) return cudaSuccess;
  ++g_launches;
  launch_k(lift_block_approx_kernel, gs((int64_t)(k + l) * s), 256, 0, st, k, s, l, P0, P, L);
  return cudaGetLastError();
}

// X <- X T with T = R^{-1} over the kept pivots (deflated columns of X become 0): T is
// obtained by the same right-side triangular solve applied to the l x l identity, then one
// DMMA GEMM applies it to all rows (instead of latency-bound row-wise substitutions).
cudaError_t apply_rinv(cudaStream_t st, const double* R, int64_t l, const int32_t* keep, double* X, int64_t rows,
                       Scratch& ws) {
  if (rows == 0) return cudaSuccess;
  if (rows <= 2 * l) return trsm_right_upper(st, R, l, keep, X, rows);
  double* T = ws.alloc<double>((size_t)l * l);
  double* tmp = ws.alloc<double>((size_t)rows * l);
  if (ws.err) return ws.err;
  cudaError_t e;
  if ((e = set_identity(st, T, (int)l))) return e;
  if ((e = trsm_right_upper(st, R, l, keep, T, l))) return e;
  if ((e = dgemm_rm(st, false, false, rows, l, l, 1.0, X, l, T, l, 0.0, tmp, l))) return e;
  return cudaMemcpyAsync(X, tmp, (size_t)rows * l * sizeof(double), cudaMemcpyDeviceToDevice, st);
}

namespace {
__global__ void zero_lower_kernel(double* G, int64_t l) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < l * l; e += (int64_t)gridDim.x * blockDim.x)
    if (e / l > e % l) G[e] = 0.0;
}
}  // namespace

// T = R^+ from the tile-DAG Cholesky's factor R (l x l row-major, upper) and its diagonal-tile
// inverses (Tb: tile q holds Y_q = R_qq^{+T}, row-major 64 x 64) by block back substitution
//   T_jj = Y_j^T,   T_ij = -T_ii sum_{i<k<=j} R_ik T_kj   (i = j-1 .. 0)
// One CTA per (block column j, 16-column quarter); the column panel of T in shared memory.
// (The DAG back substitution R T = I it replaces is built for s x k right-hand sides with
// s in the thousands: 133 us at l = 256 against ~10 us here.)
__global__ void __launch_bounds__(256) tri_inv_tb_kernel(const double* __restrict__ R, int64_t l, int nt,
                                                          const double* __restrict__ Tb, double* __restrict__ T) {
  pdl_begin();
  extern __shared__ double sh_ti[];
  double* Tp = sh_ti;              // nt*64 x 16 panel of T (block rows 0..j)
  double* Sacc = Tp + nt * 64 * 16;  // 64 x 16
  const int j = blockIdx.x, q = blockIdx.y, tid = threadIdx.x;
  const int r = tid >> 2, cq = (tid & 3) * 4;
  const int64_t jend = min((int64_t)(j + 1) * 64, l);
  const int64_t c0 = (int64_t)j * 64 + q * 16;
  for (int i = j; i >= 0; --i) {
    const int64_t row = (int64_t)i * 64 + r;
    double val[4];
    if (i == j) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t cl = q * 16 + cq + u;  // local column in tile j
        // (T_jj = Y_j^T is upper triangular: entries below its diagonal are exact zeros)
        val[u] = (row < l && c0 + cq + u < jend && r <= cl) ? Tb[(int64_t)j * 4096 + cl * 64 + r] : 0.0;
      }
    } else {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      if (row < l) {
        const double* rr = R + row * l;
        for (int64_t kk = (int64_t)(i + 1) * 64; kk < jend; ++kk) {
          const double a = rr[kk];
          const double* tp = Tp + kk * 16 + cq;
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[u] = fma(a, tp[u], acc[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) Sacc[r * 16 + cq + u] = acc[u];
      __syncthreads();
      const int nbi = (int)min((int64_t)64, l - (int64_t)i * 64);
#pragma unroll
      for (int u = 0; u < 4; ++u) val[u] = 0.0;
      if (row < l) {
        const double* y = Tb + (int64_t)i * 4096;
        for (int a = 0; a < nbi; ++a) {
          const double ya = y[a * 64 + r];   // T_ii[r][a] = Y_i[a][r]
#pragma unroll
          for (int u = 0; u < 4; ++u) val[u] = fma(-ya, Sacc[a * 16 + cq + u], val[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) Tp[(i * 64 + r) * 16 + cq + u] = val[u];
    __syncthreads();
  }
  // write the panel: block rows <= j from Tp, zeros below
  for (int e = tid; e < (int)(l - (int64_t)0) * 16 && e < nt * 64 * 16; e += 256) {
    const int64_t rr = e / 16;
    const int cc = e % 16;
    if (rr >= l || c0 + cc >= jend) continue;
    T[rr * l + c0 + cc] = (rr < (int64_t)(j + 1) * 64) ? Tp[rr * 16 + cc] : 0.0;
  }
}

// Cholesky with deflation of the l x l Gram G (upper part; reading R8: pivot i deflated when its
// Schur diagonal <= tau en[i], en = null: G's diagonal) into R (in G) and T = R^+ (l x l
// row-major: the inverse on the kept pivots, zero rows / columns at deflated ones).  l <= 128:
// one CTA (chol_inv_small); larger l: the tile-DAG Cholesky (which leaves the diagonal-tile
// inverses in Tb) and the tile-DAG back substitution R T = I — two persistent launches instead
// of ~2 l / 32 row-block solves.  zero_lower: R returned with a zero strict lower triangle.
cudaError_t chol_rinv(cudaStream_t st, double* G, int64_t l, const double* en, double tau, int32_t* keep, double* T,
                      Scratch& ws, bool zero_lower) {
  cudaError_t e;
  if (l <= 128) return chol_inv_small(st, G, (int)l, en, tau, keep, T);
  double* Tb = ws.alloc<double>((size_t)((l + 63) / 64) * 64 * 64);
  double* enl = en ? nullptr : ws.alloc<double>(l);
  if (ws.err) return ws.err;
  if (!en) {
    if ((e = copy_diag(st, G, l, enl))) return e;
    en = enl;
  }
  if ((l & 1) == 0) {  // the tile DAG's 16-byte row paths need an even leading dimension
    if ((e = chol_deflate(st, G, l, en, tau, keep, Tb))) return e;
    const int nt = (int)((l + 63) / 64);
    const size_t smem = ((size_t)nt * 64 * 16 + 64 * 16) * sizeof(double);
    if (smem > 48 * 1024) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(tri_inv_tb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
      }
    }
    ++g_launches;
    {
      KScope sc(KC_PANEL, (double)l * l * l / 3.0, 8.0 * 2.0 * l * l);
      launch_k(tri_inv_tb_kernel, dim3(nt, 4), 256, smem, st, G, l, nt, Tb, T);
    }
    if (zero_lower) {
      ++g_launches;
      launch_k(zero_lower_kernel, gs(l * l), 256, 0, st, G, l);
    }
    return cudaGetLastError();
  }
  if ((e = chol_deflate(st, G, l, en, tau, keep))) return e;
  if ((e = set_identity(st, T, (int)l))) return e;
  return trsm_right_upper(st, G, l, keep, T, l);
}

namespace {
double* other_buf_chunk(Scratch& ws, int64_t count) { return ws.alloc<double>((size_t)count); }
}  // namespace

// passes of Cholesky-QR with deflation on a dense block X (rows x l row-major): per pass the
// Gram (upper triangle), R and T = R^+ (chol_rinv), and one GEMM X T into the other buffer of a
// ping-pong pair.  The result lands in Xout if given (X is then scratch), else in X.
// R (optional, l x l upper row-major) accumulates the product of the passes' factors.
cudaError_t cholqr_dense(cudaStream_t st, double* X, int64_t rows, int64_t l, double tau, int passes, double* R,
                         Scratch& ws, double* Xout) {
  double* G = ws.alloc<double>((size_t)l * l);
  double* Racc = R ? ws.alloc<double>((size_t)l * l) : nullptr;
  int32_t* keep = ws.alloc<int32_t>(l);
  double* T = ws.alloc<double>((size_t)l * l);
  if (ws.err) return ws.err;
  cudaError_t e;
  // buffers: the passes alternate between two blocks; the last one writes the destination
  double* dest = Xout ? Xout : X;
  double* other = nullptr;
  auto other_buf = [&]() -> double* {
    if (!other) other = ws.alloc<double>((size_t)std::max<int64_t>(rows, 1) * l);
    return other;
  };
  double* cur = X;
  // blocks beyond 2 GB (the F1 range finder on configs[4]: 18M x 272) are updated in place by
  // row chunks through a 512 MB buffer instead of a second full-size block
  const bool chunked = !Xout && (double)rows * l * 8.0 > 2.0 * (1ull << 30);
  const int64_t crow = chunked ? std::max<int64_t>(1, ((int64_t)64 << 20) / l) : rows;
  for (int pass = 0; pass < passes; ++pass) {
    if ((e = dgemm_rm(st, true, false, l, l, rows, 1.0, cur, l, cur, l, 0.0, G, l, 1))) return e;
    if ((e = chol_rinv(st, G, l, nullptr, tau, keep, T, ws, R != nullptr))) return e;
    if (chunked) {
      double* tmp = other_buf_chunk(ws, crow * l);
      if (!tmp) return ws.err ? ws.err : cudaErrorMemoryAllocation;
      for (int64_t r0 = 0; r0 < rows; r0 += crow) {
        const int64_t nr = std::min(crow, rows - r0);
        if ((e = dgemm_rm_btri(st, nr, l, l, X + r0 * l, l, T, l, tmp, l))) return e;
        if ((e = cudaMemcpyAsync(X + r0 * l, tmp, (size_t)nr * l * sizeof(double), cudaMemcpyDeviceToDevice, st)))
          return e;
      }
      if (R) {
        if (pass == 0) {
          if ((e = cudaMemcpyAsync(R, G, (size_t)l * l * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
        } else {
          if ((e = cudaMemcpyAsync(Racc, R, (size_t)l * l * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
          if ((e = dgemm_rm(st, false, false, l, l, l, 1.0, G, l, Racc, l, 0.0, R, l))) return e;
        }
      }
      continue;
    }
    double* dst;
    if (pass + 1 < passes) dst = (cur == X) ? other_buf() : X;
    else dst = (cur != dest) ? dest : ((cur == X) ? other_buf() : X);
    if (!dst) return ws.err ? ws.err : cudaErrorMemoryAllocation;
    if ((e = dgemm_rm_btri(st, rows, l, l, cur, l, T, l, dst, l))) return e;   // T upper triangular
    cur = dst;
    if (R) {
      if (pass == 0) {
        if ((e = cudaMemcpyAsync(R, G, (size_t)l * l * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
      } else {
        if ((e = cudaMemcpyAsync(Racc, R, (size_t)l * l * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
        if ((e = dgemm_rm(st, false, false, l, l, l, 1.0, G, l, Racc, l, 0.0, R, l))) return e;
      }
    }
  }
  if (cur != dest)
    if ((e = cudaMemcpyAsync(dest, cur, (size_t)rows * l * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
  return cudaSuccess;
}

cudaError_t cholqr2_dense(cudaStream_t st, double* X, int64_t rows, int64_t l, double tau, Scratch& ws) {
  return cholqr_dense(st, X, rows, l, tau, 2, nullptr, ws);
}

cudaError_t cholqr2_r(cudaStream_t st, double* X, int64_t rows, int64_t l, double tau, double* R, Scratch& ws) {
  return cholqr_dense(st, X, rows, l, tau, 2, R, ws);
}

cudaError_t cholqr2_tuple(cudaStream_t st, double* BJ, int64_t nJ, double* Cp, int k, int64_t l, double tau,
                          Scratch& ws) {
  double* G = ws.alloc<double>((size_t)l * l);
  double* en = ws.alloc<double>(l);
  int32_t* keep = ws.alloc<int32_t>(l);
  if (ws.err) return ws.err;
  cudaError_t e;
  for (int pass = 0; pass < 2; ++pass) {
    // Lemma 2 Gram of the tuples: B'^T B' - C'^T C'; deflation reference ||b'_i||^2
    if ((e = dgemm_rm(st, true, false, l, l, nJ, 1.0, BJ, l, BJ, l, 0.0, G, l, 1))) return e;
    if ((e = copy_diag(st, G, l, en))) return e;
    if ((e = dgemm_rm(st, true, false, l, l, k, -1.0, Cp, l, Cp, l, 1.0, G, l, 1))) return e;
    if ((e = chol_deflate(st, G, l, en, tau, keep))) return e;
    if ((e = apply_rinv(st, G, l, keep, BJ, nJ, ws))) return e;
    if ((e = apply_rinv(st, G, l, keep, Cp, k, ws))) return e;
  }
  return cudaSuccess;
}

cudaError_t gkl_basis(cudaStream_t st, const DevCSR& E, const DevCSC& C, const double* P0, int k, const double* p1,
                      int l, double tau, double* BJ, double* Cp, double* P, Scratch& ws) {
  const int64_t s = E.s, nJ = C.nJ;
  double* Pm = ws.alloc<double>((size_t)s * (l + 1));  // col-major p_1 .. p_{l+1}
  double* Bc = ws.alloc<double>((size_t)std::max<int64_t>(nJ, 1) * l);   // col-major b'_i
  double* Cc = ws.alloc<double>((size_t)k * l);          // col-major c'_i
  double* alpha = ws.alloc<double>(l);
  double* beta = ws.alloc<double>(l + 1);
  double* h = ws.alloc<double>(l + 1);
  double* pnorm = ws.alloc<double>(1);
  if (ws.err) return ws.err;
  cudaError_t e;
  if ((e = cudaMemcpyAsync(Pm, p1, s * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
  g_launches += 1;
  launch_k(norm_scale_kernel, 1, 1024, 0, st, s, Pm, nullptr, nullptr, 0.0);   // ||p_1|| = 1 (Alg 6 line 2)
  for (int i = 0; i < l; ++i) {
    double* p = Pm + (int64_t)i * s;
    double* pn = Pm + (int64_t)(i + 1) * s;
    double* b = Bc + (int64_t)i * nJ;
    double* c = Cc + (int64_t)i * k;
    const double* bprev = i ? Bc + (int64_t)(i - 1) * nJ : nullptr;
    const double* cprev = i ? Cc + (int64_t)(i - 1) * k : nullptr;
    const double* bp = i ? beta + (i - 1) : nullptr;
    g_launches += 4;
    if (nJ) launch_k(gkl_b_kernel, cdiv(nJ * 32, 256), 256, 0, st, nJ, C.J, C.colptr, C.row, C.val, p, bp, bprev, b);
    launch_k(gkl_c_kernel, k, 256, 0, st, s, k, P0, p, bp, cprev, c);
    launch_k(gkl_alpha_kernel, 1, 1024, 0, st, nJ, k, b, c, tau, alpha + i);
    launch_k(gkl_p_kernel, cdiv(s * 32, 256), 256, 0, st, s, E.row_ptr, E.col_idx, E.val, C.jpos, b, k, P0, c, alpha + i,
                                                     p, pn);
    // reference norm for the breakdown test: ||p_next|| before orthogonalisation
    g_launches += 1 + 2 * 2 + 1;
    launch_k(multi_dot_kernel, 1, 256, 0, st, s, pn, pn, pnorm);
    for (int pass = 0; pass < 2; ++pass) {  // Alg 6 line 10, classical Gram-Schmidt twice
      launch_k(multi_dot_kernel, i + 1, 256, 0, st, s, Pm, pn, h);
      launch_k(sub_comb_kernel, cdiv(s, 256), 256, 0, st, s, i + 1, Pm, h, pn);
    }
    launch_k(norm_scale_kernel, 1, 1024, 0, st, s, pn, beta + i, pnorm, 1e-28);
  }
  g_launches += 3;
  launch_k(gkl_combine_kernel, gs(s * l), 256, 0, st, s, l, Pm, alpha, beta, P);
  if (nJ) launch_k(transpose_cm_to_rm, gs(nJ * l), 256, 0, st, Bc, nJ, l, BJ);
  launch_k(transpose_cm_to_rm, gs((int64_t)k * l), 256, 0, st, Cc, k, l, Cp);
  return cudaGetLastError();
}

}  // namespace tsvd
