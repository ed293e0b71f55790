// jacobi.cu — K7/K8: one-sided block Jacobi SVD of the core (SVD_k of PAPER.md:81,
// Alg 3 line 2 P:364, Alg 4 line 3 P:381, Alg 9 line 2 P:1192).
//
// Hestenes' one-sided Jacobi orthogonalises the columns of the (tall) core K by
// plane rotations applied from the right; at convergence K V = F Θ with V the product
// of the rotations (right singular vectors) and F Θ the mutually orthogonal columns.
// Blocked for the GPU: the n columns are split into blocks of B = 16; each round of the
// round-robin tournament pairs the blocks, and one CTA per pair
//   1. forms the 32 x 32 Gram of its column slab on the DMMA pipe (mma.sync f64),
//   2. if any pair of the slab is not yet orthogonal (|g_ij| > tol max(g_ii, g_jj)),
//      diagonalises the Gram with a cyclic two-sided Jacobi in shared memory
//      (16 disjoint rotations per step), and
//   3. applies the accumulated 32 x 32 rotation to the slab of K and of V (DMMA).
// A sweep is nb-1 rounds; the host reads one rotation counter per sweep and stops at a
// sweep with no rotation (or fails with TSVD_E_SVD_FAIL after kMaxSweeps).
// Finally the column norms are the singular values; they are sorted descending, the
// leading kk columns normalised give F, the matching columns of V give G.
#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "ops.h"

namespace tsvd {

namespace {
// small pinned read-back buffers, allocated once per thread and call site (cudaMallocHost /
// cudaFreeHost per call cost far more than the kernels they read back from)
template <int SITE>
void* pinned_slot(size_t bytes) {
  static thread_local void* p = nullptr;
  static thread_local size_t sz = 0;
  if (bytes > sz) {
    if (p) cudaFreeHost(p);
    if (cudaMallocHost(&p, bytes) != cudaSuccess) {
      p = nullptr;
      sz = 0;
      return nullptr;
    }
    sz = bytes;
  }
  return p;
}
constexpr int JB = 16;          // block width
constexpr int JS = 2 * JB;      // slab width (32)
constexpr int JT = 256;         // threads per CTA
constexpr int kMaxSweeps = 60;
constexpr int kInnerSweeps = 12;

__device__ __forceinline__ int rr_block(int pos, int round, int nb) {
  return pos == 0 ? 0 : 1 + (pos - 1 + round) % (nb - 1);
}

struct JacobiSmem {
  double part[8][JS * JS];     // per-warp partial Grams
  double G[JS][JS + 1];        // Gram / working matrix
  double R[JS][JS + 1];        // accumulated rotation
  double cs[16], sn[16];
  int pp[16], qq[16];
  double red[8];
  int flag;
};

__global__ void __launch_bounds__(JT) jacobi_round_kernel(double* __restrict__ W, int64_t ldw, int64_t m, int nb,
                                                          int round, double tol, const double* __restrict__ normA2,
                                                          int* __restrict__ counter) {
  pdl_begin();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  JacobiSmem& sm = *reinterpret_cast<JacobiSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int bi = rr_block(blockIdx.x, round, nb), bj = rr_block(nb - 1 - blockIdx.x, round, nb);
  auto colidx = [&](int c) -> int64_t { return c < JB ? (int64_t)bi * JB + c : (int64_t)bj * JB + (c - JB); };
  int64_t cidx[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) cidx[q] = colidx(q * 8 + g);

  // ---- 1. Gram of the slab (upper 4x4 tile triangle), rows interleaved across warps
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int64_t r0 = (int64_t)warp * 4; r0 < m; r0 += 64) {
    const int64_t ra = r0 + t, rb = r0 + 32 + t;
    double a[4], b[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a[q] = ra < m ? W[cidx[q] * ldw + ra] : 0.0;
      b[q] = rb < m ? W[cidx[q] * ldw + rb] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = i; j < 4; ++j) {
        dmma8x8x4(acc[i][j][0], acc[i][j][1], a[i], a[j]);
        dmma8x8x4(acc[i][j][0], acc[i][j][1], b[i], b[j]);
      }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = i; j < 4; ++j) {
      sm.part[warp][(i * 8 + g) * JS + j * 8 + 2 * t] = acc[i][j][0];
      sm.part[warp][(i * 8 + g) * JS + j * 8 + 2 * t + 1] = acc[i][j][1];
    }
  __syncthreads();
  for (int e = tid; e < JS * JS; e += JT) {
    const int r = e / JS, c = e % JS;
    if ((c >> 3) >= (r >> 3)) {  // upper tile triangle
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += sm.part[w][e];
      sm.G[r][c] = s;
      if ((c >> 3) > (r >> 3)) sm.G[c][r] = s;
    }
  }
  __syncthreads();
  // within diagonal tiles only the c >= r half is exact-symmetric by construction; mirror it
  for (int e = tid; e < JS * JS; e += JT) {
    const int r = e / JS, c = e % JS;
    if ((c >> 3) == (r >> 3) && c < r) sm.G[r][c] = sm.G[c][r];
  }
  __syncthreads();

  // ---- 2. convergence test
  // pair (r, c) is orthogonal when |g_rc| <= tol sqrt(g_rr g_cc) max(1, 1e-2 / rho),
  // rho = sqrt(min/max) of the two squared norms: the plain relative test for columns of
  // comparable size, relaxed towards tol 1e-2 max(g_rr, g_cc) for very unequal ones,
  // whose relative orthogonality the Gram cannot resolve (error ~ eps / rho).
  const double floor2 = 1e-28 * (*normA2);
  double off = 0.0;
  for (int e = tid; e < JS * JS; e += JT) {
    const int r = e / JS, c = e % JS;
    if (c > r) {
      const double a = sm.G[r][r], b = sm.G[c][c];
      const double mx = fmax(a, b), mn = fmin(a, b);
      if (mx > floor2 && mn > 0.0) {
        const double rho = sqrt(mn / mx);
        const double scale = sqrt(a * b) * fmax(1.0, 1e-2 / rho);
        off = fmax(off, fabs(sm.G[r][c]) / scale);
      } else if (mx > floor2) {
        off = fmax(off, fabs(sm.G[r][c]) / (1e-2 * mx));
      }
    }
  }
  off = warp_max(off);
  if (lane == 0) sm.red[warp] = off;
  __syncthreads();
  if (tid == 0) {
    double o = 0.0;
    for (int w = 0; w < 8; ++w) o = fmax(o, sm.red[w]);
    sm.flag = o > tol;
    if (sm.flag) atomicAdd(counter, 1);
    atomicMax(reinterpret_cast<unsigned long long*>(counter + 2), __double_as_longlong(o));
  }
  __syncthreads();
  if (!sm.flag) return;

  // ---- 3. eigen-decomposition of the 32 x 32 Gram (cyclic Jacobi, parallel ordering)
  for (int e = tid; e < JS * JS; e += JT) sm.R[e / JS][e % JS] = (e / JS == e % JS) ? 1.0 : 0.0;
  __syncthreads();
  for (int sweep = 0; sweep < kInnerSweeps; ++sweep) {
    for (int step = 0; step < JS - 1; ++step) {
      if (tid < 16) {
        int pa = tid == 0 ? 0 : 1 + (tid - 1 + step) % (JS - 1);
        int pb = 1 + (JS - 1 - tid - 1 + step) % (JS - 1);
        int p = min(pa, pb), q = max(pa, pb);
        const double gpq = sm.G[p][q], gpp = sm.G[p][p], gqq = sm.G[q][q];
        double c = 1.0, s = 0.0;
        if (fabs(gpq) > 1e-300 && fabs(gpq) > 1e-16 * sqrt(fabs(gpp) * fabs(gqq))) {
          const double tau = (gqq - gpp) / (2.0 * gpq);
          const double tt = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + tt * tt);
          s = tt * c;
        }
        sm.pp[tid] = p;
        sm.qq[tid] = q;
        sm.cs[tid] = c;
        sm.sn[tid] = s;
      }
      __syncthreads();
      for (int e = tid; e < 16 * JS; e += JT) {  // rows p, q  <- J^T G
        const int pr = e / JS, j = e % JS;
        const int p = sm.pp[pr], q = sm.qq[pr];
        const double c = sm.cs[pr], s = sm.sn[pr];
        const double a = sm.G[p][j], b = sm.G[q][j];
        sm.G[p][j] = c * a - s * b;
        sm.G[q][j] = s * a + c * b;
      }
      __syncthreads();
      for (int e = tid; e < 16 * JS; e += JT) {  // columns p, q  <- G J ; R <- R J
        const int pr = e / JS, i = e % JS;
        const int p = sm.pp[pr], q = sm.qq[pr];
        const double c = sm.cs[pr], s = sm.sn[pr];
        double a = sm.G[i][p], b = sm.G[i][q];
        sm.G[i][p] = c * a - s * b;
        sm.G[i][q] = s * a + c * b;
        a = sm.R[i][p];
        b = sm.R[i][q];
        sm.R[i][p] = c * a - s * b;
        sm.R[i][q] = s * a + c * b;
      }
      __syncthreads();
    }
    // inner convergence
    double o = 0.0;
    for (int e = tid; e < JS * JS; e += JT) {
      const int r = e / JS, c = e % JS;
      if (c > r) {
        const double pr = sqrt(fabs(sm.G[r][r]) * fabs(sm.G[c][c]));
        if (pr > 0) o = fmax(o, fabs(sm.G[r][c]) / pr);
      }
    }
    o = warp_max(o);
    if (lane == 0) sm.red[warp] = o;
    __syncthreads();
    if (tid == 0) {
      double oo = 0.0;
      for (int w = 0; w < 8; ++w) oo = fmax(oo, sm.red[w]);
      sm.flag = oo > 1e-15;
    }
    __syncthreads();
    if (!sm.flag) {
      if (tid == 0) atomicMax(counter + 4, sweep + 1);
      break;
    }
    if (sweep == kInnerSweeps - 1 && tid == 0) atomicMax(counter + 4, kInnerSweeps + 1);
  }

  // ---- 4. apply the rotation to the slab of W (m rows), in place
  auto apply = [&](double* X, int64_t ld, int64_t rows) {
    for (int64_t r0 = (int64_t)warp * 8; r0 < rows; r0 += 64) {
      const int64_t row = r0 + g;
      double a[8];
#pragma unroll
      for (int l = 0; l < 8; ++l) a[l] = row < rows ? X[colidx(l * 4 + t) * ld + row] : 0.0;
      double o[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j][0] = o[j][1] = 0.0;
#pragma unroll
      for (int l = 0; l < 8; ++l)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma8x8x4(o[j][0], o[j][1], a[l], sm.R[l * 4 + t][j * 8 + g]);
      if (row < rows) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          X[colidx(j * 8 + 2 * t) * ld + row] = o[j][0];
          X[colidx(j * 8 + 2 * t + 1) * ld + row] = o[j][1];
        }
      }
    }
  };
  apply(W, ldw, m);
}

// ||A||_F^2 in a fixed order (deterministic): block b sums columns b, b + grid, .. into
// part[b] (rows by the threads, 128-bit loads when contiguous), then one block sums the
// partials in index order; out must be zero-initialised by the caller (it is overwritten here)
__global__ void __launch_bounds__(256) frob2_part_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                                         double* __restrict__ part) {
  pdl_begin();
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const double* col = A + j * lda;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) s = fma(col[i], col[i], s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}
__global__ void frob2_sum_kernel(const double* __restrict__ part, int np, double* out) {
  pdl_begin();
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}
cudaError_t frob2(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, double* out, Scratch& ws) {
  const int np = (int)std::max<int64_t>(1, std::min<int64_t>(n, 148 * 8));
  double* part = ws.alloc<double>(np);
  if (ws.err) return ws.err;
  g_launches += 2;
  launch_k(frob2_part_kernel, np, 256, 0, st, A, lda, m, n, part);
  launch_k(frob2_sum_kernel, 1, 1024, 0, st, part, np, out);
  return cudaGetLastError();
}

__global__ void copy_pad_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n, double* __restrict__ W,
                                int64_t ldw, int64_t npad) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ldw * npad; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / ldw, i = e % ldw;
    W[e] = (i < m && j < n) ? A[j * lda + i] : 0.0;
  }
}

__global__ void eye_kernel(double* V, int64_t n) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x)
    V[e] = (e / n == e % n) ? 1.0 : 0.0;
}

__global__ void colnorm_kernel(const double* __restrict__ W, int64_t ldw, int64_t m, int64_t n, double* __restrict__ nrm) {
  pdl_begin();
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  double s = 0.0;
  for (int64_t i = lane; i < m; i += 32) {
    const double x = W[j * ldw + i];
    s = fma(x, x, s);
  }
  s = warp_sum(s);
  if (lane == 0) nrm[j] = sqrt(s);
}

// single-CTA bitonic sort of (value desc, index asc) pairs, npow2 <= 16384
__global__ void __launch_bounds__(1024) sort_desc_kernel(const double* __restrict__ nrm, int64_t n, int npow2,
                                                         int* __restrict__ perm, double* __restrict__ theta,
                                                         int64_t ntheta) {
  pdl_begin();
  extern __shared__ unsigned char sraw[];
  double* key = reinterpret_cast<double*>(sraw);
  int* idx = reinterpret_cast<int*>(key + npow2);
  for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
    key[i] = i < n ? nrm[i] : -1.0;
    idx[i] = i;
  }
  __syncthreads();
  for (int size = 2; size <= npow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;
          const double ki = key[i], kj = key[j];
          const int ii = idx[i], ij = idx[j];
          // "a before b" in descending order with index tie-break
          const bool j_first = (kj > ki) || (kj == ki && ij < ii);
          if (desc ? j_first : !j_first) {
            key[i] = kj; key[j] = ki;
            idx[i] = ij; idx[j] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
    perm[i] = idx[i];
    if (i < ntheta) theta[i] = key[i] > 0 ? key[i] : 0.0;
  }
}

// F[:, j] = W[:, perm[j]] / sigma (col-major output), j < kk; counts the columns with sigma <= tiny
__global__ void extract_kernel(const double* __restrict__ W, int64_t ldw, int64_t m, const int* __restrict__ perm,
                               const double* __restrict__ nrm, int kk, double tiny, double* __restrict__ F, int64_t ldf,
                               int* __restrict__ deficient) {
  pdl_begin();
  const int j = blockIdx.y;
  const int pj = perm[j];
  const double sg = nrm[pj];
  const bool ok = sg > tiny;
  if (!ok && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(deficient, 1);
  const double inv = ok ? 1.0 / sg : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    F[j * ldf + i] = W[(int64_t)pj * ldw + i] * inv;
}

// X[:, j] *= 1 / theta[j] (0 where theta[j] <= tiny), col-major rows x cols
__global__ void scale_cols_kernel(double* __restrict__ X, int64_t ldx, int64_t rows, int cols,
                                  const double* __restrict__ theta, double tiny) {
  pdl_begin();
  const int j = blockIdx.y;
  const double t = theta[j];
  const double inv = t > tiny ? 1.0 / t : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    X[j * ldx + i] *= inv;
}

// perm = identity, nrm = theta (for complete_kernel on outputs already in sorted order)
__global__ void ident_perm_kernel(int* perm, int n) {
  pdl_begin();
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
}

// out[j] = ||X[:, j] - ...|| : squared norms of the columns of R = HYU - G diag(theta^2), col-major
__global__ void resid_kernel(const double* __restrict__ HYU, const double* __restrict__ G, int64_t n, int cols,
                             const double* __restrict__ theta, double* __restrict__ out) {
  pdl_begin();
  __shared__ double red[8];
  const int j = blockIdx.x;
  const double t2 = theta[j] * theta[j];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double r = HYU[j * n + i] - t2 * G[j * n + i];
    a = fma(r, r, a);
  }
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    out[j] = sqrt(t);
  }
}

__global__ void trace_kernel(const double* __restrict__ H, int64_t n, double* out) {
  pdl_begin();
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a += H[i * n + i];
  a = warp_sum(a);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += red[w];
    *out = t;
  }
}

// Y (n x b row-major): columns j < k0 = e_j, the rest keep the K12 draw already written
__global__ void init_basis_kernel(double* Y, int64_t n, int b, int k0) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * b; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / b;
    const int j = (int)(e % b);
    if (j < k0) Y[e] = (i == j) ? 1.0 : 0.0;
    else if (i < k0) Y[e] = 0.0;  // the other columns projected off span(e_1 .. e_k0)
  }
}

// Orthonormal completion of the F columns whose singular value is ~0:
// for each such column, Gram-Schmidt (twice) a unit vector e_c against all other columns.
__global__ void __launch_bounds__(256) complete_kernel(double* F, int64_t ldf, int64_t m, int kk,
                                                       const int* __restrict__ perm, const double* __restrict__ nrm,
                                                       double tiny_h, const double* __restrict__ tiny_dev = nullptr) {
  pdl_begin();
  const double tiny = tiny_dev ? *tiny_dev : tiny_h;
  __shared__ double red[8];
  __shared__ double coef;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int cand = 0;
  for (int j = 0; j < kk; ++j) {
    if (nrm[perm[j]] > tiny) continue;
    double* f = F + (int64_t)j * ldf;
    for (int attempt = 0; attempt < 4 * kk + 8 && cand < m; ++attempt, ++cand) {
      for (int64_t i = tid; i < m; i += 256) f[i] = (i == cand) ? 1.0 : 0.0;
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int l = 0; l < kk; ++l) {
          if (l == j) continue;
          const double* fl = F + (int64_t)l * ldf;
          bool valid = (nrm[perm[l]] > tiny) || (l < j);
          if (!valid) continue;
          double s = 0.0;
          for (int64_t i = tid; i < m; i += 256) s = fma(fl[i], f[i], s);
          s = warp_sum(s);
          if (lane == 0) red[w] = s;
          __syncthreads();
          if (tid == 0) { double a = 0; for (int q = 0; q < 8; ++q) a += red[q]; coef = a; }
          __syncthreads();
          for (int64_t i = tid; i < m; i += 256) f[i] -= coef * fl[i];
          __syncthreads();
        }
      }
      double s = 0.0;
      for (int64_t i = tid; i < m; i += 256) s = fma(f[i], f[i], s);
      s = warp_sum(s);
      if (lane == 0) red[w] = s;
      __syncthreads();
      if (tid == 0) { double a = 0; for (int q = 0; q < 8; ++q) a += red[q]; coef = sqrt(a); }
      __syncthreads();
      const double nn = coef;
      if (nn > 0.5) {
        for (int64_t i = tid; i < m; i += 256) f[i] /= nn;
        __syncthreads();
        ++cand;
        break;
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- K7: CTA-resident Jacobi
// The whole m x n core (m, n <= 128) lives in shared memory; one CTA of 512 threads runs
// every sweep without leaving the kernel: per step the n/2 disjoint column pairs of the
// round-robin tournament are rotated, one pair per 16-lane group (2 pairs per warp, 32
// warps; dot products in two independent chains, reduced with 4 xor-shuffles), and a
// block-wide rotation count ends the sweeps.
// Then theta = column norms (descending, index tie-break) and F = the leading kk
// normalised columns.
constexpr int K7_MAX = 128;
constexpr int K7_SWEEPS = 40;
constexpr int K7_THREADS = 1024;
constexpr int K7_GL = 16;                 // lanes per column pair
constexpr int K7_GPW = 32 / K7_GL;        // pairs per warp

__device__ __forceinline__ int k7_pos(int slot, int step, int N) {  // tournament: slot -> player
  const int x = slot - 1 + step;  // < 2 (N - 1): one conditional subtraction, no division
  return slot == 0 ? 0 : 1 + (x >= N - 1 ? x - (N - 1) : x);
}

template <int GL>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = GL / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// NU: rows per lane of a 16-lane group, ceil(m / 16) <= NU; NT threads = 16 per column pair.
// m <= 96 (so n <= 96, 48 pairs): NU = 6 with 768 threads — no idle groups issuing every round,
// and 85 registers per thread instead of 64 (no spills); else NU = 8 with 1024.
template <int NU, int NT, int GL = K7_GL, bool FULL = false>  // FULL: m == NU * GL (no row predicates)
__global__ void __launch_bounds__(NT) jacobi_cta_kernel(const double* __restrict__ A, int64_t lda, int m, int n,
                                                                int kk, double tol, double* __restrict__ theta,
                                                                double* __restrict__ F, int64_t ldf,
                                                                int* __restrict__ info, double* __restrict__ tiny_out) {
  pdl_begin();
  extern __shared__ double Wsm[];                  // column-major, ld = mp
  __shared__ int rot_count;
  __shared__ double nrm2_s[K7_MAX];
  __shared__ double nrm_s[K7_MAX + 1];
  __shared__ int rank_s[K7_MAX + 1];
  const int mp = m | 1;                            // odd pitch: conflict-free column walks
  const int N = (n + 1) & ~1;                      // even player count (a zero column if n odd)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int GPW = 32 / GL;  // pairs per warp
  const int grp = lane / GL, li = lane % GL;
  for (int e = tid; e < mp * N; e += blockDim.x) {
    const int j = e / mp, i = e % mp;
    Wsm[e] = (i < m && j < n) ? A[(int64_t)j * lda + i] : 0.0;
  }
  __syncthreads();
  int sweep = 0;
  for (; sweep < K7_SWEEPS; ++sweep) {
    if (tid == 0) rot_count = 0;
    for (int j = warp; j < N; j += NT / 32) {  // exact squared column norms
      double a = 0.0;
      for (int i = lane; i < m; i += 32) a = fma(Wsm[j * mp + i], Wsm[j * mp + i], a);
      a = warp_sum(a);
      if (lane == 0) nrm2_s[j] = a;
    }
    __syncthreads();
    int local = 0;
    for (int step = 0; step < N - 1; ++step) {
      // one barrier per round: every group dots its pair (held in registers), reads the pair's
      // carried squared norms, computes the rotation itself (all its lanes the same values from
      // the same inputs) and rotates — the parameters for a column pair of round r are made
      // only by its own group, and the norms it writes are read by other groups only in round
      // r + 1, after the barrier.  (One lane per pair in two warps between two more barriers
      // left 22 warps idle through the divide / square-root chain.)
      const int pr = warp * GPW + grp;
      const bool live = pr < N / 2;
      const int p0 = live ? k7_pos(pr, step, N) : 0, q0 = live ? k7_pos(N - 1 - pr, step, N) : 0;
      const int p = min(p0, q0), q = max(p0, q0);
      double* xp = Wsm + p * mp;
      double* xq = Wsm + q * mp;
      double u[NU], v[NU];
      double c0 = 0.0, c1 = 0.0;  // two chains
#pragma unroll
      for (int x = 0; x < NU; ++x) {
        const int i = li + GL * x;
        const bool in = live && (FULL || i < m);
        u[x] = in ? xp[i] : 0.0;
        v[x] = in ? xq[i] : 0.0;
        if (x & 1) c1 = fma(u[x], v[x], c1);
        else c0 = fma(u[x], v[x], c0);
      }
      const double cc = group_sum<GL>(c0 + c1);
      if (live) {
        // the squared norms are carried through the rotation (a' = a - t c, b' = b + t c) and
        // recomputed exactly at every sweep start, so a round only dots the pair once
        const double a = nrm2_s[p], b = nrm2_s[q];
        // |c| > tol sqrt(a b) squared: no square root on the round's chain
        const bool rot = a > 0.0 && b > 0.0 && cc * cc > (tol * tol) * (a * b);
        if (rot) {  // uniform within the group
          // t = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (b - a) / 2c, without forming
          // zeta: t = g / D with g = 2c sgn(b - a), D = |b - a| + sqrt((b - a)^2 + 4c^2); and
          // cs = 1 / sqrt(1 + t^2) = D rsqrt(D^2 + g^2), sn = g rsqrt(D^2 + g^2): the rsqrt and
          // the division for t (needed only by the carried norms) both start from D
          const double c2 = 2.0 * cc, h = b - a, g2 = h >= 0 ? c2 : -c2;
          const double D = fabs(h) + sqrt(fma(h, h, c2 * c2));
          const double qn = rsqrt(fma(D, D, c2 * c2));
          const double cs = D * qn, sn = g2 * qn;
#pragma unroll
          for (int x = 0; x < NU; ++x) {
            const int i = li + GL * x;
            if (FULL || i < m) {
              xp[i] = cs * u[x] - sn * v[x];
              xq[i] = sn * u[x] + cs * v[x];
            }
          }
          if (li == 0) {
            const double t = g2 / D;
            nrm2_s[p] = fma(-t, cc, a);
            nrm2_s[q] = fma(t, cc, b);
            ++local;
          }
        }
      }
      __syncthreads();
    }
    if (local) atomicAdd(&rot_count, local);
    __syncthreads();
    if (rot_count == 0) break;
    __syncthreads();
  }
  // column norms, descending rank (index tie-break)
  const int nwarps = blockDim.x >> 5;
  for (int j = warp; j < n; j += nwarps) {
    double a = 0.0;
    for (int i = lane; i < m; i += 32) a = fma(Wsm[j * mp + i], Wsm[j * mp + i], a);
    a = warp_sum(a);
    if (lane == 0) nrm_s[j] = sqrt(a);
  }
  __syncthreads();
  for (int j = tid; j < n; j += blockDim.x) {
    const double v = nrm_s[j];
    int r = 0;
    for (int l = 0; l < n; ++l) r += (nrm_s[l] > v) || (nrm_s[l] == v && l < j);
    rank_s[j] = r;
    theta[r] = v;
  }
  __syncthreads();
  double fro = 0.0;
  for (int j = 0; j < n; ++j) fro = fma(nrm_s[j], nrm_s[j], fro);
  const double tiny = 1e-14 * sqrt(fro) + 1e-300;
  for (int j = warp; j < n; j += nwarps) {
    const int r = rank_s[j];
    if (r >= kk) continue;
    const double inv = nrm_s[j] > tiny ? 1.0 / nrm_s[j] : 0.0;
    for (int i = lane; i < m; i += 32) F[(int64_t)r * ldf + i] = Wsm[j * mp + i] * inv;
  }
  if (tid == 0 && info) {
    info[0] = sweep + 1;
    info[1] = sweep < K7_SWEEPS;
    *tiny_out = tiny;
  }
}
}  // namespace

// One-sided block Jacobi of A (m x n col-major, m >= n) without accumulating the
// rotations: theta (all n values, descending), F (m x kk, ldf) = the normalised leading
// columns (left singular vectors), orthonormally completed where theta ~ 0.
// async_info (K7 path only, no profiling): no synchronisation — the completion is enqueued
// unconditionally (a no-op unless theta ~ 0; its result unused if the sweeps did not converge)
// and *async_info receives the pinned host buffer {sweeps, converged, tiny} the caller reads
// after its own next synchronisation
// top_only > 0 (K9 path): only the top_only largest values / vectors are needed (ops.h jacobi_cluster)
cudaError_t jacobi_cols(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, int kk, double* theta,
                        double* F, int64_t ldf, int* sweeps, bool* converged, Scratch& ws, KProf* prof,
                        double* tiny_out, const int** async_info = nullptr, int top_only = 0) {
  long long* launches = &g_launches;
  *sweeps = 0;
  *converged = false;
  if (n <= 0 || m <= 0) { *converged = true; return cudaSuccess; }
  if (m < n) return cudaErrorInvalidValue;
  static const bool k9_on = !(getenv("TSVD_K9") && atoi(getenv("TSVD_K9")) == 0);
  // K7 (one CTA) only up to 64 columns: above, K9 on a 4- or 8-CTA cluster is faster — the
  // one-CTA round moves every column through one SM's shared memory (n = 116: 1.8 vs 1.0 ms
  // per C1 core, 1.5 vs 1.2 ms per C2 step); TSVD_K7_MAXN overrides (tuning)
  static const int k7_maxn = getenv("TSVD_K7_MAXN") ? atoi(getenv("TSVD_K7_MAXN")) : 64;
  const bool use_k9 = (n > k7_maxn || !(m <= K7_MAX && n <= K7_MAX)) && k9_on && k9_supported(m, n);
  if ((m <= K7_MAX && n <= K7_MAX) || use_k9) {
    // K7: the whole core resident in one CTA's shared memory; K9: in one CTA cluster
    int* d_info = ws.alloc<int>(4);
    int* perm = ws.alloc<int>(K7_MAX);
    double* d_tiny = reinterpret_cast<double*>(d_info + 2);
    int* h_info = nullptr;
    if (ws.err) return ws.err;
    cudaError_t e;
    h_info = static_cast<int*>(pinned_slot<1>(4 * sizeof(int)));
    if (!h_info) return cudaErrorMemoryAllocation;
    const int mp = (int)(m | 1), N = (int)((n + 1) & ~1);
    const size_t smem = (size_t)mp * N * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(jacobi_cta_kernel<6, 768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(jacobi_cta_kernel<6, 768, K7_GL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      cudaFuncSetAttribute(jacobi_cta_kernel<12, 384, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(jacobi_cta_kernel<8, K7_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    const int pidx = g_prof ? g_prof->begin(KC_JACOBI, 0.0, 0.0) : -1;
    // (8 lanes per pair on 12 warps measured slower: 2.06 vs 1.62 ms per batch — the rounds are
    // latency-bound and 24 warps hide more of it)
    static const int gl = getenv("TSVD_K7_GL") ? atoi(getenv("TSVD_K7_GL")) : 16;  // tuning
    if (use_k9) {
      if ((e = jacobi_cluster(st, A, lda, m, n, kk, 1e-14, theta, F, ldf, d_info, d_tiny, top_only))) {
        if (pidx >= 0) g_prof->end(pidx);
        return e;
      }
    } else if (m <= 96 && gl == 8)
      launch_k(jacobi_cta_kernel<12, 384, 8>, 1, 384, smem, st, A, lda, (int)m, (int)n, kk, 1e-14, theta, F, ldf, d_info,
               d_tiny);
    else if (m == 6 * K7_GL)  // the core reduction's b = 96
      launch_k(jacobi_cta_kernel<6, 768, K7_GL, true>, 1, 768, smem, st, A, lda, (int)m, (int)n, kk, 1e-14, theta, F, ldf,
               d_info, d_tiny);
    else if (m <= 6 * K7_GL)
      launch_k(jacobi_cta_kernel<6, 768>, 1, 768, smem, st, A, lda, (int)m, (int)n, kk, 1e-14, theta, F, ldf, d_info, d_tiny);
    else
      launch_k(jacobi_cta_kernel<8, K7_THREADS>, 1, K7_THREADS, smem, st, A, lda, (int)m, (int)n, kk, 1e-14, theta, F, ldf, d_info, d_tiny);
    *launches += 1;   // (before the class scope closes: counted as a core_jacobi launch)
    if (pidx >= 0) g_prof->end(pidx);
    cudaMemcpyAsync(h_info, d_info, 4 * sizeof(int), cudaMemcpyDeviceToHost, st);
    if (async_info && pidx < 0) {
      if (kk > 0) {
        launch_k(ident_perm_kernel, 1, 256, 0, st, perm, kk);
        launch_k(complete_kernel, 1, 256, 0, st, F, ldf, m, kk, perm, theta, 0.0, d_tiny);
        *launches += 2;
      }
      *async_info = h_info;
      return cudaGetLastError();
    }
    if ((e = cudaStreamSynchronize(st)) == cudaSuccess) e = cudaGetLastError();
    *sweeps = h_info[0];
    *converged = h_info[1] != 0;
    if (pidx >= 0) {
      // per sweep: n(n-1)/2 pair dot products (3 m flops x 2) + rotations (6 m flops)
      const double fl = (double)h_info[0] * n * (n - 1) / 2.0 * 12.0 * m;
      g_prof->set(pidx, fl, 8.0 * m * n * 2.0);
    }
    double tiny = 0.0;
    memcpy(&tiny, h_info + 2, sizeof(double));
    if (tiny_out) *tiny_out = tiny;
    if (e == cudaSuccess && *converged && kk > 0) {
      // orthonormal completion of columns with theta ~ 0 (no-op otherwise)
      launch_k(ident_perm_kernel, 1, 256, 0, st, perm, kk);
      launch_k(complete_kernel, 1, 256, 0, st, F, ldf, m, kk, perm, theta, 0.0, d_tiny);
      *launches += 2;
      e = cudaGetLastError();
    }
    return e;
  }
  const int64_t npad = ((n + JS - 1) / JS) * JS;
  const int nb = (int)(npad / JB);
  const int64_t ldw = ((m + 7) / 8) * 8;
  double* W = ws.alloc<double>((size_t)ldw * npad);
  double* nrm = ws.alloc<double>(npad + 1);
  int* counter = ws.alloc<int>(8);
  int* perm = ws.alloc<int>(16384);
  int* h_cnt = nullptr;
  if (ws.err) return ws.err;
  cudaError_t e;
  h_cnt = static_cast<int*>(pinned_slot<2>(8 * sizeof(int)));
  if (!h_cnt) return cudaErrorMemoryAllocation;
  static const bool trace = getenv("TSVD_TRACE") != nullptr;
  const unsigned gbig = 148 * 8;
  launch_k(copy_pad_kernel, gbig, 256, 0, st, A, lda, m, n, W, ldw, npad);
  double* normA2 = nrm + npad;
  cudaMemsetAsync(normA2, 0, sizeof(double), st);
  if ((e = frob2(st, W, ldw, ldw, npad, normA2, ws))) return e;
  *launches += 1;
  static bool attr = false;
  const size_t smem = sizeof(JacobiSmem);
  if (!attr) {
    cudaFuncSetAttribute(jacobi_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const double tol = 1e-13;
  // algorithmic work of one round-kernel CTA: the slab Gram (m x JS,
  // symmetric: m JS (JS+1) flops, reads m JS 8 B) and, if the slab is not yet orthogonal,
  // its rotation (2 m JS^2 flops, read + write of the slab).
  const double gram_flops = (double)m * JS * (JS + 1), gram_bytes = (double)m * JS * 8.0;
  const double rot_flops = 2.0 * (double)m * JS * JS, rot_bytes = 2.0 * (double)m * JS * 8.0;
  for (int sw = 0; sw < kMaxSweeps; ++sw) {
    cudaMemsetAsync(counter, 0, 8 * sizeof(int), st);
    const int pidx = g_prof ? g_prof->begin(KC_JACOBI, 0.0, 0.0) : -1;
    for (int r = 0; r < nb - 1; ++r) {
      launch_k(jacobi_round_kernel, nb / 2, JT, smem, st, W, ldw, m, nb, r, tol, normA2, counter);
      ++*launches;
    }
    if (pidx >= 0) g_prof->end(pidx);
    if ((e = cudaGetLastError())) break;
    cudaMemcpyAsync(h_cnt, counter, 8 * sizeof(int), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st))) break;
    if (trace) {
      double mo;
      memcpy(&mo, h_cnt + 2, sizeof(double));
      fprintf(stderr, "[jacobi] m=%lld n=%lld sweep %d active %d/%d max_off %.3e inner_sweeps %d\n", (long long)m,
              (long long)n, sw, h_cnt[0], (nb - 1) * (nb / 2), mo, h_cnt[4]);
    }
    if (pidx >= 0) {
      const double ctas = (double)(nb - 1) * (nb / 2);
      g_prof->set(pidx, ctas * gram_flops + (double)h_cnt[0] * rot_flops, ctas * gram_bytes + (double)h_cnt[0] * rot_bytes);
    }
    *sweeps = sw + 1;
    if (h_cnt[0] == 0) {
      *converged = true;
      break;
    }
  }
  if (e == cudaSuccess && *converged) {
    launch_k(colnorm_kernel, cdiv(npad * 32, 256), 256, 0, st, W, ldw, m, npad, nrm);
    int p2 = 1;
    while (p2 < npad) p2 <<= 1;
    if (p2 > 16384) {
      e = cudaErrorInvalidValue;
    } else {
      const size_t ssm = (size_t)p2 * (sizeof(double) + sizeof(int));
      static bool attr2 = false;
      if (!attr2) {
        cudaFuncSetAttribute(sort_desc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr2 = true;
      }
      launch_k(sort_desc_kernel, 1, 1024, ssm, st, nrm, npad, p2, perm, theta, n);
      // tiny: singular values below 1e-14 ||A||_F are treated as exact zeros
      double h_norm2 = 0.0;
      cudaMemcpyAsync(&h_norm2, normA2, sizeof(double), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const double tiny = 1e-14 * sqrt(h_norm2) + 1e-300;
      if (tiny_out) *tiny_out = tiny;
      cudaMemsetAsync(counter + 1, 0, sizeof(int), st);
      dim3 grid(std::max<unsigned>(1, std::min<unsigned>(cdiv(m, 256), 64)), kk);
      if (kk > 0) launch_k(extract_kernel, grid, 256, 0, st, W, ldw, m, perm, nrm, kk, tiny, F, ldf, counter + 1);
      cudaMemcpyAsync(&h_cnt[1], counter + 1, sizeof(int), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      if (h_cnt[1] > 0) launch_k(complete_kernel, 1, 256, 0, st, F, ldf, m, kk, perm, nrm, tiny, nullptr);
      *launches += 4;
      e = cudaGetLastError();
    }
  }
  (void)prof;
  return e;
}

namespace {
// G (n x kk col-major, ldg) = A^T F diag(1/theta)  (right singular vectors from the left
// ones: A^T f_j = theta_j g_j), completed orthonormally where theta ~ 0.
cudaError_t right_from_left(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, int kk,
                            const double* F, int64_t ldf, const double* theta, double tiny, double* G, int64_t ldg,
                            Scratch& ws) {
  if (kk <= 0) return cudaSuccess;
  cudaError_t e = dgemm(st, n, kk, m, 1.0, CMat{A, lda, 1}, CMat{F, 1, ldf}, 0.0, Mat{G, 1, ldg}, 0);
  if (e) return e;
  dim3 grid(std::max<unsigned>(1, std::min<unsigned>(cdiv(n, 256), 64)), kk);
  g_launches += 2;
  launch_k(scale_cols_kernel, grid, 256, 0, st, G, ldg, n, kk, theta, tiny);
  int* perm = ws.alloc<int>(kk);
  if (ws.err) return ws.err;
  launch_k(ident_perm_kernel, 1, 256, 0, st, perm, kk);
  // completion where theta_j <= tiny (the same columns F completed)
  g_launches += 1;
  launch_k(complete_kernel, 1, 256, 0, st, G, ldg, n, kk, perm, theta, tiny, nullptr);
  return cudaGetLastError();
}

// F (m x kk col-major) = A G diag(1/theta), completed where theta ~ 0
cudaError_t left_from_right(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, int kk,
                            const double* G, int64_t ldg, const double* theta, double tiny, double* F, int64_t ldf,
                            Scratch& ws) {
  if (kk <= 0) return cudaSuccess;
  cudaError_t e = dgemm(st, m, kk, n, 1.0, CMat{A, 1, lda}, CMat{G, 1, ldg}, 0.0, Mat{F, 1, ldf}, 0);
  if (e) return e;
  dim3 grid(std::max<unsigned>(1, std::min<unsigned>(cdiv(m, 256), 64)), kk);
  g_launches += 3;
  launch_k(scale_cols_kernel, grid, 256, 0, st, F, ldf, m, kk, theta, tiny);
  int* perm = ws.alloc<int>(kk);
  if (ws.err) return ws.err;
  launch_k(ident_perm_kernel, 1, 256, 0, st, perm, kk);
  launch_k(complete_kernel, 1, 256, 0, st, F, ldf, m, kk, perm, theta, tiny, nullptr);
  return cudaGetLastError();
}
}  // namespace

// Full-spectrum path (kept for tsvd_k_jacobi_svd): theta (n), F (m x kk), G (n x kk).
cudaError_t jacobi_svd(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, int kk, double* theta,
                       double* F, int64_t ldf, double* G, int64_t ldg, int* sweeps, bool* converged, Scratch& ws,
                       KProf* prof) {
  double tiny = 0.0;
  cudaError_t e = jacobi_cols(st, A, lda, m, n, kk, theta, F, ldf, sweeps, converged, ws, prof, &tiny);
  if (e || !*converged) return e;
  return right_from_left(st, A, lda, m, n, kk, F, ldf, theta, tiny, G, ldg, ws);
}

// SVD_kk of the core (DESIGN.md §6 "core SVD"): see ops.h.
namespace {
// per 64-row block of A (Z = A Y) and of A^T (A^T Z): the K range holding the block's
// structurally nonzero entries (CoreShape)
__global__ void core_kr_kernel(int k, int64_t r, const int32_t* __restrict__ klist, int64_t mc, int64_t nc,
                               int2* __restrict__ krZ, int nbZ, int2* __restrict__ krH, int nbH) {
  pdl_begin();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nbZ) {
    const int64_t i = min((int64_t)(t + 1) * 64, mc) - 1;  // last row of the block
    int64_t kend;
    if (i < k) {
      kend = i + 1;
    } else {  // k + #{c : klist[c] <= i - k}
      int64_t lo = 0, hi = r;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (klist[mid] <= i - k) lo = mid + 1;
        else hi = mid;
      }
      kend = k + lo;
    }
    krZ[t] = make_int2(0, (int)kend);
  }
  if (t < nbH) {
    const int64_t j0 = (int64_t)t * 64;
    // (started at an even index — one structurally zero row more at most — so that the GEMM's
    // k offsets stay even and its 16-byte pair staging aligned)
    krH[t] = make_int2((int)(j0 < k ? j0 : k + klist[j0 - k]) & ~1, (int)mc);
  }
}
}  // namespace

cudaError_t core_svd(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, int kk, double* theta,
                     double* F, int64_t ldf, double* G, int64_t ldg, CoreInfo* info, Scratch& ws, KProf* prof,
                     const CoreShape* shape) {
  info->path = 0;
  info->iters = 0;
  info->sweeps = 0;
  info->converged = false;
  cudaError_t e;
  static const bool trace = getenv("TSVD_TRACE") != nullptr;
  static const int force_full = getenv("TSVD_CORE_FULL") ? atoi(getenv("TSVD_CORE_FULL")) : 0;
  double* h = nullptr;
  h = static_cast<double*>(pinned_slot<3>(4 * sizeof(double)));
  if (!h) return cudaErrorMemoryAllocation;
  // energy = ||A||_F^2 (= sum of all theta^2)
  double* d_en = ws.alloc<double>(1);
  if (ws.err) return ws.err;
  cudaMemsetAsync(d_en, 0, sizeof(double), st);
  if ((e = frob2(st, A, lda, m, n, d_en, ws))) return e;
  // read back with the next synchronisation (the first Ritz check or the Jacobi), not now
  cudaMemcpyAsync(h, d_en, sizeof(double), cudaMemcpyDeviceToHost, st);

  static const bool cheb_on = !(getenv("TSVD_CORE_CHEB") && atoi(getenv("TSVD_CORE_CHEB")) == 0);
  // subspace width: kk + extra (default extra = max(32, kk / 2): b = 96 at kk = 64 measured
  // best on configs[1], against 128 and 160); TSVD_CORE_EXTRA overrides (tuning)
  static const int extra_env = getenv("TSVD_CORE_EXTRA") ? atoi(getenv("TSVD_CORE_EXTRA")) : 0;
  const int extra = extra_env > 0 ? extra_env : std::max(32, kk / 2);
  // a previous update of the stream that saw the Ritz values collapse right after kk (configs[3]:
  // (theta_144 / theta_128)^2 ~ 1e-4) suggests a narrower subspace: a cheaper Ritz Jacobi, the
  // same iterations
  const int b = info->b_hint > kk ? (int)std::min<int64_t>(n, info->b_hint)
                                   : (int)std::min<int64_t>(n, ((kk + extra + 31) / 32) * 32);
  // the reduction pays once the direct Jacobi would leave the one-CTA K7 (n > 128): its cost is
  // a few b x b Rayleigh-Ritz Jacobis on a nearly diagonal matrix instead of one on the n x n core
  static const int rr_min = getenv("TSVD_RR_MIN") ? atoi(getenv("TSVD_RR_MIN")) : 129;  // tuning
  // (tall cores below 512 columns keep the Cholesky-QR2 + Jacobi path)
  const bool subspace = !force_full && b <= n / 2 && (n >= 512 || (n >= rr_min && m < 2 * n));
  if (subspace) {
    // ---- Rayleigh-Ritz on a subspace iteration with A^T A applied as A^T (A Y)
    info->path = 2;
    double* Y = ws.alloc<double>((size_t)n * b);       // row-major n x b, orthonormal
    double* HY = ws.alloc<double>((size_t)n * b);      // row-major: A^T A Y
    double* Z = ws.alloc<double>((size_t)m * b);       // row-major: A Y
    double* Zq = ws.alloc<double>((size_t)m * b);      // row-major: Q factor of Z (check iterations)
    double* Rz = ws.alloc<double>((size_t)b * b);      // row-major upper = R_z^T col-major
    double* th = ws.alloc<double>(b);
    double* Ux = ws.alloc<double>((size_t)b * b);         // col-major b x b (Ritz rotation)
    double* Gc = ws.alloc<double>((size_t)n * (kk + 1));  // col-major
    double* HU = ws.alloc<double>((size_t)n * (kk + 1));  // col-major
    double* res = ws.alloc<double>(kk + 1);
    int* perm = ws.alloc<int>(kk + 1);
    if (ws.err) return ws.err;
    // start: the first kk coordinate directions (the previous singular directions in the
    // update cores) plus K12 Gaussian columns
    if ((e = counter_gaussian(st, 0x5eed5eedull, 2, n, b, Y))) return e;
    ++g_launches;
    launch_k(init_basis_kernel, 148 * 4, 256, 0, st, Y, n, b, std::min(kk, b));
    // [e_1 .. e_k0 | G] with G's first k0 rows zeroed: the coordinate block is orthonormal and
    // orthogonal to G, so Cholesky-QR2 of G alone gives the basis Cholesky-QR2 of the whole
    // block would (its Gram is [I 0; 0 G^T G]) — two (b - k0)-column factorisations (configs[3]:
    // 16 columns, one CTA) instead of two b-column tile-DAG ones on the serial core path
    if (const int k0 = std::min(kk, b); b > k0) {
      double* Gt = ws.alloc<double>((size_t)n * (b - k0));
      if (ws.err) return ws.err;
      const size_t w = (size_t)(b - k0) * sizeof(double);
      if ((e = cudaMemcpy2DAsync(Gt, w, Y + k0, (size_t)b * sizeof(double), w, n, cudaMemcpyDeviceToDevice, st)))
        return e;
      if ((e = cholqr2_dense(st, Gt, n, b - k0, 1e-14, ws))) return e;
      if ((e = cudaMemcpy2DAsync(Y + k0, (size_t)b * sizeof(double), Gt, w, w, n, cudaMemcpyDeviceToDevice, st)))
        return e;
    }
    // structure of the exact core: per-block K ranges for the two products
    int2 *krZ = nullptr, *krH = nullptr;
    double fZ = 1.0, fH = 1.0;
    if (shape && shape->k + shape->s == m && shape->k + shape->r == n && shape->r > 0) {
      const int nbZ = (int)cdiv(m, 64), nbH = (int)cdiv(n, 64);
      krZ = ws.alloc<int2>(nbZ);
      krH = ws.alloc<int2>(nbH);
      if (ws.err) return ws.err;
      ++g_launches;
      kr_plan_epoch_bump();  // new K ranges: the cached split plans of older ones are stale
      launch_k(core_kr_kernel, cdiv(std::max(nbZ, nbH), 128), 128, 0, st, shape->k, shape->r, shape->klist, m, n, krZ, nbZ, krH,
                                                                    nbH);
      if (g_prof) {  // nonzero fractions for the flop accounting (profiling pass only)
        std::vector<int2> hz(nbZ), hh(nbH);
        cudaMemcpyAsync(hz.data(), krZ, nbZ * sizeof(int2), cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(hh.data(), krH, nbH * sizeof(int2), cudaMemcpyDeviceToHost, st);
        if ((e = cudaStreamSynchronize(st))) return e;
        double az = 0.0, ah = 0.0;
        for (int q = 0; q < nbZ; ++q) az += (double)std::min<int64_t>(64, m - 64 * q) * (hz[q].y - hz[q].x);
        for (int q = 0; q < nbH; ++q) ah += (double)std::min<int64_t>(64, n - 64 * q) * (hh[q].y - hh[q].x);
        fZ = az / ((double)m * n);
        fH = ah / ((double)n * m);
      }
    }
    const int maxit = 120;
    int next_check = info->hint >= 3 ? std::min(info->hint, 40) : 4;
    // (theta_1 / theta_b)^2: conditioning gained per power step; before this update's first
    // check, the previous update's value (x2 margin) if the caller has one, else unknown
    double growth = info->growth > 0 ? 2.0 * info->growth : 1e30;
    int since_orth = 0;
    // Chebyshev acceleration: with c a lower bound of theta_b^2 (the b-th Ritz value of the
    // last check, or of the previous update's), the two steps between orthonormalisations apply
    // T_2(2H/c - I) = 2 (2H/c - I)^2 - I instead of H^2: the same two products, but an
    // eigenvalue lambda = r c of H gains T_2(2r - 1) = 2(2r-1)^2 - 1 over the damped part
    // [0, c] instead of r^2 (at the configs[1] ratio r ~ 9: 550 vs 81 per pair).
    double cheb_c = info->thb2;
    int pair_pos = 0;
    int last_check = -1;
    double* Y0 = ws.alloc<double>((size_t)n * b);
    if (ws.err) return ws.err;
    const Scratch::Mark loop_mark = ws.mark();
    for (int it = 1; it <= maxit; ++it) {
      ws.rewind(loop_mark);  // the previous iteration's Cholesky-QR / Jacobi workspaces
      if ((e = dgemm(st, m, b, n, 1.0, CMat{A, 1, lda}, CMat{Y, b, 1}, 0.0, Mat{Z, b, 1}, 0, krZ, fZ))) return e;
      if ((e = dgemm(st, n, b, m, 1.0, CMat{A, lda, 1}, CMat{Z, b, 1}, 0.0, Mat{HY, b, 1}, 0, krH, fH))) return e;
      info->iters = it;
      if (it == next_check) {
        // Rayleigh-Ritz by one-sided Jacobi on R_z^T, Z = A Y = Q_z R_z
        if ((e = cudaMemcpyAsync(Zq, Z, (size_t)m * b * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
        if ((e = cholqr2_r(st, Zq, m, b, 1e-14, Rz, ws))) return e;
        int sw = 0;
        bool conv = false;
        double tiny = 0.0;
        // K7's status is read with the residuals below (one synchronisation for both)
        const int* hinfo = nullptr;
        // (b > 128, K9: only the leading kk + 1 Ritz pairs must converge; the rest of U_x is a
        // basis of the remaining subspace, re-orthonormalised by the next Cholesky-QR)
        if ((e = jacobi_cols(st, Rz, b, b, b, b, th, Ux, b, &sw, &conv, ws, nullptr, &tiny, &hinfo,
                             b > 128 ? kk + 1 : 0)))
          return e;
        // Ritz vectors G = Y U_x and residuals ||H g_j - theta_j^2 g_j||, j <= kk
        if ((e = dgemm(st, n, kk + 1, b, 1.0, CMat{Y, b, 1}, CMat{Ux, 1, b}, 0.0, Mat{Gc, 1, n}, 0))) return e;
        if ((e = dgemm(st, n, kk + 1, b, 1.0, CMat{HY, b, 1}, CMat{Ux, 1, b}, 0.0, Mat{HU, 1, n}, 0))) return e;
        ++g_launches;
        launch_k(resid_kernel, kk + 1, 256, 0, st, HU, Gc, n, kk + 1, th, res);
        std::vector<double> hr(kk + 1), ht(b);
        cudaMemcpyAsync(hr.data(), res, (kk + 1) * sizeof(double), cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(ht.data(), th, b * sizeof(double), cudaMemcpyDeviceToHost, st);
        if ((e = cudaStreamSynchronize(st))) return e;
        if (hinfo) {
          sw = hinfo[0];
          conv = hinfo[1] != 0;
        }
        info->sweeps += sw;
        if (!conv) break;
        info->energy = h[0];
        // convergence of the leading kk Ritz pairs (the returned subspace); the (kk+1)-th Ritz
        // value — theta_{k+1}, reported, not used by the update — is accurate to second order in
        // its residual without its vector converging (rate (theta_{b+1} / theta_kk)^2 per step
        // instead of (theta_{b+1} / theta_{kk+1})^2: on the configs[3] cores 3 iterations, not 8)
        double rmax = 0.0;
        for (int j = 0; j < kk; ++j) rmax = std::max(rmax, hr[j]);
        const double scale = ht[0] * ht[0];
        if (trace)
          fprintf(stderr, "[core] m=%lld n=%lld b=%d it %d jacobi_sweeps %d max_resid/theta1^2 %.3e growth %.3g\n",
                  (long long)m, (long long)n, b, it, sw, scale > 0 ? rmax / scale : 0.0,
                  ht[b - 1] > 0 ? std::pow(ht[0] / ht[b - 1], 2.0) : 0.0);
        if (rmax <= 1e-12 * scale) {
          // iterations the next update of this stream probably needs: this count less the
          // margin the residual shows (80 % of it, at this check's convergence rate)
          {
            const double rho = (ht[kk - 1] > 0) ? std::pow(ht[b - 1] / ht[kk - 1], 2.0) : 0.5;
            double rate = rho;
            if (cheb_on && rho > 0 && rho < 0.5) {
              const double x = 2.0 / rho - 1.0;
              rate = 1.0 / std::sqrt(2.0 * x * x - 1.0);
            }
            int spare = 0;
            if (rmax > 0 && rate > 0 && rate < 0.999)
              spare = (int)std::floor(0.8 * std::log(1e-12 * scale / rmax) / std::log(1.0 / rate));
            info->hint_next = std::max(3, it - std::max(0, spare));
            if (trace)
              fprintf(stderr, "[core] converged at it %d: rho %.3f rate %.3f margin %.3g spare %d -> next first check %d\n",
                      it, rho, rate, 1e-12 * scale / rmax, spare, info->hint_next);
          }
          info->b_next = 0;
          if (trace)
            for (int bb = kk + 16; bb <= b; bb += 16)
              fprintf(stderr, "[core] ritz ratio (theta_%d / theta_%d)^2 = %.3e\n", bb, kk,
                      ht[kk - 1] > 0 ? std::pow(ht[bb - 1] / ht[kk - 1], 2.0) : 0.0);
          for (int bb = kk + 16; bb <= b && ht[kk - 1] > 0; bb += 16)
            if (std::pow(ht[bb - 1] / ht[kk - 1], 2.0) < 1e-3) {  // 1e-12 in four power steps
              info->b_next = bb;
              break;
            }
          const double tiny_k = 1e-14 * sqrt(info->energy) + 1e-300;
          cudaMemcpyAsync(theta, th, (kk + 1) * sizeof(double), cudaMemcpyDeviceToDevice, st);
          double* hn = (info->defer_theta_next && info->theta_next_dst) ? info->theta_next_dst : h + 1;
          cudaMemcpyAsync(hn, th + kk, sizeof(double), cudaMemcpyDeviceToHost, st);
          if ((e = cudaMemcpy2DAsync(G, ldg * sizeof(double), Gc, n * sizeof(double), n * sizeof(double), kk,
                                     cudaMemcpyDeviceToDevice, st)))
            return e;
          // F = Z U_x diag(1/theta)  (= A G diag(1/theta)), completed where theta ~ 0
          if ((e = dgemm(st, m, kk, b, 1.0, CMat{Z, b, 1}, CMat{Ux, 1, b}, 0.0, Mat{F, 1, ldf}, 0))) return e;
          dim3 grid(std::max<unsigned>(1, std::min<unsigned>(cdiv(m, 256), 64)), kk);
          g_launches += 2;
          launch_k(scale_cols_kernel, grid, 256, 0, st, F, ldf, m, kk, theta, tiny_k);
          launch_k(ident_perm_kernel, 1, 256, 0, st, perm, kk);
          launch_k(complete_kernel, 1, 256, 0, st, F, ldf, m, kk, perm, theta, tiny_k, nullptr);
          if (info->defer_theta_next) {  // read after the caller's next synchronisation
            info->theta_next_host = hn;
            info->converged = true;
            return cudaGetLastError();
          }
          if ((e = cudaStreamSynchronize(st))) return e;
          info->theta_next = h[1];
          info->converged = true;
          return cudaSuccess;
        }
        // not yet: rotate the basis onto the Ritz vectors (so the next Rayleigh-Ritz Jacobi
        // starts nearly diagonal) and predict the iterations left from the Ritz-value ratio
        // rho = (theta_b / theta_{kk+1})^2 per iteration
        if ((e = dgemm(st, n, b, b, 1.0, CMat{HY, b, 1}, CMat{Ux, 1, b}, 0.0, Mat{Z, b, 1}, 0))) return e;
        if ((e = cudaMemcpyAsync(HY, Z, (size_t)n * b * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
        const double rho = (ht[kk - 1] > 0) ? std::pow(ht[b - 1] / ht[kk - 1], 2.0) : 0.5;
        growth = ht[b - 1] > 0 ? std::pow(ht[0] / ht[b - 1], 2.0) : 1e30;
        info->growth = growth;
        cheb_c = ht[b - 1] * ht[b - 1];
        info->thb2 = cheb_c;
        // residual reduction per iteration: rho for power steps, T_2(2/rho - 1)^(-1/2) filtered
        double rate = rho;
        if (cheb_on && rho > 0 && rho < 0.5) {
          const double x = 2.0 / rho - 1.0;
          rate = 1.0 / std::sqrt(2.0 * x * x - 1.0);
        }
        int q = 3;
        if (rate > 0 && rate < 0.999 && rmax > 0) q = (int)std::ceil(std::log(0.3e-12 * scale / rmax) / std::log(rate));
        next_check = it + std::min(std::max(q, 1), 30);
        last_check = it;
      }
      // Y <- orth(A^T A Y): once a Rayleigh-Ritz check has shown the per-step growth
      // (theta_1 / theta_b)^2 <= 1e4, one Cholesky-QR pass keeps the basis well conditioned
      // for the next power step (orthogonality ~ eps growth^2); otherwise, and for the basis
      // entering a check, two passes (orthonormal to ~eps)
      // Chebyshev pair (see above) on the steps after an orthonormalisation, not across a check
      const bool cheb = cheb_on && cheb_c > 0 && it != last_check && it != next_check;
      bool rotated = false;
      if (cheb) {
        if (pair_pos == 0) {  // Y1 = (2/c) H Y0 - Y0, Y0 the orthonormal basis
          if ((e = mat_axpby(st, n, b, -1.0, CMat{Y, b, 1}, 2.0 / cheb_c, Mat{HY, b, 1}))) return e;
          // three-way rotation instead of a copy: Y0 keeps the basis, Y takes Y1
          double* fr = Y0;
          Y0 = Y;
          Y = HY;
          HY = fr;
          rotated = true;
          pair_pos = 1;
        } else {  // Y2 = (4/c) H Y1 - 2 Y1 - Y0
          if ((e = mat_axpby(st, n, b, -2.0, CMat{Y, b, 1}, 4.0 / cheb_c, Mat{HY, b, 1}))) return e;
          if ((e = mat_axpby(st, n, b, -1.0, CMat{Y0, b, 1}, 1.0, Mat{HY, b, 1}))) return e;
          pair_pos = 2;
        }
      }
      if (!rotated) std::swap(Y, HY);
      if (cheb_on && cheb_c > 0) {  // filtered mode: orthonormalise after every pair / check
        if (it + 1 != next_check && it != last_check && pair_pos == 1) continue;
        pair_pos = 0;
        since_orth = 0;
        const int passes = (it + 1 == next_check || growth > 1e4) ? 2 : 1;
        // orthonormal basis into HY's buffer (free: it holds the previous basis), then swapped
        if ((e = cholqr_dense(st, Y, n, b, 1e-14, passes, nullptr, ws, HY))) return e;
        std::swap(Y, HY);
        continue;
      }
      // once the growth per step is known to be small, every other step skips the pass
      // (two unnormalised steps raise the condition to growth^2 <= 2.5e7; one Cholesky-QR pass
      // then leaves a basis orthogonal to eps growth^4 <= 0.06, well conditioned for the
      // next power step)
      // generally: q = floor(log(2.5e7) / log(growth)) unnormalised steps between passes (cap 4)
      const int q = growth <= 1.0 ? 4 : std::max(1, std::min(4, (int)std::floor(std::log(2.5e7) / std::log(growth))));
      if (it + 1 != next_check && ++since_orth < q) continue;
      since_orth = 0;
      const int passes = (it + 1 == next_check || growth > 1e4) ? 2 : 1;
      if ((e = cholqr_dense(st, Y, n, b, 1e-14, passes, nullptr, ws))) return e;
    }
    if (trace) fprintf(stderr, "[core] subspace path did not converge in %d iterations: full Jacobi\n", info->iters);
  }
  // ---- direct path: one-sided Jacobi of A itself (tall A preconditioned by Cholesky-QR2)
  double* th_all = ws.alloc<double>(n);
  if (ws.err) return ws.err;
  int sw = 0;
  bool conv = false;
  double tiny = 0.0;
  if (m >= 2 * n && n >= 32) {
    info->path = 1;
    double* Ar = ws.alloc<double>((size_t)m * n);   // row-major copy of A
    double* R = ws.alloc<double>((size_t)n * n);
    double* Gu = ws.alloc<double>((size_t)n * kk);
    if (ws.err) return ws.err;
    if ((e = colmajor_to_rowmajor(st, A, lda, m, n, Ar, n))) return e;
    if ((e = cholqr2_r(st, Ar, m, n, 1e-14, R, ws))) return e;
    // A = Q R: the right singular vectors of A are the left ones of R^T (col-major = R row-major)
    if ((e = jacobi_cols(st, R, n, n, n, kk, th_all, Gu, n, &sw, &conv, ws, prof, &tiny, nullptr,
                         (int)std::min<int64_t>(n, kk + 1))))
      return e;
    info->sweeps += sw;
    if (!conv) return cudaSuccess;
    if ((e = cudaMemcpy2DAsync(G, ldg * sizeof(double), Gu, n * sizeof(double), n * sizeof(double), kk,
                               cudaMemcpyDeviceToDevice, st)))
      return e;
    info->energy = h[0];  // (jacobi_cols synchronised)
    if ((e = left_from_right(st, A, lda, m, n, kk, G, ldg, th_all, 1e-14 * sqrt(info->energy), F, ldf, ws))) return e;
  } else {
    info->path = 0;
    if ((e = jacobi_cols(st, A, lda, m, n, kk, th_all, F, ldf, &sw, &conv, ws, prof, &tiny, nullptr,
                         (int)std::min<int64_t>(n, kk + 1))))
      return e;
    info->sweeps += sw;
    if (!conv) return cudaSuccess;
    if ((e = right_from_left(st, A, lda, m, n, kk, F, ldf, th_all, tiny, G, ldg, ws))) return e;
  }
  const int nt = (int)std::min<int64_t>(n, kk + 1);
  cudaMemcpyAsync(theta, th_all, nt * sizeof(double), cudaMemcpyDeviceToDevice, st);
  h[1] = 0.0;
  if (n > kk) cudaMemcpyAsync(h + 1, th_all + kk, sizeof(double), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st))) return e;
  info->energy = h[0];
  info->theta_next = h[1];
  info->converged = true;
  return cudaSuccess;
}

}  // namespace tsvd
