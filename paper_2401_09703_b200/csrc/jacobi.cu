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

#include "ops.h"

namespace tsvd {

namespace {
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

__global__ void __launch_bounds__(JT) jacobi_round_kernel(double* __restrict__ W, int64_t ldw, int64_t m,
                                                          double* __restrict__ V, int64_t ldv, int64_t nv, int nb,
                                                          int round, double tol, const double* __restrict__ normA2,
                                                          int* __restrict__ counter) {
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
        if (fabs(gpq) > 1e-300 && fabs(gpq) > 1e-18 * fmax(fabs(gpp), fabs(gqq))) {
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
        const double mx = fmax(fabs(sm.G[r][r]), fabs(sm.G[c][c]));
        if (mx > 0) o = fmax(o, fabs(sm.G[r][c]) / mx);
      }
    }
    o = warp_max(o);
    if (lane == 0) sm.red[warp] = o;
    __syncthreads();
    if (tid == 0) {
      double oo = 0.0;
      for (int w = 0; w < 8; ++w) oo = fmax(oo, sm.red[w]);
      sm.flag = oo > 1e-17;
    }
    __syncthreads();
    if (!sm.flag) break;
  }

  // ---- 4. apply the rotation to the slab of W (m rows) and of V (nv rows), in place
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
  apply(V, ldv, nv);
}

__global__ void frob2_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n, double* out) {
  double s = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m * n; e += (int64_t)gridDim.x * blockDim.x) {
    const double x = A[(e / m) * lda + e % m];
    s = fma(x, x, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

__global__ void copy_pad_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n, double* __restrict__ W,
                                int64_t ldw, int64_t npad) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ldw * npad; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / ldw, i = e % ldw;
    W[e] = (i < m && j < n) ? A[j * lda + i] : 0.0;
  }
}

__global__ void eye_kernel(double* V, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x)
    V[e] = (e / n == e % n) ? 1.0 : 0.0;
}

__global__ void colnorm_kernel(const double* __restrict__ W, int64_t ldw, int64_t m, int64_t n, double* __restrict__ nrm) {
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

// F[:, j] = W[:, perm[j]] / sigma, G[:, j] = V[0:n, perm[j]], j < kk (col-major outputs)
__global__ void extract_kernel(const double* __restrict__ W, int64_t ldw, int64_t m, const double* __restrict__ V,
                               int64_t ldv, int64_t n, const int* __restrict__ perm, const double* __restrict__ nrm,
                               int kk, double tiny, double* __restrict__ F, int64_t ldf, double* __restrict__ G,
                               int64_t ldg, int* __restrict__ deficient) {
  const int j = blockIdx.y;
  const int pj = perm[j];
  const double sg = nrm[pj];
  const bool ok = sg > tiny;
  if (!ok && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(deficient, 1);
  const double inv = ok ? 1.0 / sg : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    F[j * ldf + i] = W[(int64_t)pj * ldw + i] * inv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    G[j * ldg + i] = V[(int64_t)pj * ldv + i];
}

// Orthonormal completion of the F columns whose singular value is ~0:
// for each such column, Gram-Schmidt (twice) a unit vector e_c against all other columns.
__global__ void __launch_bounds__(256) complete_kernel(double* F, int64_t ldf, int64_t m, int kk,
                                                       const int* __restrict__ perm, const double* __restrict__ nrm,
                                                       double tiny) {
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
}  // namespace

cudaError_t jacobi_svd(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, int kk, double* theta,
                       double* F, int64_t ldf, double* G, int64_t ldg, int* sweeps, bool* converged, Scratch& ws,
                       KProf* prof) {
  long long* launches = &g_launches;
  *sweeps = 0;
  *converged = false;
  if (n <= 0 || m <= 0) { *converged = true; return cudaSuccess; }
  if (m < n) return cudaErrorInvalidValue;
  const int64_t npad = ((n + JS - 1) / JS) * JS;
  const int nb = (int)(npad / JB);
  const int64_t ldw = ((m + 7) / 8) * 8;
  double* W = ws.alloc<double>((size_t)ldw * npad);
  double* V = ws.alloc<double>((size_t)npad * npad);
  double* nrm = ws.alloc<double>(npad + 1);
  int* counter = ws.alloc<int>(2);
  int* perm = ws.alloc<int>(16384);
  int* h_cnt = nullptr;
  if (ws.err) return ws.err;
  cudaError_t e;
  if ((e = cudaMallocHost(&h_cnt, 2 * sizeof(int)))) return e;
  const unsigned gbig = 148 * 8;
  copy_pad_kernel<<<gbig, 256, 0, st>>>(A, lda, m, n, W, ldw, npad);
  eye_kernel<<<gbig, 256, 0, st>>>(V, npad);
  double* normA2 = nrm + npad;
  cudaMemsetAsync(normA2, 0, sizeof(double), st);
  frob2_kernel<<<gbig, 256, 0, st>>>(W, ldw, ldw, npad, normA2);
  *launches += 3;
  static bool attr = false;
  const size_t smem = sizeof(JacobiSmem);
  if (!attr) {
    cudaFuncSetAttribute(jacobi_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const double tol = 1e-13;
  cudaEvent_t pe[2] = {nullptr, nullptr};
  if (prof) {
    cudaEventCreate(&pe[0]);
    cudaEventCreate(&pe[1]);
  }
  // algorithmic work of one round-kernel CTA: the slab Gram
  // (m x JS, symmetric: m JS (JS+1) flops, reads m JS 8 B) and, if the slab is not yet
  // orthogonal, the rotation of the W and V slabs (2 (m + npad) JS^2 flops, read + write).
  const double gram_flops = (double)m * JS * (JS + 1), gram_bytes = (double)m * JS * 8.0;
  const double rot_flops = 2.0 * (double)(m + npad) * JS * JS, rot_bytes = 2.0 * (double)(m + npad) * JS * 8.0;
  for (int sw = 0; sw < kMaxSweeps; ++sw) {
    cudaMemsetAsync(counter, 0, sizeof(int), st);
    if (prof) cudaEventRecord(pe[0], st);
    for (int r = 0; r < nb - 1; ++r) {
      jacobi_round_kernel<<<nb / 2, JT, smem, st>>>(W, ldw, m, V, npad, npad, nb, r, tol, normA2, counter);
      ++*launches;
    }
    if (prof) cudaEventRecord(pe[1], st);
    if ((e = cudaGetLastError())) break;
    cudaMemcpyAsync(h_cnt, counter, sizeof(int), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st))) break;
    if (prof) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, pe[0], pe[1]);
      prof->ms += ms;
      prof->launches += nb - 1;
      const double ctas = (double)(nb - 1) * (nb / 2);
      prof->flops += ctas * gram_flops + (double)h_cnt[0] * rot_flops;
      prof->bytes += ctas * gram_bytes + (double)h_cnt[0] * rot_bytes;
    }
    *sweeps = sw + 1;
    if (h_cnt[0] == 0) {
      *converged = true;
      break;
    }
  }
  if (e == cudaSuccess && *converged) {
    colnorm_kernel<<<cdiv(npad * 32, 256), 256, 0, st>>>(W, ldw, m, npad, nrm);
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
      sort_desc_kernel<<<1, 1024, ssm, st>>>(nrm, npad, p2, perm, theta, n);
      // tiny: singular values below 1e-14 ||K||_F are treated as exact zeros
      double h_norm2 = 0.0;
      cudaMemcpyAsync(&h_cnt[1], counter, sizeof(int), cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(&h_norm2, normA2, sizeof(double), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const double tiny = 1e-14 * sqrt(h_norm2) + 1e-300;
      cudaMemsetAsync(counter + 1, 0, sizeof(int), st);
      dim3 grid(std::max<unsigned>(1, std::min<unsigned>(cdiv(std::max(m, n), 256), 64)), kk);
      extract_kernel<<<grid, 256, 0, st>>>(W, ldw, m, V, npad, n, perm, nrm, kk, tiny, F, ldf, G, ldg, counter + 1);
      cudaMemcpyAsync(&h_cnt[1], counter + 1, sizeof(int), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      if (h_cnt[1] > 0) complete_kernel<<<1, 256, 0, st>>>(F, ldf, m, kk, perm, nrm, tiny);
      *launches += 4;
      e = cudaGetLastError();
    }
  }
  cudaFreeHost(h_cnt);
  if (pe[0]) cudaEventDestroy(pe[0]);
  if (pe[1]) cudaEventDestroy(pe[1]);
  return e;
}

}  // namespace tsvd
