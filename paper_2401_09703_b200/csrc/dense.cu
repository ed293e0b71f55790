// dense.cu — the s x s / k x k dense steps of the update (FP64).
//
//   K5 chol_deflate   Alg 2 realised as a blocked right-looking
//                     Cholesky of the SV-LCOV Gram E E^T - C0^T C0 (Lemma 2),
//                     with the deflation reading of Alg 2's unguarded α (R8/R9).
//   K6 trsm_upper     Y = R^{-1} X over the kept pivots (Eq (5) P:326 needs B F[k:] with
//                     B = E R^{-1}; the paper's C = C0 R^{-1} is never formed).
//   K15 inverse_gj    the inverse of the NEW multiplier (Eq (5), Alg 9 lines 4/7,
//                     DESIGN.md R7) and its 1-norm condition number (MII test, R18).
//   K11 materialize   X' <- X' M in place (reset of PAPER.md:349-351), DMMA.
//   core formation    Alg 9 line 2 (read as [Σ,0; E_r V_k, R^T], R1) and
//                     Alg 4 line 3.
#include <algorithm>
#include <cfloat>

#include <cooperative_groups.h>

#include "ops.h"
#include "potrf.cuh"

namespace tsvd {

namespace {
constexpr int CNB = 64;  // Cholesky / TRSM panel width

// Unblocked Cholesky with deflation of the nb x nb (nb <= 64) diagonal block at (p, p),
// outer-product order.  Fixed 2-D ownership: thread t updates column t % 64 at rows
// t / 64 + 4q (16 independent elements), so each pivot costs three barriers and 16
// independent FMAs per thread (no index divisions, no serial per-thread chains).
__global__ void __launch_bounds__(256) chol_panel_factor(double* G, int64_t s, int64_t p, int nb,
                                                         const double* __restrict__ enorm2, double tau,
                                                         int32_t* __restrict__ keep, int64_t pp, int nbp) {
  pdl_begin();
  // fused look-ahead: when pp >= 0 the previous panel's contribution (rows pp..pp+nbp of R)
  // to this diagonal block is subtracted here instead of by a separate GEMM
  extern __shared__ double dsm_pf[];
  double (*A)[CNB + 1] = reinterpret_cast<double (*)[CNB + 1]>(dsm_pf);
  double (*B)[CNB + 1] = reinterpret_cast<double (*)[CNB + 1]>(dsm_pf + CNB * (CNB + 1));
  __shared__ double en_s[CNB];
  __shared__ int kp_s;
  __shared__ double rinv_s;
  const int tid = threadIdx.x;
  const int c = tid & (CNB - 1), r0 = tid >> 6;  // column, first row (rows r0 + 4q)
  for (int e = tid; e < CNB * CNB; e += blockDim.x) {
    const int r = e >> 6, cc = e & (CNB - 1);
    A[r][cc] = (r < nb && cc < nb && cc >= r) ? G[(p + r) * s + p + cc] : 0.0;
    if (pp >= 0) B[r][cc] = (r < nbp && cc < nb) ? G[(pp + r) * s + p + cc] : 0.0;
  }
  __syncthreads();
  if (pp >= 0) {  // A -= B^T B on the DMMA pipe: 36 upper 8x8 tiles over 8 warps
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    for (int tile = warp; tile < 64; tile += 8) {
      const int tr = tile >> 3, tc = tile & 7;
      if (tr > tc) continue;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll 4
      for (int kk = 0; kk < CNB; kk += 4) dmma8x8x4(c0, c1, B[kk + t][tr * 8 + g], B[kk + t][tc * 8 + g]);
      const int r = tr * 8 + g, cc = tc * 8 + 2 * t;
      if (r <= cc) A[r][cc] -= c0;
      if (r <= cc + 1) A[r][cc + 1] -= c1;
    }
    __syncthreads();
  }
  if (tid < nb) en_s[tid] = enorm2[p + tid];
  __syncthreads();
  for (int i = 0; i < nb; ++i) {
    if (tid == 0) {
      const double en = en_s[i], d = A[i][i];
      const int kp = !(en == 0.0 || d <= tau * en);
      kp_s = kp;
      keep[p + i] = kp;
      const double r = kp ? sqrt(d) : 0.0;
      A[i][i] = r;
      rinv_s = kp ? 1.0 / r : 0.0;
    }
    __syncthreads();
    const int kp = kp_s;
    if (tid > i && tid < nb) A[i][tid] *= rinv_s;  // one division per pivot, not per element
    __syncthreads();
    if (kp && c > i && c < nb) {
      const double ric = A[i][c];
#pragma unroll
      for (int q = 0; q < CNB / 4; ++q) {
        const int r = r0 + 4 * q;
        if (r > i && r <= c) A[r][c] -= A[i][r] * ric;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int r = e / nb, cc = e % nb;
    G[(p + r) * s + p + cc] = (cc >= r) ? A[r][cc] : 0.0;
  }
}

// Cholesky with deflation of a small l x l Gram (l <= 128) and the inverse of its factor in
// one CTA of 1024 threads — the Cholesky-QR passes of the core reduction run this instead of
// the ~15 launches of the blocked path.  Iterative blocked algorithm on a 128 x 128 padded
// matrix (rows / columns >= l are an identity that never couples to the real block), 16-wide
// panels:
//   factor:  per panel j: warp 0 factors the 16 x 16 diagonal block (outer-product order, the
//            deflation test of DESIGN.md R8 on the current Schur diagonal), one thread per
//            column solves the panel's row block, and all 32 warps apply the rank-16
//            trailing update as 8 x 8 DMMA tiles (mma.sync m8n8k4 f64);
//   inverse: the eight 16 x 16 diagonal inverses in parallel (one warp each), then block
//            back substitution T[i,:] = Tii (I[i,:] - sum_{q>i} R_iq T[q,:]) for i = 7..0,
//            every step a set of DMMA tiles.
// T = R^+ is the inverse on the kept pivots (zero rows / columns for deflated ones) — what
// the right-side substitution X R^{-1} of trsm_right_upper applies.  Shared layout (one
// 128 x 132 array, 135 KB): R upper (diagonal included); T's strict upper triangle stored
// transposed in the strict lower triangle, T's diagonal in tdiag.
constexpr int CSMALL = 128;
constexpr int CLD = CSMALL + 4;  // pitch = 4 (mod 16) doubles: conflict-free 8x4 / 4x8 fragments
constexpr int CPW = 16;          // panel width

__global__ void __launch_bounds__(1024) chol_inv_small_kernel(double* G, int l, const double* __restrict__ enorm2,
                                                              double tau, int32_t* __restrict__ keep,
                                                              double* __restrict__ T) {
  pdl_begin();
  extern __shared__ double smem_ci[];
  double* A = smem_ci;                  // CSMALL x CLD: R (upper) | T^T (strict lower)
  __shared__ double rinv[CSMALL];
  __shared__ double tdiag[CSMALL];
#define TGET(r, c) ((r) < (c) ? A[(c) * CLD + (r)] : ((r) == (c) ? tdiag[(r)] : 0.0))
#define TSET(r, c, v)                   \
  do {                                  \
    if ((r) < (c)) A[(c) * CLD + (r)] = (v); \
    else if ((r) == (c)) tdiag[(r)] = (v);   \
  } while (0)
  __shared__ double en_s[CSMALL];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int LP = (l + CPW - 1) / CPW * CPW;  // the blocked algorithm runs on l rounded up to 16
  for (int e = tid; e < CSMALL * CSMALL; e += blockDim.x) {
    const int r = e >> 7, c = e & (CSMALL - 1);
    double v;
    if (r < l && c < l) v = (c >= r) ? G[(int64_t)r * l + c] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;  // identity padding
    A[r * CLD + c] = v;
  }
  __syncthreads();
  if (tid < CSMALL) en_s[tid] = tid < l ? (enorm2 ? enorm2[tid] : A[tid * CLD + tid]) : 1.0;
  __syncthreads();
  // ------------------------------------------------------------------ factorisation
  for (int j0 = 0; j0 < LP; j0 += CPW) {
    const int j1 = j0 + CPW;
    if (warp == 0) {  // (a) diagonal block, 16 pivots
      for (int i = j0; i < j1; ++i) {
        if (lane == 0) {
          const double d = A[i * CLD + i];
          const bool real = i < l;
          const int kp = real && !(en_s[i] == 0.0 || d <= tau * en_s[i]);
          if (real) keep[i] = kp;
          const double sq = sqrt(kp ? d : 1.0), inv = 1.0 / sq;  // unconditional: no branch
          const double r = kp ? sq : (real ? 0.0 : 1.0);
          A[i * CLD + i] = r;
          rinv[i] = kp ? inv : (real ? 0.0 : 1.0);
        }
        __syncwarp();
        const double ri = rinv[i];
        if (lane > i - j0 && lane < CPW) A[i * CLD + j0 + lane] *= ri;
        __syncwarp();
        if (ri != 0.0) {
          // rank-1 update of the block's remaining upper triangle: (r, c) = lane / 16.., 8 each
          for (int e = lane; e < CPW * CPW; e += 32) {
            const int r = j0 + (e >> 4), c = j0 + (e & 15);
            if (r > i && c >= r) A[r * CLD + c] -= A[i * CLD + r] * A[i * CLD + c];
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (j1 < LP) {
      // (b) row block: R[j0:j1, c] = R_jj^{-T} A[j0:j1, c] for c >= j1, one thread per column
      if (tid < LP - j1) {
        const int c = j1 + tid;
        double x[CPW];
#pragma unroll
        for (int q = 0; q < CPW; ++q) {
          double v = A[(j0 + q) * CLD + c];
#pragma unroll
          for (int u = 0; u < q; ++u) v = fma(-A[(j0 + u) * CLD + j0 + q], x[u], v);
          x[q] = v * rinv[j0 + q];
          A[(j0 + q) * CLD + c] = x[q];
        }
      }
      __syncthreads();
      // (c) trailing update A[j1:, j1:] -= R[j0:j1, j1:]^T R[j0:j1, j1:]  (upper 8x8 tiles)
      const int nt = (LP - j1) / 8;
      for (int tile = warp; tile < nt * nt; tile += 32) {
        const int tr = tile / nt, tc = tile % nt;
        if (tr > tc) continue;
        const int r0 = j1 + tr * 8, c0 = j1 + tc * 8;
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < CPW; kk += 4)
          dmma8x8x4(acc0, acc1, A[(j0 + kk + t) * CLD + r0 + g], A[(j0 + kk + t) * CLD + c0 + g]);
        const int r = r0 + g, c = c0 + 2 * t;
        if (r <= c) A[r * CLD + c] -= acc0;
        if (r <= c + 1) A[r * CLD + c + 1] -= acc1;
      }
      __syncthreads();
    }
  }
  // write R (upper) back
  for (int e = tid; e < l * l; e += blockDim.x) {
    const int r = e / l, c = e % l;
    G[(int64_t)r * l + c] = (c >= r) ? A[r * CLD + c] : 0.0;
  }
  // ------------------------------------------------------------------ inverse
  // (1) diagonal 16 x 16 inverses, warp w < 8 takes block w; lane c < 16 owns column c
  if (warp < LP / CPW && lane < CPW) {
    const int o = warp * CPW, c = lane;
    double x[CPW];
#pragma unroll
    for (int q = CPW - 1; q >= 0; --q) {  // back substitution R_bb x = e_c
      double v = (q == c) ? 1.0 : 0.0;
#pragma unroll
      for (int u = q + 1; u < CPW; ++u) v = fma(-A[(o + q) * CLD + o + u], x[u], v);
      x[q] = (q <= c) ? v * rinv[o + q] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < CPW; ++q)
      if (q <= c) TSET(o + q, o + c, x[q]);
  }
  __syncthreads();
  // (2) block back substitution: rows of block i, columns > its diagonal block
  for (int bi = LP / CPW - 2; bi >= 0; --bi) {
    const int i0 = bi * CPW, i1 = i0 + CPW;
    // W = sum_{q >= i1} R[i0:i1, q] T[q, c] for c >= i1 (16 x (128 - i1)), in 8x8 tiles
    const int ntc = (LP - i1) / 8;
    double w0 = 0.0, w1 = 0.0;
    int myt = warp < 2 * ntc ? warp : -1;  // 2 row tiles x ntc column tiles <= 28 <= 32 warps
    if (myt >= 0) {
      const int tr = myt / ntc, tc = myt % ntc;
      const int r0 = i0 + tr * 8, c0 = i1 + tc * 8;
      for (int kk = i1; kk < c0 + 8; kk += 4)  // T[q, c] = 0 for q > c
        dmma8x8x4(w0, w1, A[(r0 + g) * CLD + kk + t], TGET(kk + t, c0 + g));
    }
    __syncthreads();
    if (myt >= 0) {  // stash -W in the T rows of block i (they are still zero there)
      const int tr = myt / ntc, tc = myt % ntc;
      TSET(i0 + tr * 8 + g, i1 + tc * 8 + 2 * t, -w0);
      TSET(i0 + tr * 8 + g, i1 + tc * 8 + 2 * t + 1, -w1);
    }
    __syncthreads();
    // T[i0:i1, c] = T_ii * (-W[:, c]) for c >= i1: 16 x 16 times 16 x (128 - i1)
    double v0 = 0.0, v1 = 0.0;
    if (myt >= 0) {
      const int tr = myt / ntc, tc = myt % ntc;
      const int r0 = tr * 8, c0 = i1 + tc * 8;
#pragma unroll
      for (int kk = 0; kk < CPW; kk += 4)
        dmma8x8x4(v0, v1, TGET(i0 + r0 + g, i0 + kk + t), TGET(i0 + kk + t, c0 + g));
    }
    __syncthreads();
    if (myt >= 0) {
      const int tr = myt / ntc, tc = myt % ntc;
      TSET(i0 + tr * 8 + g, i1 + tc * 8 + 2 * t, v0);
      TSET(i0 + tr * 8 + g, i1 + tc * 8 + 2 * t + 1, v1);
    }
    __syncthreads();
  }
  for (int e = tid; e < l * l; e += blockDim.x) {
    const int r = e / l, c = e % l;
    T[(int64_t)r * l + c] = TGET(r, c);
  }
#undef TGET
#undef TSET
}

// l <= 96: the same factor + inverse by the augmented [A | I] factorisation of potrf.cuh
// (register pivots, no separate back substitution), on N = l rounded up to 16.
template <int N>
__global__ void __launch_bounds__(512) chol_aug_small_kernel(double* G, int l, const double* __restrict__ enorm2,
                                                             double tau, int32_t* __restrict__ keep,
                                                             double* __restrict__ T) {
  pdl_begin();
  constexpr int ALDN = 2 * N + 4;
  extern __shared__ double sm_ca[];
  __shared__ double en_loc[N];
  double* A = sm_ca;
  const int tid = threadIdx.x;
  for (int e = tid; e < N * N; e += 512) {
    const int r = e / N, c = e - r * N;
    A[r * ALDN + c] = (r < l && c < l) ? (c >= r ? G[(int64_t)r * l + c] : 0.0) : (r == c ? 1.0 : 0.0);
    A[r * ALDN + N + c] = (r == c) ? 1.0 : 0.0;
  }
  if (tid < N) en_loc[tid] = tid < l ? (enorm2 ? enorm2[tid] : G[(int64_t)tid * l + tid]) : 1.0;
  __syncthreads();
  potrf_core_t<N, 512>(A, l, en_loc, tau, keep);
  for (int e = tid; e < l * l; e += 512) {
    const int r = e / l, c = e - r * l;
    G[e] = c >= r ? A[r * ALDN + c] : 0.0;
    T[e] = A[c * ALDN + N + r];  // T = Y^T = R^+ (upper)
  }
}

template <int N>
cudaError_t launch_chol_aug(cudaStream_t st, double* G, int l, const double* enorm2, double tau, int32_t* keep,
                            double* T) {
  const size_t smem = (size_t)N * (2 * N + 4) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(chol_aug_small_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  launch_k(chol_aug_small_kernel<N>, 1, 512, smem, st, G, l, enorm2, tau, keep, T);
  return cudaGetLastError();
}

// R[p:p+nb, j] = R_pp^{-T} G[p:p+nb, j] for the columns j in [c0, c1) (thread per column).
__global__ void __launch_bounds__(128) chol_panel_rows(double* G, int64_t s, int64_t p, int nb,
                                                       const int32_t* __restrict__ keep, int64_t c0, int64_t c1) {
  pdl_begin();
  __shared__ double R[CNB][CNB + 1];
  __shared__ int kp[CNB];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int i = e / nb, j = e % nb;
    R[i][j] = (j >= i) ? G[(p + i) * s + p + j] : 0.0;
  }
  for (int i = threadIdx.x; i < nb; i += blockDim.x) kp[i] = keep[p + i];
  __syncthreads();
  const int64_t j = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= c1) return;
  double x[CNB];
#pragma unroll
  for (int i = 0; i < CNB; ++i) {
    if (i < nb) {
      double g = G[(p + i) * s + j];
#pragma unroll
      for (int l = 0; l < i; ++l) g -= R[l][i] * x[l];
      x[i] = kp[i] ? g / R[i][i] : 0.0;
      G[(p + i) * s + j] = x[i];
    }
  }
}

// Triangular solves with the nb x nb (nb <= 64) upper block R (at (p, p) of a row-major
// matrix, ld ldr, kept pivots only) for the columns [c0, c1) of the row block X[p:p+nb, :]
// (ld ldx), in place: FORWARD solves R^T x = b (Cholesky panel rows), else R x = b
// (back substitution).  One warp per column: lane l holds rows l and l + 32; each of the nb
// sequential steps finalises one unknown and broadcasts it with a shuffle.
template <bool FORWARD>
__global__ void __launch_bounds__(256) tri_solve_warp_kernel(const double* __restrict__ R, int64_t ldr, int64_t p,
                                                             int nb, const int32_t* __restrict__ keep, double* X,
                                                             int64_t ldx, int64_t c0, int64_t c1, int64_t pp = -1,
                                                             int nbp = 0) {
  pdl_begin();
  // pp >= 0 (forward only): first subtract the previous panel's contribution
  // X[p:p+nb, col] -= R[pp:pp+nbp, p:p+nb]^T R[pp:pp+nbp, col] (the fused look-ahead update)
  extern __shared__ double dsm_ts[];
  double (*Rs)[CNB + 1] = reinterpret_cast<double (*)[CNB + 1]>(dsm_ts);
  double (*Bs)[CNB + 1] = reinterpret_cast<double (*)[CNB + 1]>(dsm_ts + CNB * (CNB + 1));
  __shared__ double rinv[CNB];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    Rs[i][j] = (j >= i) ? R[(p + i) * ldr + p + j] : 0.0;
  }
  if (pp >= 0)
    for (int e = threadIdx.x; e < nbp * nb; e += blockDim.x) {
      const int q = e / nb, j = e % nb;
      Bs[q][j] = R[(pp + q) * ldr + p + j];
    }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x) rinv[i] = keep[p + i] ? 1.0 / Rs[i][i] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t col0 = c0 + (int64_t)blockIdx.x * 8;
  const int64_t col = col0 + warp;
  double xa, xb;
  if (FORWARD && pp >= 0) {
    // X[p:p+nb, col0:col0+8] -= Bs^T Y with Y = R[pp:pp+nbp, col0:col0+8]: one 8x8 DMMA tile
    // per warp (rows warp*8..), through a shared tile (coalesced 64-byte row loads)
    __shared__ double Ys[CNB][8];
    __shared__ double Xs[CNB][9];
    for (int e = threadIdx.x; e < CNB * 8; e += blockDim.x) {
      const int r = e >> 3, cc = e & 7;
      const bool inc = col0 + cc < c1;
      Ys[r][cc] = (r < nbp && inc) ? R[(pp + r) * ldr + col0 + cc] : 0.0;
      Xs[r][cc] = (r < nb && inc) ? X[(p + r) * ldx + col0 + cc] : 0.0;
    }
    __syncthreads();
    {
      const int g = lane >> 2, t = lane & 3;
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 4
      for (int kk = 0; kk < CNB; kk += 4)
        dmma8x8x4(acc0, acc1, (kk + t < nbp) ? Bs[kk + t][warp * 8 + g] : 0.0, Ys[kk + t][g]);
      Xs[warp * 8 + g][2 * t] -= acc0;
      Xs[warp * 8 + g][2 * t + 1] -= acc1;
    }
    __syncthreads();
    if (col >= c1) return;
    xa = lane < nb ? Xs[lane][warp] : 0.0;
    xb = lane + 32 < nb ? Xs[lane + 32][warp] : 0.0;
  } else {
    if (col >= c1) return;
    const double* x0 = X + p * ldx + col;
    xa = lane < nb ? x0[(int64_t)lane * ldx] : 0.0;
    xb = lane + 32 < nb ? x0[(int64_t)(lane + 32) * ldx] : 0.0;
  }
  double* x = X + p * ldx + col;
  if (FORWARD) {
    for (int i = 0; i < nb; ++i) {
      const double xi = __shfl_sync(0xffffffffu, i < 32 ? xa : xb, i & 31) * rinv[i];
      if (lane == (i & 31)) {
        if (i < 32) xa = xi; else xb = xi;
      }
      if (lane > i) xa = fma(-Rs[i][lane], xi, xa);
      if (lane + 32 > i && lane + 32 < nb) xb = fma(-Rs[i][lane + 32], xi, xb);
    }
  } else {
    for (int i = nb - 1; i >= 0; --i) {
      const double xi = __shfl_sync(0xffffffffu, i < 32 ? xa : xb, i & 31) * rinv[i];
      if (lane == (i & 31)) {
        if (i < 32) xa = xi; else xb = xi;
      }
      if (lane < i) xa = fma(-Rs[lane][i], xi, xa);
      if (lane + 32 < i) xb = fma(-Rs[lane + 32][i], xi, xb);
    }
  }
  if (lane < nb) x[(int64_t)lane * ldx] = xa;
  if (lane + 32 < nb) x[(int64_t)(lane + 32) * ldx] = xb;
}

__global__ void zero_lower_kernel(double* G, int64_t s) {
  pdl_begin();
  const int64_t i = blockIdx.y, j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t row = i; row < s; row += gridDim.y)
    for (int64_t j = j0; j < row && j < s; j += (int64_t)gridDim.x * blockDim.x) G[row * s + j] = 0.0;
}

// Backward substitution on the nb x nb diagonal block for every RHS column c.
__global__ void __launch_bounds__(64) trsm_diag_kernel(const double* __restrict__ Rm, int64_t s, int64_t p, int nb,
                                                       const int32_t* __restrict__ keep, double* X, int k) {
  pdl_begin();
  __shared__ double R[CNB][CNB + 1];
  __shared__ int kp[CNB];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int i = e / nb, j = e % nb;
    R[i][j] = (j >= i) ? Rm[(p + i) * s + p + j] : 0.0;
  }
  for (int i = threadIdx.x; i < nb; i += blockDim.x) kp[i] = keep[p + i];
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k) return;
  double x[CNB];
#pragma unroll
  for (int ii = CNB - 1; ii >= 0; --ii) {
    if (ii < nb) {
      double g = X[(p + ii) * k + c];
#pragma unroll
      for (int l = ii + 1; l < CNB; ++l)
        if (l < nb) g -= R[ii][l] * x[l];
      x[ii] = kp[ii] ? g / R[ii][ii] : 0.0;
      X[(p + ii) * k + c] = x[ii];
    }
  }
}

// Gauss-Jordan inverse with partial pivoting of aug = [M | I] (k x 2k, global scratch).
__global__ void __launch_bounds__(1024) gj_kernel(const double* __restrict__ M, int k, double* aug,
                                                  double* __restrict__ Minv, double* __restrict__ cond) {
  pdl_begin();
  extern __shared__ double fac[];  // k factors
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int piv;
  __shared__ double pval;
  __shared__ int singular;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5;
  const int k2 = 2 * k;
  for (int e = tid; e < k * k2; e += nt) {
    int i = e / k2, j = e % k2;
    aug[e] = (j < k) ? M[i * k + j] : (j - k == i ? 1.0 : 0.0);
  }
  if (tid == 0) singular = 0;
  // ||M||_1 = max column abs sum
  double cmax = 0.0;
  for (int j = tid; j < k; j += nt) {
    double a = 0.0;
    for (int i = 0; i < k; ++i) a += fabs(M[i * k + j]);
    cmax = fmax(cmax, a);
  }
  cmax = warp_max(cmax);
  if (lane == 0) red_v[w] = cmax;
  __syncthreads();
  double norm1 = 0.0;
  for (int i = 0; i < (nt + 31) / 32; ++i) norm1 = fmax(norm1, red_v[i]);
  __syncthreads();
  for (int c = 0; c < k; ++c) {
    // pivot search over rows c..k-1 of column c
    double best = -1.0;
    int bi = c;
    for (int r = c + tid; r < k; r += nt) {
      double a = fabs(aug[r * k2 + c]);
      if (a > best) { best = a; bi = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) { red_v[w] = best; red_i[w] = bi; }
    __syncthreads();
    if (tid == 0) {
      double b = -1.0;
      int ii = c;
      for (int q = 0; q < (nt + 31) / 32; ++q)
        if (red_v[q] > b || (red_v[q] == b && red_i[q] < ii)) { b = red_v[q]; ii = red_i[q]; }
      piv = ii;
      pval = aug[ii * k2 + c];
      if (!(b > 0.0)) singular = 1;
    }
    __syncthreads();
    if (singular) break;
    // swap rows c and piv, scale row c
    const double inv = 1.0 / pval;
    for (int j = tid; j < k2; j += nt) {
      double a = aug[c * k2 + j], b = aug[piv * k2 + j];
      if (piv != c) aug[piv * k2 + j] = a;
      aug[c * k2 + j] = b * inv;
    }
    __syncthreads();
    for (int r = tid; r < k; r += nt) fac[r] = (r == c) ? 0.0 : aug[r * k2 + c];
    __syncthreads();
    for (int e = tid; e < k * k2; e += nt) {
      int r = e / k2, j = e % k2;
      double f = fac[r];
      if (f != 0.0) aug[e] -= f * aug[c * k2 + j];
    }
    __syncthreads();
  }
  if (singular) {
    if (tid == 0) *cond = INFINITY;
    return;
  }
  double imax = 0.0;
  for (int j = tid; j < k; j += nt) {
    double a = 0.0;
    for (int i = 0; i < k; ++i) {
      double x = aug[i * k2 + k + j];
      Minv[i * k + j] = x;
      a += fabs(x);
    }
    imax = fmax(imax, a);
  }
  imax = warp_max(imax);
  __syncthreads();
  if (lane == 0) red_v[w] = imax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < (nt + 31) / 32; ++i) m = fmax(m, red_v[i]);
    *cond = norm1 * m;
  }
}

// The same Gauss-Jordan inverse (identical pivot choices and operation order per element) with
// [M | I] resident in shared memory, for k <= GJ_SMEM_K: the per-column passes are shared-memory
// sweeps with a fixed thread -> (row, column) map instead of global read-modify-writes.
constexpr int GJ_SMEM_K = 96;
__global__ void __launch_bounds__(1024) gj_smem_kernel(const double* __restrict__ M, int k, double* __restrict__ Minv,
                                                       double* __restrict__ cond) {
  pdl_begin();
  extern __shared__ double aug_s[];  // k x (2k + 1)
  __shared__ double fac[GJ_SMEM_K];
  __shared__ double red_v[32];
  __shared__ int piv;
  __shared__ double pval;
  __shared__ int singular;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5;
  const int k2 = 2 * k, ld = k2 + 1;
  for (int e = tid; e < k * k2; e += nt) {
    const int i = e / k2, j = e - i * k2;
    aug_s[i * ld + j] = (j < k) ? M[i * k + j] : (j - k == i ? 1.0 : 0.0);
  }
  if (tid == 0) singular = 0;
  double cmax = 0.0;
  for (int j = tid; j < k; j += nt) {
    double a = 0.0;
    for (int i = 0; i < k; ++i) a += fabs(M[i * k + j]);
    cmax = fmax(cmax, a);
  }
  cmax = warp_max(cmax);
  if (lane == 0) red_v[w] = cmax;
  __syncthreads();
  double norm1 = 0.0;
  for (int i = 0; i < (nt + 31) / 32; ++i) norm1 = fmax(norm1, red_v[i]);
  // fixed map: column j = tid % k2, rows tid / k2 + q * rstep
  const int jj = tid % k2, r0 = tid / k2, rstep = nt / k2;
  const bool active = r0 < rstep;
  for (int c = 0; c < k; ++c) {
    if (w == 0) {  // pivot search (first maximum, as gj_kernel)
      double best = -1.0;
      int bi = c;
      for (int r = c + lane; r < k; r += 32) {
        const double a = fabs(aug_s[r * ld + c]);
        if (a > best) { best = a; bi = r; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) {
        piv = bi;
        pval = 1.0 / aug_s[bi * ld + c];  // the reciprocal once, not in all 1024 threads
        if (!(best > 0.0)) singular = 1;
      }
    }
    __syncthreads();
    if (singular) break;
    const int pr = piv;
    const double inv = pval;
    for (int j = tid; j < k2; j += nt) {
      const double a = aug_s[c * ld + j], b = aug_s[pr * ld + j];
      if (pr != c) aug_s[pr * ld + j] = a;
      aug_s[c * ld + j] = b * inv;
    }
    __syncthreads();
    for (int r = tid; r < k; r += nt) fac[r] = (r == c) ? 0.0 : aug_s[r * ld + c];
    __syncthreads();
    if (active) {
      // eight rows at a time: all loads, then the fmas and stores — a row at a time the
      // compiler cannot move the next row's load above this row's store (same shared array),
      // and every update paid the full load -> fma -> store latency (~140 cycles)
      const double pc = aug_s[c * ld + jj];
      for (int r1 = r0; r1 < k; r1 += 8 * rstep) {
        double f[8], x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int r = r1 + u * rstep;
          f[u] = r < k ? fac[r] : 0.0;
          x[u] = r < k ? aug_s[r * ld + jj] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int r = r1 + u * rstep;
          if (r < k && f[u] != 0.0) aug_s[r * ld + jj] = x[u] - f[u] * pc;
        }
      }
    }
    __syncthreads();
  }
  if (singular) {
    if (tid == 0) *cond = INFINITY;
    return;
  }
  for (int e = tid; e < k * k; e += nt) {
    const int i = e / k, j = e - i * k;
    Minv[e] = aug_s[i * ld + k + j];
  }
  double imax = 0.0;
  for (int j = tid; j < k; j += nt) {
    double a = 0.0;
    for (int i = 0; i < k; ++i) a += fabs(aug_s[i * ld + k + j]);
    imax = fmax(imax, a);
  }
  imax = warp_max(imax);
  __syncthreads();
  if (lane == 0) red_v[w] = imax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < (nt + 31) / 32; ++i) m = fmax(m, red_v[i]);
    *cond = norm1 * m;
  }
}

// Blocked in-place Gauss-Jordan with partial pivoting for k <= 128, one CTA, the k x k matrix
// (rounded up to KP = 16 m with an identity pad) in shared memory.  Per panel of 16 columns:
//   (P) the 16 pivot steps on the panel's columns only: warp 0 searches the pivot (first
//       maximum over rows >= c), the full rows c and p are interchanged, the pivot row's panel
//       part is scaled (its pivot entry becomes 1 / pivot) and every other row's panel part
//       updated, column c <- -f / pivot (the in-place elimination of gj_inplace_kernel,
//       restricted to 16 columns);
//   (U) the other KP - 16 columns in one rank-16 DMMA product: with T = the panel's 16 pivot
//       rows there (interchanges applied, not yet transformed) and N = the transformed panel,
//       A[r][j] <- [r not a pivot row] A[r][j] + sum_q N[r][q] T[q][j] — the block form of the
//       same 16 elimination steps (A11^-1 A12 on the pivot rows, A22 - A21 A11^-1 A12 elsewhere).
// The unblocked variants moved the whole k x k matrix through shared memory (or registers) at
// every pivot and were instruction-bound: 346 us at k = 128, twice per configs[3] update.
constexpr int GJB_K = 128, GJB_LD = GJB_K + 4;  // pitch 4 (mod 16) doubles: conflict-free A and B fragments
__global__ void __launch_bounds__(1024) gj_blk_kernel(const double* __restrict__ M, int k, double* __restrict__ Minv,
                                                      double* __restrict__ cond) {
  pdl_begin();
  extern __shared__ double gjb_sm[];
  double* A = gjb_sm;                         // KP x GJB_LD
  double* Tb = A + GJB_K * GJB_LD;            // 16 x GJB_LD: the panel's pivot rows (other columns)
  __shared__ double fcol[GJB_K];              // column c after the interchange (the multipliers)
  __shared__ double prow[16], crow[16];       // panel parts of old rows p and c
  __shared__ double red_v[32];
  __shared__ int perm_s[GJB_K], src_s[GJB_K];
  __shared__ int piv_s, sing_s;
  __shared__ double inv_s;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int KP = (k + 15) & ~15;
  for (int e = tid; e < KP * KP; e += 1024) {
    const int r = e / KP, c = e - r * KP;
    A[r * GJB_LD + c] = (r < k && c < k) ? M[r * k + c] : (r == c ? 1.0 : 0.0);
  }
  if (tid == 0) sing_s = 0;
  __syncthreads();
  // ||M||_1
  double cmax = 0.0;
  if (tid < k) {
    double cs = 0.0;
    for (int r = 0; r < k; ++r) cs += fabs(A[r * GJB_LD + tid]);
    cmax = cs;
  }
  cmax = warp_max(cmax);
  if (lane == 0) red_v[w] = cmax;
  __syncthreads();
  double norm1 = 0.0;
  for (int q = 0; q < 32; ++q) norm1 = fmax(norm1, red_v[q]);
  const int er = tid >> 4, ej = tid & 15;  // panel element (er, ej) and (er + 64, ej)
  for (int c0 = 0; c0 < KP; c0 += 16) {
    // ---------------------------------------------------------------- (P) panel steps
    for (int c = c0; c < c0 + 16; ++c) {
      if (w == 0) {
        double best = -1.0;
        int bi = KP;
        for (int r = c + lane; r < KP; r += 32) {
          const double a = fabs(A[r * GJB_LD + c]);
          if (a > best) { best = a; bi = r; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) {
          piv_s = bi;
          perm_s[c] = bi;
          if (!(best > 0.0)) sing_s = 1;
        }
      }
      __syncthreads();
      if (sing_s) break;
      const int p = piv_s;
      // stage: panel parts of rows p and c, column c with the interchange applied, 1 / pivot;
      // interchange rows c and p outside the panel (not read until (U))
      if (tid < 16) {
        prow[tid] = A[p * GJB_LD + c0 + tid];
        crow[tid] = A[c * GJB_LD + c0 + tid];
      } else if (tid >= 32 && tid < 32 + KP) {
        const int r = tid - 32;
        fcol[r] = A[(r == c ? p : (r == p ? c : r)) * GJB_LD + c];
      } else if (tid >= 256 && tid < 256 + KP && p != c) {
        const int j = tid - 256;
        if (j < c0 || j >= c0 + 16) {
          const double x = A[c * GJB_LD + j];
          A[c * GJB_LD + j] = A[p * GJB_LD + j];
          A[p * GJB_LD + j] = x;
        }
      } else if (tid == 1023) {
        inv_s = 1.0 / A[p * GJB_LD + c];
      }
      __syncthreads();
      const double inv = inv_s;
      const int jc = c - c0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = er + 64 * h;
        if (r >= KP) continue;
        const double pr = (ej == jc ? 1.0 : prow[ej]) * inv;  // the new row c
        double v;
        if (r == c) {
          v = pr;
        } else {
          const double f = fcol[r];
          const double x = (r == p) ? crow[ej] : A[r * GJB_LD + c0 + ej];
          v = (ej == jc) ? -f * inv : ((f != 0.0) ? x - f * pr : x);
        }
        A[r * GJB_LD + c0 + ej] = v;
      }
      __syncthreads();
    }
    if (sing_s) break;
    if (KP == 16) break;
    // ---------------------------------------------------------------- (U) rank-16 update
    for (int e = tid; e < 16 * KP; e += 1024) {
      const int q = e / KP, j = e - q * KP;
      Tb[q * GJB_LD + j] = (j >= c0 && j < c0 + 16) ? 0.0 : A[(c0 + q) * GJB_LD + j];
    }
    __syncthreads();
    {
      const int nrt = KP / 8, nct = KP / 8;
      for (int tile = w; tile < nrt * nct; tile += 32) {
        const int tr = tile / nct, tc = tile - tr * nct;
        const int r0 = tr * 8, j0 = tc * 8;
        if (j0 >= c0 && j0 < c0 + 16) continue;  // the panel itself
        const bool pivrows = (r0 >= c0 && r0 < c0 + 16);
        double acc0 = pivrows ? 0.0 : A[(r0 + g) * GJB_LD + j0 + 2 * t];
        double acc1 = pivrows ? 0.0 : A[(r0 + g) * GJB_LD + j0 + 2 * t + 1];
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4)
          dmma8x8x4(acc0, acc1, A[(r0 + g) * GJB_LD + c0 + kk + t], Tb[(kk + t) * GJB_LD + j0 + g]);
        A[(r0 + g) * GJB_LD + j0 + 2 * t] = acc0;
        A[(r0 + g) * GJB_LD + j0 + 2 * t + 1] = acc1;
      }
    }
    __syncthreads();
  }
  if (sing_s) {
    if (tid == 0) *cond = INFINITY;
    return;
  }
  // (P M)^{-1} P = M^{-1}: the row interchanges, applied in reverse as column interchanges
  if (tid == 0) {
    for (int j = 0; j < KP; ++j) src_s[j] = j;
    for (int c = KP - 1; c >= 0; --c) {
      const int pp = perm_s[c];
      const int x = src_s[c];
      src_s[c] = src_s[pp];
      src_s[pp] = x;
    }
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += 1024) {
    const int r = e / k, j = e - r * k;
    Minv[e] = A[r * GJB_LD + src_s[j]];
  }
  double imax = 0.0;
  if (tid < k) {
    double cs = 0.0;
    const int sj = src_s[tid];
    for (int r = 0; r < k; ++r) cs += fabs(A[r * GJB_LD + sj]);
    imax = cs;
  }
  imax = warp_max(imax);
  __syncthreads();
  if (lane == 0) red_v[w] = imax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int q = 0; q < 32; ++q) m = fmax(m, red_v[q]);
    *cond = norm1 * m;
  }
}

// In-place Gauss-Jordan with partial pivoting for GJ_SMEM_K < k <= GJ_INPLACE_K: only the k x k
// matrix lives in shared memory (k = 128: 132 KB; [M | I] would need 263 KB) — column c of the
// working matrix holds column c of the inverse-so-far once it has been the pivot column (the
// classic in-place elimination); half the shared-memory traffic per pivot of the augmented form.
// The row interchanges become column interchanges of the result, undone at the store.
constexpr int GJ_INPLACE_K = 160;
__global__ void __launch_bounds__(1024) gj_inplace_kernel(const double* __restrict__ M, int k,
                                                          double* __restrict__ Minv, double* __restrict__ cond) {
  pdl_begin();
  extern __shared__ double A_s[];  // k x ld
  __shared__ double fac[GJ_INPLACE_K];
  __shared__ int perm_s[GJ_INPLACE_K];
  __shared__ int src_s[GJ_INPLACE_K];
  __shared__ double red_v[32];
  __shared__ int piv;
  __shared__ double pval;
  __shared__ int singular;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5;
  const int ld = k | 1;
  for (int e = tid; e < k * k; e += nt) {
    const int i = e / k, j = e - i * k;
    A_s[i * ld + j] = M[e];
  }
  if (tid == 0) singular = 0;
  double cmax = 0.0;
  for (int j = tid; j < k; j += nt) {
    double a = 0.0;
    for (int i = 0; i < k; ++i) a += fabs(M[i * k + j]);
    cmax = fmax(cmax, a);
  }
  cmax = warp_max(cmax);
  if (lane == 0) red_v[w] = cmax;
  __syncthreads();
  double norm1 = 0.0;
  for (int i = 0; i < (nt + 31) / 32; ++i) norm1 = fmax(norm1, red_v[i]);
  const int jj = tid % k, r0 = tid / k, rstep = nt / k;
  const bool active = r0 < rstep;
  for (int c = 0; c < k; ++c) {
    if (w == 0) {  // pivot search (first maximum)
      double best = -1.0;
      int bi = c;
      for (int r = c + lane; r < k; r += 32) {
        const double a = fabs(A_s[r * ld + c]);
        if (a > best) { best = a; bi = r; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) {
        piv = bi;
        perm_s[c] = bi;
        pval = 1.0 / A_s[bi * ld + c];
        if (!(best > 0.0)) singular = 1;
      }
    }
    __syncthreads();
    if (singular) break;
    const int pr = piv;
    const double inv = pval;
    // interchange rows c and pr; scale the pivot row (its pivot entry becomes 1 / pivot)
    for (int j = tid; j < k; j += nt) {
      const double a = A_s[c * ld + j], b = A_s[pr * ld + j];
      if (pr != c) A_s[pr * ld + j] = a;
      A_s[c * ld + j] = (j == c ? 1.0 : b) * inv;
    }
    __syncthreads();
    for (int r = tid; r < k; r += nt) fac[r] = (r == c) ? 0.0 : A_s[r * ld + c];
    __syncthreads();
    if (active) {
      const double pc = A_s[c * ld + jj];
      const bool colc = jj == c;  // the pivot column's old entries are eliminated (taken as 0)
      for (int r1 = r0; r1 < k; r1 += 8 * rstep) {
        double f[8], x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int r = r1 + u * rstep;
          f[u] = r < k ? fac[r] : 0.0;
          x[u] = (r < k && !colc) ? A_s[r * ld + jj] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int r = r1 + u * rstep;
          if (r < k && f[u] != 0.0) A_s[r * ld + jj] = x[u] - f[u] * pc;
        }
      }
    }
    __syncthreads();
  }
  if (singular) {
    if (tid == 0) *cond = INFINITY;
    return;
  }
  // (P M)^{-1} P = M^{-1}: the row interchanges, applied in reverse as column interchanges
  if (tid == 0) {
    for (int j = 0; j < k; ++j) src_s[j] = j;
    for (int c = k - 1; c >= 0; --c) {
      const int p = perm_s[c];
      const int t = src_s[c];
      src_s[c] = src_s[p];
      src_s[p] = t;
    }
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += nt) {
    const int i = e / k, j = e - i * k;
    Minv[e] = A_s[i * ld + src_s[j]];
  }
  double imax = 0.0;
  for (int j = tid; j < k; j += nt) {
    double a = 0.0;
    const int sj = src_s[j];
    for (int i = 0; i < k; ++i) a += fabs(A_s[i * ld + sj]);
    imax = fmax(imax, a);
  }
  imax = warp_max(imax);
  __syncthreads();
  if (lane == 0) red_v[w] = imax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < (nt + 31) / 32; ++i) m = fmax(m, red_v[i]);
    *cond = norm1 * m;
  }
}

// In-place Gauss-Jordan with partial pivoting for GJ_INPLACE_K < k <= 512 on one thread-block
// cluster: CTA q of C holds the columns [q w, q w + w) of the working matrix in shared memory
// (k = 256: C = 4, 133 KB each).  Per pivot step c the owner of column c searches the pivot
// (first maximum, as gj_inplace_kernel) and publishes the pivot row, 1 / pivot and the
// column's pre-interchange entries in a ping-pong slot of its shared memory; one cluster
// barrier; every CTA reads them by DSMEM and applies the interchange, the scaling of row c and
// the elimination to its own columns — the same operations per element as gj_inplace_kernel.
// The slots alternate, so the next step's owner never overwrites a slot another CTA may still
// be reading (readers finish before arriving at the next barrier).  (The single-CTA kernel on
// [M | I] in global memory took 8.2 ms at k = 256, twice per configs[4] update.)
namespace cgx = cooperative_groups;
__global__ void __launch_bounds__(1024) gj_cluster_kernel(const double* __restrict__ M, int k, int w,
                                                          double* __restrict__ Minv, double* __restrict__ cond) {
  pdl_begin();
  cgx::cluster_group cl = cgx::this_cluster();
  const int C = (int)cl.num_blocks(), q = (int)cl.block_rank();
  extern __shared__ double gsm[];
  const int ld = w | 1;
  double* A_s = gsm;                            // k x ld: columns c0 .. c0 + w - 1
  double* slot = A_s + (size_t)k * ld;          // 2 x (k + 2): pre-interchange column, then piv, 1/pivot
  double* fac = slot + 2 * (k + 2);             // k
  int* perm_s = reinterpret_cast<int*>(fac + k);  // k
  int* src_s = perm_s + k;                      // k
  __shared__ double red_v[32];
  __shared__ int sing_s;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wp = tid >> 5;
  const int c0 = q * w, wl = max(0, min(w, k - c0));
  for (int e = tid; e < k * wl; e += nt) {
    const int i = e / wl, j = e - i * wl;
    A_s[i * ld + j] = M[(int64_t)i * k + c0 + j];
  }
  double cmax = 0.0;  // ||M||_1 over this CTA's columns
  for (int j = tid; j < wl; j += nt) {
    double a = 0.0;
    for (int i = 0; i < k; ++i) a += fabs(M[(int64_t)i * k + c0 + j]);
    cmax = fmax(cmax, a);
  }
  cmax = warp_max(cmax);
  if (lane == 0) red_v[wp] = cmax;
  if (tid == 0) sing_s = 0;
  __syncthreads();
  double norm1 = 0.0;
  for (int i = 0; i < (nt + 31) / 32; ++i) norm1 = fmax(norm1, red_v[i]);
  cl.sync();
  bool singular = false;
  for (int c = 0; c < k; ++c) {
    const int owner = c / w;
    double* my_slot = slot + (c & 1) * (k + 2);
    if (q == owner) {
      const int cl_ = c - c0;
      for (int r = tid; r < k; r += nt) my_slot[r] = A_s[r * ld + cl_];
      if (wp == 0) {
        double best = -1.0;
        int bi = c;
        for (int r = c + lane; r < k; r += 32) {
          const double a = fabs(A_s[r * ld + cl_]);
          if (a > best) { best = a; bi = r; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) {
          my_slot[k] = (double)bi;
          my_slot[k + 1] = best > 0.0 ? 1.0 / A_s[bi * ld + cl_] : 0.0;
        }
      }
    }
    cl.sync();
    const double* os = cl.map_shared_rank(slot + (c & 1) * (k + 2), owner);
    const int pr = (int)os[k];
    const double inv = os[k + 1];
    if (inv == 0.0) {
      singular = true;
      break;
    }
    // the pivot column after the interchange (row c excluded), from the owner's copy
    for (int r = tid; r < k; r += nt) fac[r] = (r == c) ? 0.0 : os[r == pr ? c : r];
    if (tid == 0) perm_s[c] = pr;
    __syncthreads();
    // interchange rows c and pr, scale the pivot row (its pivot entry becomes 1 / pivot)
    for (int j = tid; j < wl; j += nt) {
      const double a = A_s[c * ld + j], b = A_s[pr * ld + j];
      if (pr != c) A_s[pr * ld + j] = a;
      A_s[c * ld + j] = (c0 + j == c ? 1.0 : b) * inv;
    }
    __syncthreads();
    // eliminate: thread -> (column j, rows r0 + u rstep), eight rows' loads before their stores
    if (wl > 0) {
      const int jj = tid % wl, r0 = tid / wl, rstep = nt / wl;
      if (r0 < rstep) {
        const double pc = A_s[c * ld + jj];
        const bool colc = c0 + jj == c;
        for (int r1 = r0; r1 < k; r1 += 8 * rstep) {
          double f[8], x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int r = r1 + u * rstep;
            f[u] = r < k ? fac[r] : 0.0;
            x[u] = (r < k && !colc) ? A_s[r * ld + jj] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int r = r1 + u * rstep;
            if (r < k && f[u] != 0.0) A_s[r * ld + jj] = x[u] - f[u] * pc;
          }
        }
      }
    }
    __syncthreads();
  }
  if (singular) {
    if (q == 0 && tid == 0) *cond = INFINITY;
    cl.sync();
    return;
  }
  // (P M)^{-1} P = M^{-1}: column j of the inverse is working column src[j]
  if (tid == 0) {
    for (int j = 0; j < k; ++j) src_s[j] = j;
    for (int c = k - 1; c >= 0; --c) {
      const int p = perm_s[c], t = src_s[c];
      src_s[c] = src_s[p];
      src_s[p] = t;
    }
  }
  __syncthreads();
  double imax = 0.0;
  for (int j = wp; j < k; j += nt / 32) {  // warp per output column whose source is local
    const int sj = src_s[j];
    if (sj < c0 || sj >= c0 + wl) continue;
    double a = 0.0;
    for (int i = lane; i < k; i += 32) {
      const double x = A_s[i * ld + (sj - c0)];
      Minv[(int64_t)i * k + j] = x;
      a += fabs(x);
    }
    imax = fmax(imax, warp_sum(a));
  }
  imax = warp_max(imax);
  __syncthreads();
  if (lane == 0) red_v[wp] = imax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < (nt + 31) / 32; ++i) m = fmax(m, red_v[i]);
    slot[0] = m;
    slot[1] = norm1;
  }
  cl.sync();
  if (q == 0 && tid == 0) {
    double m = 0.0, n1 = 0.0;
    for (int r = 0; r < C; ++r) {
      const double* o = cl.map_shared_rank(slot, r);
      m = fmax(m, o[0]);
      n1 = fmax(n1, o[1]);
    }
    *cond = n1 * m;
  }
  cl.sync();
}

// X <- X M in place: 32 rows per CTA staged in shared memory, DMMA 8x8x4.
__global__ void __launch_bounds__(128) materialize_kernel(double* X, int64_t rows, int k,
                                                          const double* __restrict__ M) {
  pdl_begin();
  extern __shared__ double T[];  // 32 x (k + 4)
  const int ld = k + 4;
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int tid = threadIdx.x;
  for (int e = tid; e < 32 * k; e += 128) {
    int r = e / k, c = e % k;
    T[r * ld + c] = (r0 + r < rows) ? X[(r0 + r) * k + c] : 0.0;
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int rb = warp * 8;
  for (int c0 = 0; c0 < k; c0 += 8) {
    double c_0 = 0.0, c_1 = 0.0;
    for (int l = 0; l < k; l += 4) {
      double a = T[(rb + g) * ld + l + t];
      double b = M[(int64_t)(l + t) * k + c0 + g];
      dmma8x8x4(c_0, c_1, a, b);
    }
    const int64_t row = r0 + rb + g;
    if (row < rows) {
      X[row * k + c0 + 2 * t] = c_0;
      X[row * k + c0 + 2 * t + 1] = c_1;
    }
  }
}

__global__ void materialize_generic(double* X, int64_t rows, int k, const double* __restrict__ M) {
  pdl_begin();
  extern __shared__ double T[];
  const int64_t r = blockIdx.x;
  for (int c = threadIdx.x; c < k; c += blockDim.x) T[c] = X[r * k + c];
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    double a = 0.0;
    for (int l = 0; l < k; ++l) a = fma(T[l], M[l * k + c], a);
    X[r * k + c] = a;
  }
}

__global__ void identity_kernel(double* M, int k) {
  pdl_begin();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < k * k) M[e] = (e / k == e % k) ? 1.0 : 0.0;
}

// single-block compaction of the keep mask: kidx[a] = compact index or -1, klist = kept ids
__global__ void __launch_bounds__(1024) compact_keep_kernel(const int32_t* __restrict__ keep, int64_t s,
                                                            int32_t* __restrict__ kidx, int32_t* __restrict__ klist,
                                                            int64_t* d_r) {
  pdl_begin();
  __shared__ int64_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t chunk = (s + 1023) / 1024;
  const int64_t b = tid * chunk, e = (b + chunk < s) ? b + chunk : s;
  int64_t cnt = 0;
  for (int64_t i = b; i < e; ++i) cnt += keep[i] ? 1 : 0;
  int64_t inc = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    int64_t ws = wsum[lane], wi = ws;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    wsum[lane] = wi - ws;
    if (lane == 31) *d_r = wi;
  }
  __syncthreads();
  int64_t pos = wsum[w] + inc - cnt;
  for (int64_t i = b; i < e; ++i) {
    if (keep[i]) {
      kidx[i] = (int32_t)pos;
      if (klist) klist[pos] = (int32_t)i;
      ++pos;
    } else {
      kidx[i] = -1;
    }
  }
}

__global__ void copy_diag_kernel(const double* __restrict__ G, int64_t s, double* __restrict__ d) {
  pdl_begin();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < s) d[i] = G[i * s + i];
}

// K (col-major (k+s) x (k+r)) = [[diag Σ, 0], [P0, R_kept^T]]
__global__ void core_rows_kernel(int k, int64_t s, int64_t r, const double* __restrict__ Sigma,
                                 const double* __restrict__ P0, const double* __restrict__ R,
                                 const int32_t* __restrict__ klist, double* __restrict__ K) {
  pdl_begin();
  // column j of the core per blockIdx.y (grid-strided), rows by the threads: no index division
  const int64_t mr = k + s, nc = k + r;
  for (int64_t j = blockIdx.y; j < nc; j += gridDim.y) {
    double* col = K + j * mr;
    const int64_t p = j >= k ? (int64_t)klist[j - k] : 0;
    const double* Rrow = R + p * s;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < mr; i += (int64_t)gridDim.x * blockDim.x) {
      double v;
      if (i < k)
        v = (j == i) ? Sigma[i] : 0.0;
      else if (j < k)
        v = P0[(i - k) * k + j];
      else
        v = (i - k >= p) ? Rrow[i - k] : 0.0;  // R upper only
      col[i] = v;
    }
  }
}

// L (row-major (k+r) x s) = [P0^T; R_kept]
__global__ void lift_block_kernel(int k, int64_t s, int64_t r, const double* __restrict__ P0,
                                  const double* __restrict__ R, const int32_t* __restrict__ klist,
                                  double* __restrict__ L) {
  pdl_begin();
  const int64_t n = (int64_t)(k + r) * s;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / s, c = e % s;
    L[e] = (i < k) ? P0[c * k + i] : (c >= klist[i - k] ? R[(int64_t)klist[i - k] * s + c] : 0.0);  // R upper only
  }
}

__global__ void add_diag_kernel(double* K, int64_t ldk, int k, const double* __restrict__ Sigma) {
  pdl_begin();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) K[i * ldk + i] += Sigma[i];
}

// Gfull (s x k row-major): row a = Gc row (k + kidx[a]) for kept a, else 0; Gc col-major, ld ldg.
__global__ void expand_rows_kernel(const double* __restrict__ Gc, int64_t ldg, int k, int64_t s,
                                   const int32_t* __restrict__ kidx, double* __restrict__ Gfull) {
  pdl_begin();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= s * k) return;
  int64_t a, c64;
  divmod_idx(e, k, a, c64);
  const int c = (int)c64;
  const int32_t q = kidx[a];
  Gfull[e] = (q >= 0) ? Gc[(int64_t)(k + q) + (int64_t)c * ldg] : 0.0;
}

// out (rows x cols, row-major, ldo) = A (column-major, lda): 32 x 32 tiles through shared
// memory (padded rows), so both the column reads and the row writes are coalesced (the
// element-wise version read one column element per thread: 60 GB/s on configs[4]'s
// 100k x 256 blocks)
__global__ void __launch_bounds__(256) c2r_kernel(const double* __restrict__ A, int64_t lda, int64_t rows, int64_t cols,
                                                  double* __restrict__ out, int64_t ldo) {
  pdl_begin();
  __shared__ double t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // read: column j0 + ty + 8q, rows i0 + tx (contiguous in A)
    const int64_t i = i0 + tx, j = j0 + ty + 8 * q;
    if (i < rows && j < cols) t[ty + 8 * q][tx] = A[i + j * lda];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // write: row i0 + ty + 8q, columns j0 + tx (contiguous in out)
    const int64_t i = i0 + ty + 8 * q, j = j0 + tx;
    if (i < rows && j < cols) out[i * ldo + j] = t[tx][ty + 8 * q];
  }
}

__global__ void maxdev_identity_kernel(const double* __restrict__ G, int k, double* out) {
  pdl_begin();
  double m = 0.0;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) m = fmax(m, fabs(G[e] - ((e / k == e % k) ? 1.0 : 0.0)));
  m = warp_max(m);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) r = fmax(r, red[i]);
    *out = r;
  }
}

__global__ void axpby_kernel(int64_t rows, int64_t cols, double alpha, CMat A, double beta, Mat C) {
  pdl_begin();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  int64_t i, j;
  divmod_idx(e, cols, i, j);
  double* c = C.p + i * C.rs + j * C.cs;
  const double a = alpha * A.p[i * A.rs + j * A.cs];
  *c = (beta == 0.0) ? a : fma(beta, *c, a);
}

__global__ void nonfinite_kernel(const double* __restrict__ v, int64_t n, int* flag) {
  pdl_begin();
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(v[i])) bad = 1;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 2);
}
}  // namespace

// Blocked right-looking Cholesky with deflation (R8): per 64-wide panel, the
// panel factorisation in one CTA, the panel's row block R_pp^{-T} G[p, p+nb:], and the
// trailing SYRK on the DMMA GEMM.  Look-ahead: the trailing update is split into the next
// panel's row block (small GEMM, on the critical path) and the rest (big SYRK); the next
// panel's factorisation and row block run on a second stream while the big SYRK of the
// current panel runs, hiding the serial panel chain behind the trailing updates.
// (A recursive variant with large-K GEMMs measured slower at s = 5000 on B200: its many
// small TRSM leaves serialise.)
cudaError_t chol_deflate(cudaStream_t st, double* G, int64_t s, const double* enorm2, double tau, int32_t* keep,
                         double* Tb) {
  cudaError_t e;
  if (dag_enabled() && enorm2) {
    if (Tb) return chol_dag(st, G, s, enorm2, tau, keep, Tb, false);
    double* tmp = nullptr;
    if ((e = cudaMallocAsync(&tmp, (size_t)((s + CNB - 1) / CNB) * CNB * CNB * sizeof(double), st))) return e;
    if ((e = chol_dag(st, G, s, enorm2, tau, keep, tmp, true))) return e;
    return cudaFreeAsync(tmp, st);
  }
  static thread_local cudaStream_t side = nullptr;
  static thread_local cudaEvent_t ev_side = nullptr, ev_main = nullptr;
  static bool attr = false;
  const size_t sm2 = 2 * (size_t)CNB * (CNB + 1) * sizeof(double);
  if (!side) {
    if ((e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking))) return e;
    if ((e = cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming))) return e;
    if ((e = cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming))) return e;
  }
  if (!attr) {
    cudaFuncSetAttribute(chol_panel_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    cudaFuncSetAttribute(tri_solve_warp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    attr = true;
  }
  // factor + row block of panel p; pp >= 0: the contribution of panel pp (rows pp..pp+nbp of
  // R) to this panel's rows is subtracted inside both kernels (fused look-ahead update)
  auto panel = [&](cudaStream_t q, int64_t p, int64_t pp, int nbp) -> cudaError_t {
    const int nb = (int)std::min<int64_t>(CNB, s - p);
    const int64_t rest = s - p - nb;
    // K5/K6 accounting on the stream the panel kernels run on
    const int pidx = g_prof ? g_prof->begin(KC_PANEL, (double)nb * nb * nb / 3.0 + (double)nb * nb * rest +
                                                          (pp >= 0 ? 2.0 * nbp * nb * (nb / 2.0 + rest) : 0.0),
                                            8.0 * ((double)nb * nb + 2.0 * nb * rest), q)
                            : -1;
    struct End { int i; ~End() { if (i >= 0) g_prof->end(i); } } end_{pidx};
    ++g_launches;
    launch_k(chol_panel_factor, 1, 256, sm2, q, G, s, p, nb, enorm2, tau, keep, pp, nbp);
    if (rest > 0) {
      ++g_launches;
      launch_k(tri_solve_warp_kernel<true>, cdiv(rest, 8), 256, sm2, q, G, s, p, nb, keep, G, s, p + nb, s, pp, nbp);
    }
    return cudaGetLastError();
  };
  if (s <= 0) return cudaSuccess;
  if ((e = panel(st, 0, -1, 0))) return e;
  // Pipeline: panel p1 = p + nb is factored and solved on the side stream (with panel p's
  // contribution fused in) while the main stream applies panel p to the rows >= p + 2nb
  // (SYRK on the DMMA GEMM); the chain per panel is factor + row solve only.
  for (int64_t p = 0; p < s; p += CNB) {
    const int nb = (int)std::min<int64_t>(CNB, s - p);
    const int64_t p1 = p + nb;
    if (p1 >= s) break;
    const int nb1 = (int)std::min<int64_t>(CNB, s - p1);
    if ((e = cudaEventRecord(ev_main, st))) return e;       // SYRK(p - nb) and solve(p) are done
    if ((e = cudaStreamWaitEvent(side, ev_main, 0))) return e;
    if ((e = panel(side, p1, p, nb))) return e;
    if ((e = cudaEventRecord(ev_side, side))) return e;
    const int64_t p2 = p1 + nb1, rest2 = s - p2;
    if (rest2 > 0) {
      const double* Rq = G + p * s + p2;  // R[p:p+nb, p2:]
      if ((e = dgemm_rm(st, true, false, rest2, rest2, nb, -1.0, Rq, s, Rq, s, 1.0, G + p2 * s + p2, s, 1)))
        return e;
    }
    if ((e = cudaStreamWaitEvent(st, ev_side, 0))) return e;
  }
  dim3 grid(cdiv(std::max<int64_t>(s, 1), 256), (unsigned)std::min<int64_t>(std::max<int64_t>(s, 1), 4096));
  ++g_launches;
  launch_k(zero_lower_kernel, grid, 256, 0, st, G, s);
  return cudaGetLastError();
}

cudaError_t chol_inv_small(cudaStream_t st, double* G, int l, const double* enorm2, double tau, int32_t* keep,
                           double* T) {
  if (l <= 0) return cudaSuccess;
  if (l > CSMALL) return cudaErrorInvalidValue;
  const size_t smem = (size_t)CSMALL * CLD * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(chol_inv_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  KScope sc(KC_SMALLCHOL, (double)l * l * l / 3.0 * 2.0, 8.0 * 3.0 * l * l);
  ++g_launches;   // (inside the scope: the class's launch count)
  switch ((l + 15) / 16) {
    case 1: return launch_chol_aug<16>(st, G, l, enorm2, tau, keep, T);
    case 2: return launch_chol_aug<32>(st, G, l, enorm2, tau, keep, T);
    case 3: return launch_chol_aug<48>(st, G, l, enorm2, tau, keep, T);
    case 4: return launch_chol_aug<64>(st, G, l, enorm2, tau, keep, T);
    case 5: return launch_chol_aug<80>(st, G, l, enorm2, tau, keep, T);
    case 6: return launch_chol_aug<96>(st, G, l, enorm2, tau, keep, T);
    default: break;
  }
  launch_k(chol_inv_small_kernel, 1, 1024, smem, st, G, l, enorm2, tau, keep, T);
  return cudaGetLastError();
}

cudaError_t trsm_upper(cudaStream_t st, const double* R, int64_t s, const int32_t* keep, double* X, int k,
                       const double* Tb) {
  cudaError_t e;
  if (Tb && dag_enabled()) return trsm_dag(st, R, s, Tb, X, k);
  const int64_t npan = (s + CNB - 1) / CNB;
  for (int64_t q = npan - 1; q >= 0; --q) {
    const int64_t p = q * CNB;
    const int nb = (int)std::min<int64_t>(CNB, s - p);
    ++g_launches;
    {
      KScope sc(KC_PANEL, (double)nb * nb * k, 8.0 * ((double)nb * nb / 2.0 + 2.0 * nb * k));
      launch_k(tri_solve_warp_kernel<false>, cdiv(k, 8), 256, (size_t)CNB * (CNB + 1) * sizeof(double), st, R, s, p, nb,
                                                                                                     keep, X, k, 0, k, -1, 0);
    }
    if (p > 0) {
      // X[0:p] -= R[0:p, p:p+nb] X[p:p+nb]
      if ((e = dgemm_rm(st, false, false, p, k, nb, -1.0, R + p, s, X + p * k, k, 1.0, X, k))) return e;
    }
  }
  return cudaGetLastError();
}

cudaError_t inverse_gj(cudaStream_t st, const double* M, int k, double* Minv, double* cond, Scratch& ws) {
  static const bool gjb_on = !(getenv("TSVD_GJ_BLK") && atoi(getenv("TSVD_GJ_BLK")) == 0);
  if (gjb_on && k <= GJB_K) {
    const size_t smem = (size_t)(GJB_K + 16) * GJB_LD * sizeof(double);
    static bool attrb = false;
    if (!attrb) {
      cudaFuncSetAttribute(gj_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attrb = true;
    }
    ++g_launches;
    launch_k(gj_blk_kernel, 1, 1024, smem, st, M, k, Minv, cond);
    return cudaGetLastError();
  }
  if (k <= GJ_SMEM_K) {
    const size_t smem = (size_t)k * (2 * k + 1) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gj_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)((size_t)GJ_SMEM_K * (2 * GJ_SMEM_K + 1) * sizeof(double)));
      attr = true;
    }
    ++g_launches;
    static const int gjt = getenv("TSVD_GJ_THREADS") ? atoi(getenv("TSVD_GJ_THREADS")) : 512;  // tuning
    launch_k(gj_smem_kernel, 1, gjt, smem, st, M, k, Minv, cond);
    return cudaGetLastError();
  }
  if (k <= GJ_INPLACE_K) {
    const size_t smem = (size_t)k * (k | 1) * sizeof(double);
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(gj_inplace_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)((size_t)GJ_INPLACE_K * (GJ_INPLACE_K | 1) * sizeof(double)));
      attr2 = true;
    }
    ++g_launches;
    launch_k(gj_inplace_kernel, 1, 1024, smem, st, M, k, Minv, cond);
    return cudaGetLastError();
  }
  static const bool gjc_on = !(getenv("TSVD_GJ_CLUSTER") && atoi(getenv("TSVD_GJ_CLUSTER")) == 0);
  for (int C : {2, 4, 8, 16}) {
    if (!gjc_on || k > 512) break;
    const int w = (k + C - 1) / C;
    const size_t smem = ((size_t)k * (w | 1) + 2 * (k + 2) + k) * sizeof(double) + 2 * (size_t)k * sizeof(int);
    if (smem > 200 * 1024) continue;
    cudaFuncSetAttribute(gj_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (C > 8) cudaFuncSetAttribute(gj_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 2 : 1;
    ++g_launches;
    if (cudaLaunchKernelEx(&cfg, gj_cluster_kernel, M, k, w, Minv, cond) == cudaSuccess) return cudaSuccess;
    cudaGetLastError();
    --g_launches;
  }
  double* aug = ws.alloc<double>((size_t)2 * k * k);
  if (ws.err) return ws.err;
  ++g_launches;
  launch_k(gj_kernel, 1, 1024, k * sizeof(double), st, M, k, aug, Minv, cond);
  return cudaGetLastError();
}

cudaError_t materialize_rows(cudaStream_t st, double* X, int64_t rows, int k, const double* M) {
  if (rows == 0) return cudaSuccess;
  // large factors (an MII reset of configs[4]'s 18M x 256 U'): DMMA GEMMs by row chunks into a
  // bounded buffer, copied back — the one-CTA-per-32-rows kernel re-reads M (512 KB at k = 256)
  // from L2 per CTA and ran ~7x slower there
  if (rows >= 65536 && k >= 64) {
    const int64_t crow = std::min<int64_t>(rows, std::max<int64_t>(4096, ((int64_t)256 << 20) / k));
    double* tmp = nullptr;
    cudaError_t e = cudaMallocAsync(&tmp, (size_t)crow * k * sizeof(double), st);
    if (e) return e;
    for (int64_t r0 = 0; r0 < rows; r0 += crow) {
      const int64_t nr = std::min(crow, rows - r0);
      if ((e = dgemm_rm(st, false, false, nr, k, k, 1.0, X + r0 * k, k, M, k, 0.0, tmp, k))) return e;
      if ((e = cudaMemcpyAsync(X + r0 * k, tmp, (size_t)nr * k * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
    }
    return cudaFreeAsync(tmp, st);
  }
  if (k % 8 == 0) {
    const size_t smem = 32 * (size_t)(k + 4) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(materialize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    ++g_launches;
    launch_k(materialize_kernel, cdiv(rows, 32), 128, smem, st, X, rows, k, M);
  } else {
    ++g_launches;
    launch_k(materialize_generic, (unsigned)rows, 128, k * sizeof(double), st, X, rows, k, M);
  }
  return cudaGetLastError();
}

cudaError_t set_identity(cudaStream_t st, double* M, int k) {
  ++g_launches;
  launch_k(identity_kernel, cdiv((int64_t)k * k, 256), 256, 0, st, M, k);
  return cudaGetLastError();
}

cudaError_t compact_keep(cudaStream_t st, const int32_t* keep, int64_t s, int32_t* kidx, int64_t* d_r, Scratch& ws) {
  (void)ws;
  // klist is stored right after kidx (caller allocates 2 s)
  ++g_launches;
  launch_k(compact_keep_kernel, 1, 1024, 0, st, keep, s, kidx, kidx + s, d_r);
  return cudaGetLastError();
}

cudaError_t copy_diag(cudaStream_t st, const double* G, int64_t s, double* d) {
  ++g_launches;
  launch_k(copy_diag_kernel, cdiv(s, 256), 256, 0, st, G, s, d);
  return cudaGetLastError();
}

cudaError_t build_core_rows(cudaStream_t st, int k, int64_t s, int64_t r, const double* Sigma, const double* P0,
                            const double* R, const int32_t* kidx, double* K) {
  const int64_t n = (int64_t)(k + r) * (k + s);
  ++g_launches;
  (void)n;
  dim3 grid((unsigned)std::min<int64_t>(cdiv(k + s, 256), 8), (unsigned)std::min<int64_t>(k + r, 65535));
  launch_k(core_rows_kernel, grid, 256, 0, st, k, s, r, Sigma, P0, R, kidx + s, K);
  return cudaGetLastError();
}

cudaError_t build_lift_block(cudaStream_t st, int k, int64_t s, int64_t r, const double* P0, const double* R,
                             const int32_t* kidx, double* L) {
  const int64_t n = (int64_t)(k + r) * s;
  if (n == 0) return cudaSuccess;
  ++g_launches;
  launch_k(lift_block_kernel, (unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 32), 256, 0, st, k, s, r, P0, R, kidx + s, L);
  return cudaGetLastError();
}

cudaError_t add_diag_sigma(cudaStream_t st, double* K, int64_t ldk, int k, const double* Sigma, bool colmajor) {
  (void)colmajor;  // diagonal: same index either way
  ++g_launches;
  launch_k(add_diag_kernel, cdiv(k, 128), 128, 0, st, K, ldk, k, Sigma);
  return cudaGetLastError();
}

cudaError_t expand_rows(cudaStream_t st, const double* Gc, int64_t ldg, int k, int64_t s, const int32_t* kidx,
                        double* Gfull) {
  if (s == 0) return cudaSuccess;
  ++g_launches;
  launch_k(expand_rows_kernel, cdiv(s * k, 256), 256, 0, st, Gc, ldg, k, s, kidx, Gfull);
  return cudaGetLastError();
}

cudaError_t colmajor_to_rowmajor(cudaStream_t st, const double* A, int64_t lda, int64_t rows, int64_t cols,
                                 double* out, int64_t ldo) {
  if (rows * cols == 0) return cudaSuccess;
  if (cdiv(cols, 32) > 65535) return cudaErrorInvalidValue;
  ++g_launches;
  launch_k(c2r_kernel, dim3((unsigned)cdiv(rows, 32), (unsigned)cdiv(cols, 32)), 256, 0, st, A, lda, rows, cols, out, ldo);
  return cudaGetLastError();
}

namespace {
struct Mats4 {
  const double* p[4];
};
// ||A||_2 estimate of the k x k row-major matrix p[blockIdx.x] by `iters` power iterations on
// A^T A from a fixed, nowhere-zero start vector (the Rayleigh quotient from below: a lower
// estimate, exact to the top cluster); one CTA per matrix: y = A x a warp per row (coalesced
// row reads), x = A^T y by G = blockDim / k row groups per column (coalesced across columns),
// their partial sums combined in a fixed order
__global__ void __launch_bounds__(1024) norm2_est_kernel(Mats4 m, int k, int iters, double* __restrict__ out) {
  pdl_begin();
  const double* A = m.p[0];
  for (int q = 1; q < 4; ++q)
    if (blockIdx.x == q) A = m.p[q];
  extern __shared__ double sh_v[];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5, nw = nt >> 5;
  const int G = max(1, nt / k);
  double* x = sh_v;
  double* y = sh_v + k;
  double* part = sh_v + 2 * k;  // G x k
  __shared__ double red[32];
  __shared__ double nrm;
  auto block_norm = [&](const double* v) {
    double a = 0.0;
    for (int i = tid; i < k; i += nt) a = fma(v[i], v[i], a);
    a = warp_sum(a);
    if (lane == 0) red[w] = a;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < nw; ++q) t += red[q];
      nrm = sqrt(t);
    }
    __syncthreads();
    return nrm;
  };
  for (int i = tid; i < k; i += nt) x[i] = 1.0 + 0.5 * sin(0.7 * (double)i);
  __syncthreads();
  const double n0 = block_norm(x);
  for (int i = tid; i < k; i += nt) x[i] /= n0;
  __syncthreads();
  double lam = 0.0;
  for (int it = 0; it < iters; ++it) {
    for (int r = w; r < k; r += nw) {  // y = A x
      double a = 0.0;
      for (int j = lane; j < k; j += 32) a = fma(A[(int64_t)r * k + j], x[j], a);
      a = warp_sum(a);
      if (lane == 0) y[r] = a;
    }
    __syncthreads();
    for (int e = tid; e < G * k; e += nt) {  // part[g][j] = sum over rows i = g mod G of A[i][j] y[i]
      const int g = e / k, j = e - g * k;
      double a = 0.0;
      for (int i = g; i < k; i += G) a = fma(A[(int64_t)i * k + j], y[i], a);
      part[g * k + j] = a;
    }
    __syncthreads();
    for (int j = tid; j < k; j += nt) {
      double a = 0.0;
      for (int g = 0; g < G; ++g) a += part[g * k + j];
      x[j] = a;
    }
    __syncthreads();
    lam = block_norm(x);  // -> sigma_max^2
    if (!(lam > 0.0)) break;
    for (int i = tid; i < k; i += nt) x[i] /= lam;
    __syncthreads();
  }
  if (tid == 0) out[blockIdx.x] = sqrt(lam);
}
}  // namespace

// ||A||_2 estimates of up to 4 k x k row-major matrices (null entries skipped) into d_out
cudaError_t norm2_estimates(cudaStream_t st, const double* const* mats, int nm, int k, double* d_out) {
  if (nm <= 0 || nm > 4) return cudaErrorInvalidValue;
  Mats4 m{};
  for (int i = 0; i < nm; ++i) m.p[i] = mats[i];
  ++g_launches;
  const int G = std::max(1, 1024 / k);
  launch_k(norm2_est_kernel, nm, 1024, (2 + (size_t)G) * k * sizeof(double), st, m, k, 40, d_out);
  return cudaGetLastError();
}

cudaError_t check_init(cudaStream_t st, const double* X, int64_t rows, int k, double* d_maxdev, Scratch& ws) {
  double* G = ws.alloc<double>((size_t)k * k);
  if (ws.err) return ws.err;
  cudaError_t e = dgemm_rm(st, true, false, k, k, rows, 1.0, X, k, X, k, 0.0, G, k);
  if (e) return e;
  ++g_launches;
  launch_k(maxdev_identity_kernel, 1, 256, 0, st, G, k, d_maxdev);
  return cudaGetLastError();
}

cudaError_t find_nonfinite(cudaStream_t st, const double* v, int64_t n, int* d_flag) {
  if (n == 0) return cudaSuccess;
  ++g_launches;
  launch_k(nonfinite_kernel, (unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 8), 256, 0, st, v, n, d_flag);
  return cudaGetLastError();
}

cudaError_t mat_axpby(cudaStream_t st, int64_t rows, int64_t cols, double alpha, CMat A, double beta, Mat C) {
  if (rows * cols == 0) return cudaSuccess;
  ++g_launches;
  launch_k(axpby_kernel, cdiv(rows * cols, 256), 256, 0, st, rows, cols, alpha, A, beta, C);
  return cudaGetLastError();
}

}  // namespace tsvd
