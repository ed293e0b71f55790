// potrf.cuh — the blocked Cholesky with deflation of one N x N diagonal block together with
// Y = R^{-T}, as the right-looking factorisation of the augmented block [A | I] in shared memory
// (the panel solves applied to I are the forward substitution R^T Y = I, so the inverse costs
// no extra sequential steps).  16-wide sub-panels:
//   pivots:    warp 0, the 16 x 16 diagonal block in registers (lane: column lane % 16, rows
//              lane / 16 + 2m), one pivot per step with shuffles, the next pivot's Schur diagonal
//              formed redundantly in every lane; deflation test of DESIGN.md R8 on the current
//              Schur diagonal (Alg 2's unguarded alpha); r = d rsqrt(d);
//   row block: one thread per remaining column of [A | I] (always N columns);
//   trailing:  8 x 8 DMMA tiles over the upper part of A and the live part of the right block.
// Used by the tile-DAG Cholesky (dag.cu, N = 64) and the one-CTA Cholesky-QR factor (dense.cu).
// A: N x (2N + 4) doubles, [A | I] on entry (pivots >= nb an identity), [R | Y] on exit; en: the
// deflation reference (squared row norms) of the nb real pivots; keep[i] (i < nb) <- pivot kept.
#pragma once
#include "common.cuh"

namespace tsvd {
constexpr int PSUB = 16;

template <int N, int NTHR>
__device__ void potrf_core_t(double* A, int nb, const double* __restrict__ en, double tau, int32_t* __restrict__ keep) {
  constexpr int ALDN = 2 * N + 4;
  __shared__ double rinv[N], en_s[N];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  if (tid < N) en_s[tid] = tid < nb ? en[tid] : 1.0;
  __syncthreads();
  for (int j0 = 0; j0 < N; j0 += PSUB) {
    const int j1 = j0 + PSUB;
    if (warp == 0) {
      const int c = lane & 15, p = lane >> 4;
      double a[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = A[(j0 + 2 * m + p) * ALDN + j0 + c];
      // the next pivot's Schur diagonal is formed redundantly in every lane from values read
      // before this pivot's update (same fma as the owning lane's update), so the sequential
      // chain per pivot is rsqrt + two flops rather than a shuffle round trip through the update
      double d = __shfl_sync(0xffffffffu, a[0], 0);
      double myy = 0.0;
      int mykp = 0;
#pragma unroll
      for (int i = 0; i < PSUB; ++i) {
        const int src = (i & 1) * 16;
        double a01 = 0.0, a11 = 0.0;
        if (i + 1 < PSUB) {
          a01 = __shfl_sync(0xffffffffu, a[i >> 1], src + i + 1);
          a11 = __shfl_sync(0xffffffffu, a[(i + 1) >> 1], ((i + 1) & 1) * 16 + i + 1);
        }
        const int gi = j0 + i;
        const bool real = gi < nb;
        const double e = en_s[gi];
        const bool kp = real && !(e == 0.0 || d <= tau * e);
        // rsqrt of a safe argument, unconditionally, then a select: a conditional call makes the
        // compiler branch around the (warp-uniform) pivot chain, ~100 cycles per pivot
        const double y0 = rsqrt(kp ? d : 1.0);
        const double y = kp ? y0 : (real ? 0.0 : 1.0);
        const double r = kp ? d * y : (real ? 0.0 : 1.0);
        const double aic = __shfl_sync(0xffffffffu, a[i >> 1], src + c);
        double ur[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) ur[m] = __shfl_sync(0xffffffffu, a[i >> 1], src + 2 * m + p) * y;
        const double uc = (c > i) ? aic * y : (c == i ? r : aic);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const int rr = 2 * m + p;
          if (rr > i && c >= rr) a[m] = fma(-ur[m], uc, a[m]);
        }
        if (p == (i & 1)) a[i >> 1] = uc;
        if (i + 1 < PSUB) {
          const double u = a01 * y;
          d = fma(-u, u, a11);
        }
        // no divergent stores inside the pivot chain: lane i keeps pivot i's results
        if (lane == i) {
          myy = y;
          mykp = kp;
        }
      }
      if (lane < PSUB) {
        rinv[j0 + lane] = myy;
        if (j0 + lane < nb) keep[j0 + lane] = mykp;
      }
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int rr = 2 * m + p;
        if (c >= rr) A[(j0 + rr) * ALDN + j0 + c] = a[m];
      }
    }
    __syncthreads();
    // row block: rows j0..j1 of the columns j1..N-1 of A and N..N+j1 of [I] (N columns)
    if (tid < N) {
      const int col = tid < N - j1 ? j1 + tid : N + (tid - (N - j1));
      // right-looking within the 16 rows: the chain per row is one multiply + one fma (the
      // same fmas in the same order as the dot-product form)
      double v[PSUB];
#pragma unroll
      for (int q = 0; q < PSUB; ++q) v[q] = A[(j0 + q) * ALDN + col];
#pragma unroll
      for (int q = 0; q < PSUB; ++q) {
        const double x = v[q] * rinv[j0 + q];
        A[(j0 + q) * ALDN + col] = x;
#pragma unroll
        for (int q2 = q + 1; q2 < PSUB; ++q2) v[q2] = fma(-A[(j0 + q) * ALDN + j0 + q2], x, v[q2]);
      }
    }
    __syncthreads();
    if (j1 < N) {
      // trailing: A[j1:, j1:] (upper tiles) and the right block rows j1.., columns < j1
      const int ntl = (N - j1) / 8, nup = ntl * ntl, nright = ntl * (j1 / 8);
      for (int tile = warp; tile < nup + nright; tile += NTHR / 32) {
        int r0, c0;
        if (tile < nup) {
          const int tr = tile / ntl, tc = tile % ntl;
          if (tr > tc) continue;
          r0 = j1 + tr * 8;
          c0 = j1 + tc * 8;
        } else {
          const int x = tile - nup, nc = j1 / 8;
          r0 = j1 + (x / nc) * 8;
          c0 = N + (x % nc) * 8;
        }
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < PSUB; kk += 4)
          dmma8x8x4(a0, a1, A[(j0 + kk + t) * ALDN + r0 + g], A[(j0 + kk + t) * ALDN + c0 + g]);
        const int r = r0 + g, c = c0 + 2 * t;
        if (c0 >= N || r <= c) A[r * ALDN + c] -= a0;
        if (c0 >= N || r <= c + 1) A[r * ALDN + c + 1] -= a1;
      }
      __syncthreads();
    }
  }
}

}  // namespace tsvd
