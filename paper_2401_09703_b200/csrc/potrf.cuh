// potrf.cuh — the blocked Cholesky with deflation of one N x N diagonal block together with
// Y = R^{-T}, as the right-looking factorisation of the augmented block [A | I] in shared memory
// (the panel solves applied to I are the forward substitution R^T Y = I, so the inverse costs
// no extra sequential steps).  8-wide sub-panels:
//   pivots:    every lane of the N / 32 row-block warps holds the 8 x 8 diagonal block (upper
//              part, 36 registers) and factors it redundantly — no shuffle or barrier on the
//              pivot chain (one warp per SM sub-partition, so the redundant updates do not
//              compete for the FP64 pipe), which is
//              rsqrt + one multiply + one fma per pivot; deflation test of DESIGN.md R8 on the
//              current Schur diagonal (Alg 2's unguarded alpha); r = d rsqrt(d);
//   row block: one thread per remaining column of [A | I] (always N columns), the 8 x 8 factor
//              read from its own registers (so pivots and row block need no barrier between them);
//   trailing:  8 x 8 DMMA tiles over the upper part of A and the live part of the right block,
//              all of a warp's tiles in flight together.
// (A 16-wide sub-panel factored by one warp with shuffles cost ~410 cycles per pivot, 3.4x this.)
// Used by the tile-DAG Cholesky (dag.cu, N = 64) and the one-CTA Cholesky-QR factor (dense.cu).
// A: N x (2N + 4) doubles, [A | I] on entry (pivots >= nb an identity), [R | Y] on exit; en: the
// deflation reference (squared row norms) of the nb real pivots; keep[i] (i < nb) <- pivot kept.
#pragma once
#include "common.cuh"

#ifndef POTRF_MARK
#define POTRF_MARK(i)  // phase hook for tools/scratch micro benchmarks (no-op here)
#endif

namespace tsvd {
constexpr int PSUB = 8;

// DMMA without `volatile`, so the scheduler may interleave it with the surrounding loads
__device__ __forceinline__ void dmma8x8x4_nv(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// tiles of the trailing update that are not in its first tile row (rows >= j1 + 8): the upper
// triangle of the (nt - j - 1)-square block plus its strip of the right block, at most
__host__ __device__ constexpr int potrf_max_rest(int nt) {
  int m = 0;
  for (int j = 1; j < nt; ++j) {
    const int r = nt - j - 1, x = r * (r + 1) / 2 + r * j;
    m = x > m ? x : m;
  }
  return m;
}

// Pivots and row block of the sub-panel at rows j0..j0+7 (threads tid < N).
template <int N>
__device__ __forceinline__ void potrf_panel(double* A, int j0, int nb, const double* en_s, double tau,
                                            int32_t* __restrict__ keep) {
  constexpr int ALDN = 2 * N + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j1 = j0 + PSUB;
  // the diagonal block, upper part, in every lane of the row-block warps (broadcast reads)
  double R[PSUB][PSUB], y[PSUB];
#pragma unroll
  for (int p = 0; p < PSUB; ++p)
#pragma unroll
    for (int c = p; c < PSUB; ++c) R[p][c] = A[(j0 + p) * ALDN + j0 + c];
  int kpm = 0;
#pragma unroll
  for (int i = 0; i < PSUB; ++i) {
    const int gi = j0 + i;
    const bool real = gi < nb;
    const double e = en_s[gi], d = R[i][i];
    const bool kp = real && !(e == 0.0 || d <= tau * e);
    // rsqrt issued on d at once (the deflation test runs beside it), then a select: a
    // deflated d <= 0 only takes rsqrt's slow path for a result that is discarded
    const double y0 = rsqrt(d);
    y[i] = kp ? y0 : (real ? 0.0 : 1.0);
    R[i][i] = kp ? d * y0 : (real ? 0.0 : 1.0);
    kpm |= kp ? 1 << i : 0;
#pragma unroll
    for (int c = i + 1; c < PSUB; ++c) R[i][c] *= y[i];
    // row i of R is final: warp 0 stores it (every lane the same value to the same address,
    // one broadcast wavefront per store, off the pivot chain)
    if (warp == 0) {
#pragma unroll
      for (int c = i; c < PSUB; ++c) A[(j0 + i) * ALDN + j0 + c] = R[i][c];
    }
#pragma unroll
    for (int p = i + 1; p < PSUB; ++p)
#pragma unroll
      for (int c = p; c < PSUB; ++c) R[p][c] = fma(-R[i][p], R[i][c], R[p][c]);
  }
  POTRF_MARK(0);
  // row block: rows j0..j1 of the columns j1..N-1 of A and N..N+j1 of [I] (N columns);
  // right-looking within the 8 rows (chain per row: one multiply + one fma)
  const int col = tid < N - j1 ? j1 + tid : N + (tid - (N - j1));
  double v[PSUB];
#pragma unroll
  for (int q = 0; q < PSUB; ++q) v[q] = A[(j0 + q) * ALDN + col];
#pragma unroll
  for (int q = 0; q < PSUB; ++q) {
    const double x = v[q] * y[q];
    A[(j0 + q) * ALDN + col] = x;
#pragma unroll
    for (int q2 = q + 1; q2 < PSUB; ++q2) v[q2] = fma(-R[q][q2], x, v[q2]);
  }
  if (warp == 0 && lane < PSUB && j0 + lane < nb) keep[j0 + lane] = (kpm >> lane) & 1;
}

// Trailing update by the rows j0..j0+7 of the tiles first + stride * u (u < MAXT) of a set of
// count tiles, coord(tile, r0, c0) giving each tile's corner.  A warp's tiles are all in
// flight together: operand loads (an idle slot reads a valid tile), DMMAs, predicated
// write-back (diagonal tiles: upper part only).
template <int N, int MAXT, class Coord>
__device__ __forceinline__ void potrf_tiles(double* A, int j0, int first, int stride, int count, Coord coord) {
  constexpr int ALDN = 2 * N + 4;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  int r0[MAXT], c0[MAXT];
  bool ok[MAXT];
#pragma unroll
  for (int u = 0; u < MAXT; ++u) {
    const int tile = first + stride * u;
    ok[u] = tile < count;
    r0[u] = c0[u] = j0;
    if (ok[u]) coord(tile, r0[u], c0[u]);
  }
  double fa[MAXT][PSUB / 4], fb[MAXT][PSUB / 4], a0[MAXT], a1[MAXT];
#pragma unroll
  for (int u = 0; u < MAXT; ++u)
#pragma unroll
    for (int kk = 0; kk < PSUB / 4; ++kk) {
      fa[u][kk] = A[(j0 + 4 * kk + t) * ALDN + r0[u] + g];
      fb[u][kk] = A[(j0 + 4 * kk + t) * ALDN + c0[u] + g];
    }
#pragma unroll
  for (int u = 0; u < MAXT; ++u) {
    a0[u] = a1[u] = 0.0;
    if (ok[u]) {  // warp-uniform
#pragma unroll
      for (int kk = 0; kk < PSUB / 4; ++kk) dmma8x8x4_nv(a0[u], a1[u], fa[u][kk], fb[u][kk]);
    }
  }
#pragma unroll
  for (int u = 0; u < MAXT; ++u) {
    if (!ok[u]) continue;
    const int r = r0[u] + g, c = c0[u] + 2 * t;
    if (c0[u] >= N || r <= c) A[r * ALDN + c] -= a0[u];
    if (c0[u] >= N || r <= c + 1) A[r * ALDN + c + 1] -= a1[u];
  }
}

// Look-ahead over the sub-panels: after sub-panel k's row block, the row-block warps
// ("P-warps", ceil(N / 32)) apply its update to the first tile row of the trailing block
// (the rows of sub-panel k + 1), synchronise among themselves and factor sub-panel k + 1 —
// while the other warps apply sub-panel k's update to the rest of the trailing block.  One
// block barrier per sub-panel; the pivot chain runs beside the bulk of the trailing update.
template <int N, int NTHR>
__device__ void potrf_core_t(double* A, int nb, const double* __restrict__ en, double tau, int32_t* __restrict__ keep) {
  static_assert(N % PSUB == 0 && N <= NTHR, "one thread per column of the row block");
  constexpr int NW = NTHR / 32, NPW = (N + 31) / 32, NTW = NW - NPW;
  static_assert(NTW >= 1, "at least one warp for the trailing update");
  constexpr int MAX0 = (N / 8 + NPW - 1) / NPW;
  constexpr int MAXR = potrf_max_rest(N / 8) > 0 ? (potrf_max_rest(N / 8) + NTW - 1) / NTW : 1;
  __shared__ double en_s[N];
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid < N) en_s[tid] = tid < nb ? en[tid] : 1.0;
  __syncthreads();
  if (tid < N) potrf_panel<N>(A, 0, nb, en_s, tau, keep);
  __syncthreads();
  for (int j0 = 0; j0 + PSUB < N; j0 += PSUB) {
    const int j1 = j0 + PSUB, ntl = (N - j1) / 8, nc = j1 / 8;
    if (warp < NPW) {
      // first tile row: (j1, j1 + 8x) for x < ntl, then the right block's (j1, N + 8(x - ntl))
      potrf_tiles<N, MAX0>(A, j0, warp, NPW, N / 8, [&](int x, int& r0, int& c0) {
        r0 = j1;
        c0 = x < ntl ? j1 + 8 * x : N + 8 * (x - ntl);
      });
      asm volatile("bar.sync 1, %0;" ::"r"(NPW * 32) : "memory");
      if (tid < N) potrf_panel<N>(A, j1, nb, en_s, tau, keep);
    } else {
      // the rest: the packed upper triangle of the tile rows 1..ntl-1, then their right strips
      const int rr = ntl - 1, nup = rr * (rr + 1) / 2;
      potrf_tiles<N, MAXR>(A, j0, warp - NPW, NTW, nup + rr * nc, [&](int x, int& r0, int& c0) {
        if (x < nup) {
          int tr = 0;
          while (x >= rr - tr) x -= rr - tr++;
          r0 = j1 + 8 + 8 * tr;
          c0 = j1 + 8 + 8 * (tr + x);
        } else {
          x -= nup;
          r0 = j1 + 8 + 8 * (x / nc);
          c0 = N + 8 * (x % nc);
        }
      });
    }
    __syncthreads();
  }
}

}  // namespace tsvd
