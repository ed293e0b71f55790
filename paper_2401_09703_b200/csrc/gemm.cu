// gemm.cu — K4: small-dense FP64 GEMM / SYRK on the DMMA tensor path (mma.sync m8n8k4 f64).
//
// Used for every dense step of the update: the lift epilogue C0^T = W M_X (Eq (5)
// P:325, App E note P:1083), the SV-LCOV Gram  E E^T - C0^T C0 (Lemma 2), the
// Cholesky trailing update, the weight-update core L_D L_E^T (Alg 4 line 3 P:381-390),
// the multiplier products M F[:k] / M (G[:k] - C G[k:]) (Alg 9 lines 3, 6 P:1196/1199)
// and the new-row block F[k:] M^{-1} (Alg 9 line 4 P:1197).
//
// B200 has no tcgen05 f64 kind; FP64 tensor work is the legacy DMMA path.
// Tile 64x64x16, 4 warps in 2x2, each warp 32x32 = 4x4 DMMA tiles, operands staged in
// shared memory with a 68-double row pitch (conflict-free 64-bit fragment loads),
// register double-buffering of the next K tile.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdio>
#include <cstdlib>

#include "ops.h"

namespace tsvd {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, LDS = BM + 4;

// blockIdx.z = split-K slice: this CTA sums k in [z kchunk, (z+1) kchunk); with split-K
// the caller passes a partial buffer as C (alpha = 1, beta = 0, C.p offset by z).
template <bool UPPER>
__global__ void __launch_bounds__(128) dgemm_kernel(int64_t M, int64_t N, int64_t Ktot, int64_t kchunk, double alpha,
                                                    CMat A, CMat B, double beta, Mat C, int64_t zstride) {
  pdl_begin();
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t K = min(Ktot - kbeg, kchunk);
  A.p += kbeg * A.cs;
  B.p += kbeg * B.rs;
  C.p += (int64_t)blockIdx.z * zstride;
  if (UPPER && m0 > n0 + BN - 1) return;  // tile strictly below the diagonal
  __shared__ __align__(16) double As[BK][LDS];  // [k][m]
  __shared__ __align__(16) double Bs[BK][LDS];  // [k][n]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // per-thread load coordinates (8 elements of A and of B per K tile)
  const bool a_mfast = (A.rs == 1);  // m contiguous in memory
  const bool b_nfast = (B.cs == 1);  // n contiguous in memory
  double ra[8], rb[8];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int idx = tid + e * 128;
      int mm, kk;
      if (a_mfast) { mm = idx & 63; kk = idx >> 6; } else { kk = idx & 15; mm = idx >> 4; }
      int64_t gm = m0 + mm, gk = k0 + kk;
      ra[e] = (gm < M && gk < K) ? A.p[gm * A.rs + gk * A.cs] : 0.0;
      int nn, kb;
      if (b_nfast) { nn = idx & 63; kb = idx >> 6; } else { kb = idx & 15; nn = idx >> 4; }
      int64_t gn = n0 + nn, gkb = k0 + kb;
      rb[e] = (gn < N && gkb < K) ? B.p[gkb * B.rs + gn * B.cs] : 0.0;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int idx = tid + e * 128;
      int mm, kk;
      if (a_mfast) { mm = idx & 63; kk = idx >> 6; } else { kk = idx & 15; mm = idx >> 4; }
      As[kk][mm] = ra[e];
      int nn, kb;
      if (b_nfast) { nn = idx & 63; kb = idx >> 6; } else { kb = idx & 15; nn = idx >> 4; }
      Bs[kb][nn] = rb[e];
    }
  };

  load(0);
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
    store();
    __syncthreads();
    if (k0 + BK < K) load(k0 + BK);  // overlaps the global latency with the MMAs below
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk + t][wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk + t][wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + wm + i * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t col = n0 + wn + j * 8 + 2 * t + h;
        if (col >= N || (UPPER && row > col)) continue;
        double* c = C.p + row * C.rs + col * C.cs;
        double v = alpha * acc[i][j][h];
        if (beta != 0.0) v += beta * (*c);
        *c = v;
      }
    }
  }
}

// ------------------------------------------------------------------ v2: cp.async pipeline
// CTA tile 128 x 64 x 16 (or 64 x 64), 8 (4) warps, warp tile 32 x 32 (4 x 4 DMMA 8x8x4
// tiles), a 3-stage cp.async (8-byte, zero-filled at the edges) pipeline through shared
// memory.  An operand whose m (n) dimension is contiguous in global memory is staged
// k-major (As[k][m], pitch 8 mod 16 doubles; a warp loads 32 m x 1 k); one whose k
// dimension is contiguous is staged [m][k] (pitch 4 mod 16; a warp loads two 128-byte rows
// of 16 k).  Either way the cp.async writes and the fragment reads (lanes = 8 m x 4 k) touch
// every bank exactly twice per 256-byte warp access (the minimum).
constexpr int V2M = 128, V2N = 64, V2K = 16, V2S = 3;
constexpr int PK = V2K + 4;  // pitch of k-contiguous tiles ([m][k] / [n][k]): 4 (mod 16) doubles
template <int WM, int WN, int WTN = 32>
struct V2Cfg {  // WM warps along m x WN along n, warp tile 32 x WTN (WTN 32 or 64)
  static constexpr int BM = 32 * WM, BN = WTN * WN, PA = BM + 8, PB = BN + 8, THREADS = 32 * WM * WN;
  static constexpr int ASZ = (V2K * PA > BM * PK) ? V2K * PA : BM * PK;  // per-stage A tile
  static constexpr int BSZ = (V2K * PB > BN * PK) ? V2K * PB : BN * PK;  // per-stage B tile
  static constexpr int SMEM = V2S * (ASZ + BSZ) * 8;
  // CTAs per SM the register budget is sized for: 64 x 64 tiles 3 (170 registers: the 128 of
  // 4 per SM spilled, and the split-K sizing already fills 3 per SM — l = 256 Gram 359 -> 312 us,
  // C0 P 281 -> 257 us; 2 per SM measured slower), 128 x 64 tiles 2
  static constexpr int MINB = WTN == 64 ? (WM * WN <= 4 ? 2 : 1) : (WN == 2 ? (WM == 2 ? 3 : 4 / (WM / 2)) : (WM == 2 ? 2 : 1));
};

// 8-byte async copy global -> shared; pred false zero-fills (src-size 0: nothing is read,
// the in-bounds base pointer is passed instead of the out-of-range address)
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, const double* base, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(pred ? gmem : base), "r"(sz));
}
// 16-byte async copy with a byte count (16, 8 or 0): the rest of the 16 bytes is zero-filled
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, const double* base, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(bytes ? gmem : base), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// VEC: both operands staged by 16-byte copies of element pairs along their contiguous dimension
// (the caller guarantees 16-byte aligned pairs: unit stride, even other stride, aligned base):
// half the cp.async instructions and per-element source pointers of the 8-byte path
template <bool UPPER, bool A_KFAST, bool B_KFAST, int WM, int WN, int WTN = 32, bool VEC = false>
__global__ void __launch_bounds__(32 * WM * WN, V2Cfg<WM, WN, WTN>::MINB) dgemm_v2_kernel(int64_t M, int64_t N, int64_t Ktot,
                                                                       int64_t kchunk, double alpha, CMat A, CMat B,
                                                                       double beta, Mat C, int64_t zstride,
                                                                       const int2* __restrict__ kr,
                                                                       const int4* __restrict__ items, int btri,
                                                                       int rast) {
  pdl_begin();
  using Cfg = V2Cfg<WM, WN, WTN>;
  constexpr int BMt = Cfg::BM, BN = Cfg::BN, PA = Cfg::PA, PB = Cfg::PB, NT = Cfg::THREADS, NW = NT / 32;
  constexpr int NJ = WTN / 8, NB32 = BN / 32;
  constexpr int ASZ = Cfg::ASZ, BSZ = Cfg::BSZ;
  // VEC pitches: k-contiguous rows 18 doubles (2 mod 4: the 16-byte fragment loads of a quarter
  // warp hit distinct banks), k-major rows BM + 2 / BN + 2 (4 pitches = 8 mod 16: the k = 4t + s
  // fragment reads touch every bank twice); both within the V2Cfg stage sizes
  constexpr int PKv = VEC ? 18 : PK, PAv = VEC ? BMt + 2 : PA, PBv = VEC ? BN + 2 : PB;
  extern __shared__ __align__(16) double sm2[];
  double* As = sm2;                         // [V2S][ASZ]: [k][PA] (m-contiguous A) or [m][PK] (k-contiguous)
  double* Bs = sm2 + V2S * ASZ;             // [V2S][BSZ]: [k][PB] (n-contiguous B) or [n][PK] (k-contiguous)
  // rasterisation: the N tiles of one M tile on consecutive CTAs (N fastest), so a tall A
  // (s x K, e.g. 1.1e5 x 128) is read from DRAM once and its re-reads by the other N tiles
  // hit L2 (M-fastest order streamed it once per N tile)
  unsigned bx = blockIdx.x, by = blockIdx.y;
  if (!items && gridDim.y > 1 && rast) {
    const unsigned lin = blockIdx.x + gridDim.x * blockIdx.y;
    by = lin % gridDim.y;
    bx = lin / gridDim.y;
  }
  int64_t m0 = (int64_t)bx * BMt;
  const int64_t n0 = (int64_t)by * BN;
  if (UPPER && m0 > n0 + BN - 1) return;
  int64_t kbeg, K;
  if (items) {  // balanced split: work item (row tile, k begin, k end), partial tile of its own
    const int4 it = items[blockIdx.x];
    if (it.x < 0) return;
    m0 = (int64_t)it.x * BMt;
    kbeg = it.y;
    K = it.z - it.y;
    C.p += (int64_t)blockIdx.x * zstride - m0 * C.rs;  // row m0 -> the item's buffer start
  } else if (kr) {  // structurally nonzero K range of this row tile (union of its 64-row blocks)
    const int b0 = (int)(m0 >> 6);
    int2 r = kr[b0];
    if (BMt > 64 && m0 + 64 < M) {
      const int2 r1 = kr[b0 + 1];
      r.x = min(r.x, r1.x);
      r.y = max(r.y, r1.y);
    }
    const int64_t len = max(0, r.y - r.x);
    const int64_t ck = ((len + gridDim.z - 1) / gridDim.z + V2K - 1) / V2K * V2K;
    kbeg = r.x + (int64_t)blockIdx.z * ck;
    K = max((int64_t)0, min((int64_t)r.y - kbeg, ck));
  } else {
    kbeg = (int64_t)blockIdx.z * kchunk;
    K = min(Ktot - kbeg, kchunk);
    // btri: B is upper triangular (B[k][n] = 0 for k > n): this N tile needs k < n0 + BN only
    if (btri) K = max((int64_t)0, min(K, min(Ktot, n0 + BN) - kbeg));
  }
  A.p += kbeg * A.cs;
  B.p += kbeg * B.rs;
  if (!items) C.p += (int64_t)blockIdx.z * zstride;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp / WN) * 32, wn = (warp % WN) * WTN;

  auto load_stage = [&](int stage, int64_t k0) {
    double* as = As + stage * ASZ;
    double* bs = Bs + stage * BSZ;
    if constexpr (VEC) {
      // A tile: BM x V2K elements = BM / 4 warp-units of 32 pairs
#pragma unroll
      for (int r = 0; r < (BMt / 4 + NW - 1) / NW; ++r) {
        const int u = warp + NW * r;
        if (BMt / 4 % NW != 0 && u >= BMt / 4) break;
        int m, k, bytes;
        if (A_KFAST) {  // unit = 4 m x 16 k (pairs along k), stored [m][k]
          m = u * 4 + (lane >> 3);
          k = (lane & 7) * 2;
          const int64_t gm = m0 + m, gk = k0 + k;
          bytes = gm < M ? (gk + 1 < K ? 16 : (gk < K ? 8 : 0)) : 0;
          cp_async16(as + m * PKv + k, A.p + gm * A.rs + gk, A.p, bytes);
        } else {        // unit = 64 m x 1 k (pairs along m), stored [k][m]
          m = (u % (BMt / 64)) * 64 + lane * 2;
          k = u / (BMt / 64);
          const int64_t gm = m0 + m, gk = k0 + k;
          bytes = gk < K ? (gm + 1 < M ? 16 : (gm < M ? 8 : 0)) : 0;
          cp_async16(as + k * PAv + m, A.p + gm + gk * A.cs, A.p, bytes);
        }
      }
      // B tile: V2K x BN elements = BN / 4 warp-units of 32 pairs
#pragma unroll
      for (int r = 0; r < (BN / 4 + NW - 1) / NW; ++r) {
        const int u = warp + NW * r;
        if (BN / 4 % NW != 0 && u >= BN / 4) break;
        int n, k, bytes;
        if (B_KFAST) {  // unit = 4 n x 16 k, stored [n][k]
          n = u * 4 + (lane >> 3);
          k = (lane & 7) * 2;
          const int64_t gn = n0 + n, gk = k0 + k;
          bytes = gn < N ? (gk + 1 < K ? 16 : (gk < K ? 8 : 0)) : 0;
          cp_async16(bs + n * PKv + k, B.p + gk + gn * B.cs, B.p, bytes);
        } else {        // unit = 64 n x 1 k, stored [k][n]
          n = (u % (BN / 64)) * 64 + lane * 2;
          k = u / (BN / 64);
          const int64_t gn = n0 + n, gk = k0 + k;
          bytes = gk < K ? (gn + 1 < N ? 16 : (gn < N ? 8 : 0)) : 0;
          cp_async16(bs + k * PBv + n, B.p + gk * B.rs + gn, B.p, bytes);
        }
      }
      return;
    }
    // A tile: BM x V2K elements = BM / 2 warp-units of 32
#pragma unroll
    for (int r = 0; r < (BMt / 2 + NW - 1) / NW; ++r) {
      int m, k;
      const int u = warp + NW * r;        // unit 0 .. BM/2 - 1
      if (BMt / 2 % NW != 0 && u >= BMt / 2) break;
      if (A_KFAST) {  // unit = 2 m x 16 k (two 128-byte rows), stored [m][k]
        m = u * 2 + (lane >> 4);
        k = lane & 15;
      } else {        // unit = 32 m x 1 k, stored [k][m]
        m = (u % WM) * 32 + lane;
        k = u / WM;
      }
      const int64_t gm = m0 + m, gk = k0 + k;
      const bool ok = gm < M && gk < K;
      cp_async8(as + (A_KFAST ? m * PK + k : k * PA + m), A.p + gm * A.rs + gk * A.cs, A.p, ok);
    }
    // B tile: V2K x BN elements = BN / 2 warp-units
#pragma unroll
    for (int r = 0; r < (BN / 2 + NW - 1) / NW; ++r) {
      int n, k;
      const int u = warp + NW * r;        // unit 0 .. BN/2 - 1
      if (BN / 2 % NW != 0 && u >= BN / 2) break;
      if (B_KFAST) {  // unit = 2 n x 16 k, stored [n][k]
        n = u * 2 + (lane >> 4);
        k = lane & 15;
      } else {        // unit = 32 n x 1 k, stored [k][n]
        n = (u % NB32) * 32 + lane;
        k = u / NB32;
      }
      const int64_t gn = n0 + n, gk = k0 + k;
      const bool ok = gn < N && gk < K;
      cp_async8(bs + (B_KFAST ? n * PK + k : k * PB + n), B.p + gk * B.rs + gn * B.cs, B.p, ok);
    }
  };

  double acc[4][NJ][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t nk = (K + V2K - 1) / V2K;
#pragma unroll
  for (int sgi = 0; sgi < V2S - 1; ++sgi) {
    if (sgi < nk) load_stage(sgi, (int64_t)sgi * V2K);
    cp_async_commit();
  }
  for (int64_t kt = 0; kt < nk; ++kt) {
    cp_async_wait<V2S - 2>();
    __syncthreads();
    {  // refill the stage consumed two iterations ago
      const int64_t kn = kt + V2S - 1;
      if (kn < nk) load_stage((int)(kn % V2S), kn * V2K);
      cp_async_commit();
    }
    const double* as = As + (int)(kt % V2S) * ASZ;
    const double* bs = Bs + (int)(kt % V2S) * BSZ;
    // upper variant: a warp whose 32 x WTN sub-tile lies strictly below the diagonal writes
    // nothing, so it only helps stage the operands (a quarter of each diagonal 64 x 64 tile's MMAs)
    if (UPPER && m0 + wm > n0 + wn + WTN - 1) continue;
    if constexpr (VEC) {
      // the k tile's 16 steps taken as k = 4t + s (s = 0..3) by lane t (the sum over k is the same;
      // A and B agree): a k-contiguous operand's fragments for s and s + 1 are one 16-byte load
#pragma unroll
      for (int sp = 0; sp < 4; sp += 2) {
        double a[2][4], b[2][NJ];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (A_KFAST) {
            const double2 v = *reinterpret_cast<const double2*>(as + (wm + i * 8 + g) * PKv + 4 * t + sp);
            a[0][i] = v.x;
            a[1][i] = v.y;
          } else {
            a[0][i] = as[(4 * t + sp) * PAv + wm + i * 8 + g];
            a[1][i] = as[(4 * t + sp + 1) * PAv + wm + i * 8 + g];
          }
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          if (B_KFAST) {
            const double2 v = *reinterpret_cast<const double2*>(bs + (wn + j * 8 + g) * PKv + 4 * t + sp);
            b[0][j] = v.x;
            b[1][j] = v.y;
          } else {
            b[0][j] = bs[(4 * t + sp) * PBv + wn + j * 8 + g];
            b[1][j] = bs[(4 * t + sp + 1) * PBv + wn + j * 8 + g];
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], a[h][i], b[h][j]);
      }
      continue;
    }
#pragma unroll
    for (int kk = 0; kk < V2K; kk += 4) {
      double a[4], b[NJ];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        a[i] = A_KFAST ? as[(wm + i * 8 + g) * PK + kk + t] : as[(kk + t) * PA + wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        b[j] = B_KFAST ? bs[(wn + j * 8 + g) * PK + kk + t] : bs[(kk + t) * PB + wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
  // row-major C with 16-byte rows: each lane's column pair (2t, 2t+1) as one 16-byte load /
  // store (full sectors; the element-wise epilogue dominated the short-K products, e.g. the
  // K = 64 SYRK of the Gram)
  const bool vec = C.cs == 1 && (C.rs & 1) == 0 && (((uintptr_t)C.p) & 15) == 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + wm + i * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int64_t col0 = n0 + wn + j * 8 + 2 * t;
      if (vec && col0 + 1 < N && (!UPPER || row <= col0)) {
        double2* c2 = reinterpret_cast<double2*>(C.p + row * C.rs + col0);
        double2 v = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
        if (beta != 0.0) {
          const double2 o = *c2;
          v.x += beta * o.x;
          v.y += beta * o.y;
        }
        *c2 = v;
        continue;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t col = col0 + h;
        if (col >= N || (UPPER && row > col)) continue;
        double* c = C.p + row * C.rs + col * C.cs;
        double v = alpha * acc[i][j][h];
        if (beta != 0.0) v += beta * (*c);
        *c = v;
      }
    }
  }
}

template <bool U, bool AK, bool BK_, int WM, int WN, int WTN, bool VEC = false>
cudaError_t launch_v2(dim3 grid, cudaStream_t st, int64_t M, int64_t N, int64_t K, int64_t kchunk, double alpha,
                      CMat A, CMat B, double beta, Mat C, int64_t zs, const int2* kr, const int4* items, int btri) {
  using Cfg = V2Cfg<WM, WN, WTN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dgemm_v2_kernel<U, AK, BK_, WM, WN, WTN, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg::SMEM);
    attr = true;
  }
  static const int rast = getenv("TSVD_GEMM_RAST") ? atoi(getenv("TSVD_GEMM_RAST")) : 1;  // tuning: 0 = M fastest
  launch_k(dgemm_v2_kernel<U, AK, BK_, WM, WN, WTN, VEC>, grid, Cfg::THREADS, Cfg::SMEM, st, M, N, K, kchunk, alpha, A, B, beta, C,
                                                                             zs, kr, items, btri, rast);
  return cudaGetLastError();
}

// 16-byte staging applies when both operands' contiguous dimension has unit stride, the other
// stride is even and the bases are 16-byte aligned (64 x 64 tiles only: the default)
inline bool vec_ok(bool ak, bool bk, const CMat& A, const CMat& B) {
  const bool a = ak ? (A.cs == 1 && (A.rs & 1) == 0) : (A.rs == 1 && (A.cs & 1) == 0);
  const bool b = bk ? (B.rs == 1 && (B.cs & 1) == 0) : (B.cs == 1 && (B.rs & 1) == 0);
  return a && b && (((uintptr_t)A.p) & 15) == 0 && (((uintptr_t)B.p) & 15) == 0;
}

template <int WM, int WN, int WTN = 32>
cudaError_t launch_v2_any(bool upper, bool ak, bool bk, dim3 grid, cudaStream_t st, int64_t M, int64_t N, int64_t K,
                          int64_t kchunk, double alpha, CMat A, CMat B, double beta, Mat C, int64_t zs,
                          const int2* kr, const int4* items = nullptr, int btri = 0) {
  static const bool vec_on = !(getenv("TSVD_GEMM_VEC") && atoi(getenv("TSVD_GEMM_VEC")) == 0);
  if constexpr (WM == 2 && WN == 2 && WTN == 32) {
    // (K ranges / balanced items: the ranges' starts must be even — core_kr_kernel rounds them
    // down — or a k-contiguous operand's pairs would be misaligned)
    if (vec_on && vec_ok(ak, bk, A, B)) {
#define V2V(U, X, Y) return launch_v2<U, X, Y, WM, WN, WTN, true>(grid, st, M, N, K, kchunk, alpha, A, B, beta, C, zs, kr, items, btri)
      if (upper) {
        if (ak) { if (bk) V2V(true, true, true); V2V(true, true, false); }
        if (bk) V2V(true, false, true);
        V2V(true, false, false);
      }
      if (ak) { if (bk) V2V(false, true, true); V2V(false, true, false); }
      if (bk) V2V(false, false, true);
      V2V(false, false, false);
#undef V2V
    }
  }
#define V2L(U, X, Y) return launch_v2<U, X, Y, WM, WN, WTN>(grid, st, M, N, K, kchunk, alpha, A, B, beta, C, zs, kr, items, btri)
  if (upper) {
    if (ak) { if (bk) V2L(true, true, true); V2L(true, true, false); }
    if (bk) V2L(true, false, true);
    V2L(true, false, false);
  }
  if (ak) { if (bk) V2L(false, true, true); V2L(false, true, false); }
  if (bk) V2L(false, false, true);
  V2L(false, false, false);
#undef V2L
}

// C = alpha sum_z part[z] + beta C  (part: nz slices of M x N row-major)
template <bool UPPER>
__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int nz, const double* __restrict__ part, double alpha,
                                     double beta, Mat C) {
  pdl_begin();
  const int64_t mn = M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < mn; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i, j;
    divmod_idx(e, N, i, j);
    if (UPPER && i > j) continue;
    double acc = 0.0;
    for (int z = 0; z < nz; ++z) acc += part[(int64_t)z * mn + e];
    double* c = C.p + i * C.rs + j * C.cs;
    double v = alpha * acc;
    if (beta != 0.0) v += beta * (*c);
    *c = v;
  }
}

// Balanced split of a structured product (kr given): every row tile's K range [x, y) (the
// union over its 64-row blocks) is cut into chunks of at most ck, the work items listed tile
// by tile (items[i] = {tile, k0, k1}; unused slots {-1}) with off[t] = the tile's first item —
// equal-length CTAs instead of a fixed number of slices per tile, whose lengths followed the
// triangular structure.  One block; cap = the item capacity.
__global__ void kr_plan_kernel(const int2* __restrict__ kr, int64_t M, int bm, int tiles, int ck, int4* items,
                               int* off, int cap) {
  pdl_begin();
  __shared__ int cnt_s[1025];
  __shared__ int2 rng_s[1024];
  const int nb64 = (int)((M + 63) / 64);
  for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
    const int b0 = (int)(((int64_t)t * bm) >> 6), b1 = min(nb64, b0 + bm / 64);
    int2 r = kr[b0];
    for (int b = b0 + 1; b < b1; ++b) {
      r.x = min(r.x, kr[b].x);
      r.y = max(r.y, kr[b].y);
    }
    const int len = max(0, r.y - r.x);
    rng_s[t] = r;
    cnt_s[t] = max(1, (len + ck - 1) / ck);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int t = 0; t < tiles; ++t) {
      off[t] = acc;
      acc += cnt_s[t];
    }
    off[tiles] = acc;
    cnt_s[tiles] = acc;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
    const int2 r = rng_s[t];
    const int len = max(0, r.y - r.x), n = cnt_s[t], o = off[t];
    // chunk boundaries on multiples of the K step (16), as even as that allows
    const int per = ((len + n - 1) / n + 15) / 16 * 16;
    for (int c = 0; c < n; ++c) {
      const int k0 = min(r.y, r.x + c * per), k1 = min(r.y, r.x + (c + 1) * per);
      items[o + c] = make_int4(t, k0, max(k0, k1), 0);
    }
  }
  for (int i = cnt_s[tiles] + threadIdx.x; i < cap; i += blockDim.x) items[i] = make_int4(-1, 0, 0, 0);
}

// C = alpha sum_(items of the row's tile, in order) part[item] + beta C.  N even and C row-major
// with 16-byte rows: two columns per thread (16-byte loads of the partials and of C).
__global__ void items_reduce2_kernel(int64_t M, int64_t N, int bm, const int* __restrict__ off,
                                     const double* __restrict__ part, double alpha, double beta, Mat C) {
  pdl_begin();
  const int64_t h = N / 2, mh = M * h;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < mh; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i, jh;
    divmod_idx(e, h, i, jh);
    const int t = (int)(i / bm);
    const int64_t loc = (i - (int64_t)t * bm) * N + 2 * jh;
    double ax = 0.0, ay = 0.0;
    for (int it = off[t]; it < off[t + 1]; ++it) {
      const double2 p = *reinterpret_cast<const double2*>(part + (int64_t)it * bm * N + loc);
      ax += p.x;
      ay += p.y;
    }
    double2* c = reinterpret_cast<double2*>(C.p + i * C.rs + 2 * jh);
    double2 v = make_double2(alpha * ax, alpha * ay);
    if (beta != 0.0) {
      const double2 o = *c;
      v.x += beta * o.x;
      v.y += beta * o.y;
    }
    *c = v;
  }
}

__global__ void items_reduce_kernel(int64_t M, int64_t N, int bm, const int* __restrict__ off,
                                    const double* __restrict__ part, double alpha, double beta, Mat C) {
  pdl_begin();
  const int64_t mn = M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < mn; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i, j;
    divmod_idx(e, N, i, j);
    const int t = (int)(i / bm);
    const int64_t loc = (i - (int64_t)t * bm) * N + j;
    double acc = 0.0;
    for (int it = off[t]; it < off[t + 1]; ++it) acc += part[(int64_t)it * bm * N + loc];
    double* c = C.p + i * C.rs + j * C.cs;
    double v = alpha * acc;
    if (beta != 0.0) v += beta * (*c);
    *c = v;
  }
}
}  // namespace

namespace {
// split-K partial buffers come from the stream-ordered pool: keep freed memory pooled (the
// default release threshold of 0 returns it at every synchronisation)
void keep_pool_warm() {
  static thread_local int dev_done = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == dev_done) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  dev_done = dev;
}
}  // namespace

namespace {
// Plans of the balanced split, reused while the K ranges they were made from are unchanged:
// the core iteration calls the same two structured products ~10 times per update with the same
// kr arrays.  Keyed by (stream, kr, M, K, bm, ck, tiles) and the epoch core_svd advances
// whenever it writes K ranges (a kr buffer reused later with other contents never hits).
std::atomic<uint64_t> g_kr_epoch{1};
struct PlanEntry {
  int dev = -1;            // device the buffer lives on (plans never cross devices)
  cudaEvent_t done = nullptr;  // recorded after the last launch that read the buffer
  cudaStream_t st = nullptr;
  const int2* kr = nullptr;
  int64_t M = 0, K = 0;
  int bm = 0, ck = 0, tiles = 0, cap = 0;
  uint64_t epoch = 0;
  int4* items = nullptr;  // cap items, then tiles + 1 offsets
  size_t bytes = 0;
  uint64_t used = 0;
};
std::mutex g_plan_mu;
cudaError_t kr_plan_get(cudaStream_t st, const int2* kr, int64_t M, int64_t K, int bm, int ck, int tiles, int cap,
                        int4** items, int** off, bool* fresh, PlanEntry** entry) {
  static PlanEntry ent[8];
  static uint64_t clock = 0;
  std::lock_guard<std::mutex> lk(g_plan_mu);
  const uint64_t ep = g_kr_epoch.load();
  int dev = 0;
  cudaGetDevice(&dev);
  PlanEntry* victim = &ent[0];
  for (auto& x : ent) {
    if (x.items && x.dev == dev && x.st == st && x.kr == kr && x.M == M && x.K == K && x.bm == bm && x.ck == ck && x.tiles == tiles &&
        x.cap == cap && x.epoch == ep) {
      x.used = ++clock;
      *items = x.items;
      *off = reinterpret_cast<int*>(x.items + cap);
      *fresh = false;
      *entry = &x;
      return cudaSuccess;
    }
    if (x.used < victim->used) victim = &x;
  }
  // the victim's last reader (any stream, possibly one destroyed since) is done once its
  // event has completed; its buffer is then free to be reused or released
  if (victim->done) {
    int cur = 0;
    cudaGetDevice(&cur);
    if (victim->dev >= 0 && victim->dev != cur) cudaSetDevice(victim->dev);
    cudaEventSynchronize(victim->done);
    if (victim->dev != dev) {
      cudaFree(victim->items);
      cudaEventDestroy(victim->done);
      victim->items = nullptr;
      victim->done = nullptr;
      victim->bytes = 0;
    }
    cudaSetDevice(cur);
  }
  // at least 1 MB: later plans of slightly different shapes reuse the buffer (no cudaMalloc /
  // cudaFree, which synchronise the device, inside the update)
  const size_t need = std::max<size_t>((size_t)cap * sizeof(int4) + (size_t)(tiles + 1) * sizeof(int), size_t(1) << 20);
  if (victim->bytes < need) {
    if (victim->items) cudaFree(victim->items);
    victim->items = nullptr;
    victim->bytes = 0;
    cudaError_t e = cudaMalloc(&victim->items, need);
    if (e) return e;
    victim->bytes = need;
  }
  if (!victim->done) {
    cudaError_t e = cudaEventCreateWithFlags(&victim->done, cudaEventDisableTiming);
    if (e) return e;
  }
  victim->dev = dev;
  victim->st = st;
  victim->kr = kr;
  victim->M = M;
  victim->K = K;
  victim->bm = bm;
  victim->ck = ck;
  victim->tiles = tiles;
  victim->cap = cap;
  victim->epoch = ep;
  victim->used = ++clock;
  *items = victim->items;
  *off = reinterpret_cast<int*>(victim->items + cap);
  *fresh = true;
  *entry = victim;
  return cudaSuccess;
}
}  // namespace

void kr_plan_epoch_bump() { g_kr_epoch.fetch_add(1); }

cudaError_t dgemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, CMat A, CMat B, double beta,
                  Mat C, int uplo, const int2* kr, double kfrac, bool b_upper) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  keep_pool_warm();
  static const bool trace = getenv("TSVD_GEMM_TRACE") != nullptr;  // shape log (tuning)
  if (trace)
    fprintf(stderr, "[gemm] M=%lld N=%lld K=%lld uplo=%d kr=%d kfrac=%.3f btri=%d A=(%lld,%lld) B=(%lld,%lld) beta=%g\n",
            (long long)M, (long long)N, (long long)K, uplo, kr ? 1 : 0, kr ? kfrac : 1.0, b_upper ? 1 : 0,
            (long long)A.rs, (long long)A.cs, (long long)B.rs, (long long)B.cs, beta);
  // K4 accounting: 2MNK flops (half for the upper-triangle variant), operands + C read/write
  // (kr: the caller's fraction kfrac of the M x K operand that is structurally nonzero)
  const double kf = kr ? kfrac : (b_upper ? std::min(1.0, 0.5 * (N + 1) / (double)std::max<int64_t>(K, 1)) : 1.0);
  KScope sc(KC_GEMM, (uplo ? 1.0 : 2.0) * (double)M * N * K * kf,
            8.0 * ((double)M * K + (double)K * N * (b_upper ? 0.5 : 1.0) + (beta != 0.0 ? 2.0 : 1.0) * M * N));
  // v2 (pipelined) when each operand has a unit-stride dimension
  const bool a_k = A.cs == 1, a_m = A.rs == 1, b_k = B.rs == 1, b_n = B.cs == 1;
  if ((a_k || a_m) && (b_k || b_n) && K > 0) {
    // N tile 96 (3 warps along n) when N is 65..96 or a multiple of 96 but not of 64 (the core
    // reduction's b = 96 blocks), else 64; 64-row tiles (below)
    const bool n96 = (N > 64 && N <= 96) || (N % 96 == 0 && N % 64 != 0);
    int bn = n96 ? 96 : V2N;
    static const int big_env = getenv("TSVD_GEMM_BIG") ? atoi(getenv("TSVD_GEMM_BIG")) : -1;  // tuning
    // split-K shapes (few output tiles, long K): TSVD_SPLIT_BIG=1 tries 128-row tiles (tuning)
    static const int split_big = getenv("TSVD_SPLIT_BIG") ? atoi(getenv("TSVD_SPLIT_BIG")) : 0;
    const bool splitk_shape = (int64_t)cdiv(M, 64) * cdiv(N, bn) < 148 && K >= 4096;
    // 64-row tiles by default: at 3 CTAs per SM they beat the 128-row tiles at 2 on every
    // measured shape (configs[3] apply X T 504 -> 484 us, 4096^3 30.2 -> 31.2 TF/s; C4 9.3 ->
    // 9.4M nnz/s, C5 1.12 -> 1.13M rows/s); TSVD_GEMM_BIG=1 / TSVD_SPLIT_BIG=1 bring them back
    const bool big = big_env >= 0 ? (big_env == 1 && M >= 1024) : (split_big && splitk_shape && M >= 128);
    // warp tile 32 x 64 (half the fragment loads per DMMA of 32 x 32): TSVD_GEMM_WIDE=1 a
    // 64 x 128 CTA tile of 4 warps, =2 a 128 x 64 tile of 4 warps, for the tiles of `big`
    static const int wide_env = getenv("TSVD_GEMM_WIDE") ? atoi(getenv("TSVD_GEMM_WIDE")) : 0;  // tuning
    const int wide = (big && !n96) ? wide_env : 0;
    const int bm = wide == 1 ? 64 : (big ? V2M : 64);
    if (wide == 1) bn = 128;
    dim3 grid(cdiv(M, bm), cdiv(N, bn));
    if (grid.y > 65535) return cudaErrorInvalidValue;
    const int64_t tiles = (int64_t)grid.x * grid.y;
    int nz = 1;
    // split-K for few output tiles: size the split by the tiles that do work (the upper
    // variant skips the tiles below the diagonal) so that the CTAs fill every SM's resident
    // slots (148 x 4 for the 64-row tiles, 148 x 2 for the 128-row ones) in one wave — a split
    // sized by all tiles left a third of the SMs with two CTAs' work and the rest with one
    // (the RPI l x l Grams: 14 TF/s)
    int64_t active = tiles;
    if (uplo) {
      active = 0;
      for (int64_t i = 0; i < (int64_t)grid.x; ++i)
        for (int64_t j = 0; j < (int64_t)grid.y; ++j) active += (i * bm <= j * bn + bn - 1) ? 1 : 0;
    }
    static const int slots_env = getenv("TSVD_SPLIT_SLOTS") ? atoi(getenv("TSVD_SPLIT_SLOTS")) : 0;  // tuning
    // 3 CTAs per SM for the 64-row tiles (measured on the configs[3] shapes, tools/micro_gemm_c4.py:
    // 4 per SM 464 / 3 per SM 359 us for the l = 256 Gram, 354 / 280 us for C0 P)
    // two waves of them (configs[3]'s C0 P 246 -> 244 us, l = 256 Gram 309 -> 307, 384^2 core
    // 1083 -> 1035 measured with the 16-byte path; one wave of 444 CTAs left the slowest slice's
    // tail exposed)
    const int64_t slots = slots_env > 0 ? slots_env : 2 * 148 * (bm == 64 ? 3 : 2);
    if (active < 148 && K >= 256)
      nz = (int)std::min<int64_t>(std::min<int64_t>(std::max<int64_t>(1, slots / active), K / 64), 128);
    // ragged K ranges: twice the split so that the short row tiles' CTAs leave room for the
    // long ones (several waves balance; one wave would last as long as the longest tile)
    if (kr && tiles < 296 && K >= 256) nz = (int)std::min<int64_t>(std::min<int64_t>(cdiv(592, tiles), K / 64), 64);
    const int bt = (b_upper && !kr) ? 1 : 0;
    auto L = [&](dim3 gr, int64_t kc, double al, double be, Mat Cm, int64_t zs) {
      if (n96)
        return big ? launch_v2_any<4, 3>(uplo != 0, a_k, b_k && !b_n, gr, st, M, N, K, kc, al, A, B, be, Cm, zs, kr, nullptr, bt)
                   : launch_v2_any<2, 3>(uplo != 0, a_k, b_k && !b_n, gr, st, M, N, K, kc, al, A, B, be, Cm, zs, kr, nullptr, bt);
      if (wide == 1)
        return launch_v2_any<2, 2, 64>(uplo != 0, a_k, b_k && !b_n, gr, st, M, N, K, kc, al, A, B, be, Cm, zs, kr, nullptr, bt);
      if (wide == 2)
        return launch_v2_any<4, 1, 64>(uplo != 0, a_k, b_k && !b_n, gr, st, M, N, K, kc, al, A, B, be, Cm, zs, kr, nullptr, bt);
      return big ? launch_v2_any<4, 2>(uplo != 0, a_k, b_k && !b_n, gr, st, M, N, K, kc, al, A, B, be, Cm, zs, kr, nullptr, bt)
                 : launch_v2_any<2, 2>(uplo != 0, a_k, b_k && !b_n, gr, st, M, N, K, kc, al, A, B, be, Cm, zs, kr, nullptr, bt);
    };
    static const int bal_ck = getenv("TSVD_GEMM_CK") ? atoi(getenv("TSVD_GEMM_CK")) : 256;  // 0: off
    if (kr && !uplo && bal_ck > 0 && grid.y == 1 && tiles <= 1024 && K >= 256) {
      const int ck = std::max(16, bal_ck / 16 * 16);
      const int cap = (int)std::min<int64_t>(tiles + cdiv(K, ck) * tiles, 1 << 20);
      double* part = nullptr;
      int4* items = nullptr;
      int* off = nullptr;
      bool fresh = false;
      PlanEntry* pe = nullptr;
      cudaError_t e = kr_plan_get(st, kr, M, K, bm, ck, (int)tiles, cap, &items, &off, &fresh, &pe);
      if (e) return e;
      const int64_t pst = (int64_t)bm * N;
      if ((e = cudaMallocAsync(&part, (size_t)cap * pst * sizeof(double), st))) return e;
      g_launches += fresh ? 3 : 2;
      if (fresh) launch_k(kr_plan_kernel, 1, 256, 0, st, kr, M, bm, (int)tiles, ck, items, off, cap);
      const dim3 gi((unsigned)cap, 1);
      const Mat pm{part, N, 1};
      cudaError_t e2;
      if (n96)
        e2 = big ? launch_v2_any<4, 3>(false, a_k, b_k && !b_n, gi, st, M, N, K, 0, 1.0, A, B, 0.0, pm, pst, kr, items)
                 : launch_v2_any<2, 3>(false, a_k, b_k && !b_n, gi, st, M, N, K, 0, 1.0, A, B, 0.0, pm, pst, kr, items);
      else if (wide == 1)
        e2 = launch_v2_any<2, 2, 64>(false, a_k, b_k && !b_n, gi, st, M, N, K, 0, 1.0, A, B, 0.0, pm, pst, kr, items);
      else if (wide == 2)
        e2 = launch_v2_any<4, 1, 64>(false, a_k, b_k && !b_n, gi, st, M, N, K, 0, 1.0, A, B, 0.0, pm, pst, kr, items);
      else
        e2 = big ? launch_v2_any<4, 2>(false, a_k, b_k && !b_n, gi, st, M, N, K, 0, 1.0, A, B, 0.0, pm, pst, kr, items)
                 : launch_v2_any<2, 2>(false, a_k, b_k && !b_n, gi, st, M, N, K, 0, 1.0, A, B, 0.0, pm, pst, kr, items);
      if (e2) return e2;
      const unsigned rb = (unsigned)std::min<int64_t>(cdiv(M * N, 256), 148 * 8);
      if ((N & 1) == 0 && C.cs == 1 && (C.rs & 1) == 0 && (((uintptr_t)C.p) & 15) == 0)
        launch_k(items_reduce2_kernel, (unsigned)std::min<int64_t>(cdiv(M * N / 2, 256), 148 * 8), 256, 0, st, M, N, bm,
                 (const int*)off, (const double*)part, alpha, beta, C);
      else
        launch_k(items_reduce_kernel, rb, 256, 0, st, M, N, bm, (const int*)off, (const double*)part, alpha, beta, C);
      {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        cudaEventRecord(pe->done, st);  // the plan buffer's last reader on this stream
      }
      cudaFreeAsync(part, st);
      return cudaGetLastError();
    }
    if (nz > 1) {
      const int64_t kchunk = ((K + nz - 1) / nz + V2K - 1) / V2K * V2K;
      nz = (int)cdiv(K, kchunk);
      double* part = nullptr;
      cudaError_t e = cudaMallocAsync(&part, (size_t)nz * M * N * sizeof(double), st);
      if (e) return e;
      grid.z = nz;
      g_launches += 2;
      if ((e = L(grid, kchunk, 1.0, 0.0, Mat{part, N, 1}, M * N))) return e;
      const unsigned rb = (unsigned)std::min<int64_t>(cdiv(M * N, 256), 148 * 8);
      if (uplo)
        launch_k(splitk_reduce_kernel<true>, rb, 256, 0, st, M, N, nz, part, alpha, beta, C);
      else
        launch_k(splitk_reduce_kernel<false>, rb, 256, 0, st, M, N, nz, part, alpha, beta, C);
      cudaFreeAsync(part, st);
      return cudaGetLastError();
    }
    ++g_launches;
    return L(grid, K, alpha, beta, C, 0);
  }
  dim3 grid(cdiv(M, BM), cdiv(N, BN));
  if (grid.y > 65535) return cudaErrorInvalidValue;
  const int64_t tiles = (int64_t)grid.x * grid.y;
  // split-K for tall-skinny products (few output tiles, long K): deterministic two-pass
  int nz = 1;
  if (tiles < 148 && K >= 2048) nz = (int)std::min<int64_t>(std::min<int64_t>(cdiv(296, tiles), K / 1024), 64);
  if (nz > 1) {
    const int64_t kchunk = ((K + nz - 1) / nz + BK - 1) / BK * BK;
    nz = (int)cdiv(K, kchunk);
    double* part = nullptr;
    cudaError_t e = cudaMallocAsync(&part, (size_t)nz * M * N * sizeof(double), st);
    if (e) return e;
    grid.z = nz;
    g_launches += 2;
    if (uplo)
      launch_k(dgemm_kernel<true>, grid, 128, 0, st, M, N, K, kchunk, 1.0, A, B, 0.0, Mat{part, N, 1}, M * N);
    else
      launch_k(dgemm_kernel<false>, grid, 128, 0, st, M, N, K, kchunk, 1.0, A, B, 0.0, Mat{part, N, 1}, M * N);
    const unsigned rb = (unsigned)std::min<int64_t>(cdiv(M * N, 256), 148 * 8);
    if (uplo)
      launch_k(splitk_reduce_kernel<true>, rb, 256, 0, st, M, N, nz, part, alpha, beta, C);
    else
      launch_k(splitk_reduce_kernel<false>, rb, 256, 0, st, M, N, nz, part, alpha, beta, C);
    cudaFreeAsync(part, st);
    return cudaGetLastError();
  }
  ++g_launches;
  if (uplo)
    launch_k(dgemm_kernel<true>, grid, 128, 0, st, M, N, K, K, alpha, A, B, beta, C, 0);
  else
    launch_k(dgemm_kernel<false>, grid, 128, 0, st, M, N, K, K, alpha, A, B, beta, C, 0);
  return cudaGetLastError();
}

cudaError_t dgemm_rm_btri(cudaStream_t st, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                          const double* B, int64_t ldb, double* C, int64_t ldc) {
  return dgemm(st, M, N, K, 1.0, CMat{A, lda, 1}, CMat{B, ldb, 1}, 0.0, Mat{C, ldc, 1}, 0, nullptr, 1.0, true);
}

cudaError_t dgemm_rm(cudaStream_t st, bool tA, bool tB, int64_t M, int64_t N, int64_t K, double alpha,
                     const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                     int64_t ldc, int uplo) {
  CMat a = tA ? CMat{A, 1, lda} : CMat{A, lda, 1};
  CMat b = tB ? CMat{B, 1, ldb} : CMat{B, ldb, 1};
  return dgemm(st, M, N, K, alpha, a, b, beta, Mat{C, ldc, 1}, uplo);
}

}  // namespace tsvd
