// dag.cu — the s x s Cholesky with deflation (K5, Alg 2 PAPER.md:251-272 read as DESIGN.md
// R8/R9) and the back substitution Y = R^+ X that consumes it (K6, Eq (5)), as
// persistent tile-DAG kernels.
//
// Why: the right-looking panel algorithm is a chain of ~s/64 (factor -> row solve -> update)
// steps, each a separate launch of a few tens of microseconds, so at s ~ 5000 it is latency
// bound (~7 ms per update measured on B200, against ~1 ms of DMMA work).  Here the whole
// factorisation is ONE launch of 2 CTAs per SM that pull 64 x 64 tile tasks from an ordered
// list with an atomic ticket and track dependencies with per-tile counters in global memory:
//   P(q)      factor the diagonal tile (q,q) (deflation test on the Schur diagonal) and form
//             T_qq = R_qq^+ (inverse over the kept pivots, zero rows / columns elsewhere);
//   S(q,c)    R(q,c) = T_qq^T A(q,c) (one 64^3 DMMA product; zeroes the mirror tile (c,q));
//   U(q;i,c)  A(i,c) -= R(q,i)^T R(q,c) (q < i <= c; applied in q order per tile).
// Task order is look-ahead 1: panel j's critical tasks (P(j), S(j,.), the updates of tile row
// j+1) are listed before the bulk of panel j-1's trailing updates, so the chain
// P(j) -> S(j,j+1) -> U(j;j+1,j+1) -> P(j+1) overlaps the bulk work.  Every dependency points to
// an earlier ticket, so a CTA only waits on tasks already claimed by running CTAs: no deadlock
// without cooperative launch.  The solve is the same machinery on the row tiles of X with the
// T_qq the factorisation left behind:
//   F(i)      X_i = T_ii X_i;        V(j;i)  X_i -= R(i,j) X_j   (j > i, applied in descending j).
// All operand traffic goes through L2 (ld/st .cg) so no SM can read a stale L1 line of a tile
// another SM rewrote; producers publish with __threadfence + a release store, consumers poll
// with an acquire load.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "ops.h"
#include "potrf.cuh"

namespace tsvd {

namespace {
constexpr int TB = 64;         // tile
constexpr int TP = TB + 8;     // smem pitch of [k][m] operands (== 8 mod 16: conflict-free fragments)
constexpr int SUB = 16;        // sub-panel of the diagonal factorisation
constexpr int DAG_THREADS = 256;
// [A | I] factor tile (TB x (2 TB + 4)) + one operand tile for the chain; three operand tiles
// (A + double-buffered B) for the strips
constexpr size_t DAG_SMEM_CHAIN = ((size_t)TB * (2 * TB + 4) + (size_t)TB * TP) * sizeof(double);
constexpr size_t DAG_SMEM_STRIP = 3 * (size_t)TB * TP * sizeof(double);
constexpr size_t DAG_SMEM = DAG_SMEM_CHAIN > DAG_SMEM_STRIP ? DAG_SMEM_CHAIN : DAG_SMEM_STRIP;
// one CTA per SM with the C tiles of a strip staged too (default; TSVD_DAG_CSTAGE=0: two CTAs)
constexpr size_t DAG_SMEM_CSTAGE = 5 * (size_t)TB * TP * sizeof(double);  // A, 2 x B, 2 x C
// back substitution: the chain double-buffers R(j-1, j) ([m][k], pitch RPT) and T_{j-1} ([k][m])
// next to the current X tile; one CTA per SM
constexpr int RPT = TB + 4;
constexpr size_t TRSM_SMEM = (2 * (size_t)TB * RPT + 2 * (size_t)TB * TP + (size_t)TB * TP) * sizeof(double);

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
// task trace (thread 0 only): claimed / dependencies met / published
struct TaskTrace {
  long long* p;
  long long t0 = 0, t1 = 0;
  __device__ __forceinline__ void claimed() {
    if (p && threadIdx.x == 0) t0 = gtimer();
  }
  __device__ __forceinline__ void ready() {
    if (p && threadIdx.x == 0) t1 = gtimer();
  }
  __device__ __forceinline__ void done(int it, int type) {
    if (p && threadIdx.x == 0) {
      long long* r = p + 4 * (int64_t)it;
      r[0] = type | ((long long)smid() << 8);
      r[1] = t0;
      r[2] = t1;
      r[3] = gtimer();
    }
  }
};

__device__ __forceinline__ int tile_n(int64_t rem) { return rem < TB ? (int)rem : TB; }

enum : int { T_CHAIN = 0, T_S = 1, T_U = 2, T_W = 3, T_V = 4 };
constexpr int STRIP = 4;  // bulk updates: one task per STRIP tiles of a tile row (R(q,i) staged once)

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// thread 0 spins until *p >= v; the CTA continues together
__device__ __forceinline__ void wait_ge(const int* p, int v) {
  if (threadIdx.x == 0)
    while (ld_acquire(p) < v) __nanosleep(32);
  __syncthreads();
}
// up to three dependencies polled concurrently (thread t waits on the t-th), one barrier
__device__ __forceinline__ void wait_all(const int* p0, int v0, const int* p1 = nullptr, int v1 = 0,
                                         const int* p2 = nullptr, int v2 = 0) {
  const int t = threadIdx.x;
  const int* p = t == 0 ? p0 : (t == 1 ? p1 : (t == 2 ? p2 : nullptr));
  const int v = t == 0 ? v0 : (t == 1 ? v1 : v2);
  if (p)
    while (ld_acquire(p) < v) __nanosleep(32);
  __syncthreads();
}
__device__ __forceinline__ void publish(int* p, int v) {
  __syncthreads();
  if (threadIdx.x == 0) st_release(p, v);  // release is cumulative over the CTA's writes ordered by the barrier
}

// smem[k][m] (pitch TP) <- the 64 x 64 block at src (row-major, ld), rows < nr and cols < nc
// valid (zero elsewhere); TRANS: smem[k][m] = src[m][k].  Thread t moves column t % 64 of rows
// t / 64 + 4u; the loads of a half (8 per thread, coalesced 512-byte rows) are all issued
// before the first is consumed, so a tile costs two L2 round trips, not sixteen.
template <bool TRANS>
struct Stage {
  double* sm;
  const double* src;
  int64_t ld;
  int nr, nc;
  double v[8];
  __device__ __forceinline__ void load(int h) {
    const int c = threadIdx.x & (TB - 1), r0 = threadIdx.x >> 6;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = r0 + 4 * (8 * h + u);
      v[u] = (r < nr && c < nc) ? __ldcg(src + (int64_t)r * ld + c) : 0.0;
    }
  }
  __device__ __forceinline__ void store(int h) {
    const int c = threadIdx.x & (TB - 1), r0 = threadIdx.x >> 6;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = r0 + 4 * (8 * h + u);
      if (TRANS) sm[c * TP + r] = v[u];
      else sm[r * TP + c] = v[u];
    }
  }
};
// both operand tiles of a task, 16 loads in flight per thread
template <bool TA, bool TBT>
__device__ __forceinline__ void stage2(double* smA, const double* srcA, int64_t ldA, int nrA, int ncA, double* smB,
                                       const double* srcB, int64_t ldB, int nrB, int ncB) {
  Stage<TA> a{smA, srcA, ldA, nrA, ncA};
  Stage<TBT> b{smB, srcB, ldB, nrB, ncB};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    a.load(h);
    b.load(h);
    a.store(h);
    b.store(h);
  }
}

// acc (+)= sign * A^T B over the two staged operand tiles, the second k-half's loads in flight
// while the first half is multiplied (one barrier per half)
template <bool NEG, bool TA, bool TBT>
__device__ __forceinline__ void staged_product(double (&acc)[2][4][2], double* smA, const double* srcA, int64_t ldA,
                                               int nrA, int ncA, double* smB, const double* srcB, int64_t ldB, int nrB,
                                               int ncB, int rb, int cb);

// acc (warp's 16 x 32 block: rows rb + 8a + g, cols cb + 8b + 2t{,+1}) += sign * As^T Bs,
// As, Bs in [k][m] layout.
template <bool NEG>
__device__ __forceinline__ void mma64(double (&acc)[2][4][2], const double* As, const double* Bs, int rb, int cb,
                                      int k0 = 0, int k1 = TB) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll 4
  for (int kk = k0; kk < k1; kk += 4) {
    double a[2], b[4];
#pragma unroll
    for (int x = 0; x < 2; ++x) a[x] = NEG ? -As[(kk + t) * TP + rb + 8 * x + g] : As[(kk + t) * TP + rb + 8 * x + g];
#pragma unroll
    for (int y = 0; y < 4; ++y) b[y] = Bs[(kk + t) * TP + cb + 8 * y + g];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) dmma8x8x4(acc[x][y][0], acc[x][y][1], a[x], b[y]);
  }
}

template <bool NEG, bool TA, bool TBT>
__device__ __forceinline__ void staged_product(double (&acc)[2][4][2], double* smA, const double* srcA, int64_t ldA,
                                               int nrA, int ncA, double* smB, const double* srcB, int64_t ldB, int nrB,
                                               int ncB, int rb, int cb) {
  Stage<TA> a{smA, srcA, ldA, nrA, ncA};
  Stage<TBT> b{smB, srcB, ldB, nrB, ncB};
  a.load(0);
  b.load(0);
  a.store(0);
  b.store(0);
  a.load(1);
  b.load(1);
  __syncthreads();
  // TA: the half h = 0 holds k = m-rows 0..31 only for the untransposed layout; a transposed
  // stage fills all k for rows 0..31 of the source, so its product waits for both halves
  if (!TA && !TBT) mma64<NEG>(acc, smA, smB, rb, cb, 0, TB / 2);
  a.store(1);
  b.store(1);
  __syncthreads();
  if (!TA && !TBT) mma64<NEG>(acc, smA, smB, rb, cb, TB / 2, TB);
  else mma64<NEG>(acc, smA, smB, rb, cb);
}

// 16-byte asynchronous copy global -> shared through L2 only (.cg: no L1 line is allocated, so
// a tile another SM rewrote can never be read stale); src-size 0 zero-fills
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit_g() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_g() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
// tile (row-major, ld even, 16-byte aligned) -> smem [k][m] pitch TP, rows < nr, cols < nc (nc even)
__device__ __forceinline__ void tile_async(double* sm, const double* src, int64_t ld, int nr, int nc) {
#pragma unroll
  for (int x = 0; x < TB * TB / 2 / DAG_THREADS; ++x) {
    const int e = threadIdx.x + DAG_THREADS * x;  // chunk: row e / 32, columns 2 (e % 32) + {0, 1}
    const int r = e >> 5, c = (e & 31) * 2;
    const bool ok = r < nr && c < nc;
    cp_async16(sm + r * TP + c, ok ? src + (int64_t)r * ld + c : src, ok);
  }
}

// acc (+)= sign * A^T B with A already in smA and B staged now (second k-half in flight
// during the first half's product)
template <bool NEG>
__device__ __forceinline__ void staged_product_b(double (&acc)[2][4][2], const double* smA, double* smB,
                                                 const double* srcB, int64_t ldB, int nrB, int ncB, int rb, int cb) {
  Stage<false> b{smB, srcB, ldB, nrB, ncB};
  b.load(0);
  b.store(0);
  b.load(1);
  __syncthreads();
  mma64<NEG>(acc, smA, smB, rb, cb, 0, TB / 2);
  b.store(1);
  __syncthreads();
  mma64<NEG>(acc, smA, smB, rb, cb, TB / 2, TB);
}

// acc <-> global 64 x 64 block (row-major, ld), rows < nr, cols < nc
__device__ __forceinline__ void acc_load(double (&acc)[2][4][2], const double* C, int64_t ld, int nr, int nc, int rb,
                                         int cb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if ((ld & 1) == 0 && ((uintptr_t)C & 15) == 0) {  // 16-byte loads of the (2t, 2t+1) pairs
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int r = rb + 8 * x + g, c = cb + 8 * y + 2 * t;
        double2 v = make_double2(0.0, 0.0);
        if (r < nr && c + 1 < nc) v = __ldcg(reinterpret_cast<const double2*>(C + (int64_t)r * ld + c));
        else if (r < nr && c < nc) v.x = __ldcg(C + (int64_t)r * ld + c);
        acc[x][y][0] = v.x;
        acc[x][y][1] = v.y;
      }
    return;
  }
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int r = rb + 8 * x + g, c = cb + 8 * y + 2 * t + z;
        acc[x][y][z] = (r < nr && c < nc) ? __ldcg(C + (int64_t)r * ld + c) : 0.0;
      }
}
__device__ __forceinline__ void acc_store(const double (&acc)[2][4][2], double* C, int64_t ld, int nr, int nc, int rb,
                                          int cb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if ((ld & 1) == 0 && ((uintptr_t)C & 15) == 0) {  // 16-byte stores: full 32-byte sectors per pair of lanes
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int r = rb + 8 * x + g, c = cb + 8 * y + 2 * t;
        if (r < nr && c + 1 < nc)
          __stcg(reinterpret_cast<double2*>(C + (int64_t)r * ld + c), make_double2(acc[x][y][0], acc[x][y][1]));
        else if (r < nr && c < nc)
          __stcg(C + (int64_t)r * ld + c, acc[x][y][0]);
      }
    return;
  }
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int r = rb + 8 * x + g, c = cb + 8 * y + 2 * t + z;
        if (r < nr && c < nc) __stcg(C + (int64_t)r * ld + c, acc[x][y][z]);
      }
}
__device__ __forceinline__ void acc_zero(double (&acc)[2][4][2]) {
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
}

// P(q): Cholesky with deflation of the nb x nb diagonal tile at D (row-major, ld) together
// with Y = R^{-T} (so T_qq = R^+ = Y^T), as the right-looking factorisation of the augmented
// 64 x 128 block [A | I] (the panel solves applied to I are the forward substitution
// R^T Y = I, so the inverse costs no extra sequential steps).  16-wide sub-panels:
//   pivots:    warp 0, the 16 x 16 diagonal block in registers (lane: column lane % 16, rows
//              lane / 16 + 2m), one pivot per step with shuffles; deflation test of DESIGN.md R8
//              on the current Schur diagonal; 1/sqrt by rsqrt (r = d * rsqrt(d));
//   row block: one thread per remaining column of [A | I] (always 64 columns);
//   trailing:  8 x 8 DMMA tiles over the upper part of A and the live part of the right block.
// Pivots >= nb are an identity; Y is stored zero-padded (rows / columns >= nb).
constexpr int ALD = 2 * TB + 4;  // pitch of [A | I] (== 4 mod 16)

// [A | I] <- the diagonal tile at D (upper part; identity padding for pivots >= nb)
__device__ __forceinline__ void potrf_load(double* A, const double* D, int64_t ld, int nb) {
  const int tid = threadIdx.x;
  {
    const int c = tid & (TB - 1), r0 = tid >> 6;
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int r = r0 + 4 * u;
      v[u] = (r < nb && c < nb && c >= r) ? __ldcg(D + (int64_t)r * ld + c) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int r = r0 + 4 * u;
      A[r * ALD + c] = (r < nb && c < nb) ? v[u] : (r == c ? 1.0 : 0.0);
      A[r * ALD + TB + c] = (r == c) ? 1.0 : 0.0;
    }
  }
}

// [A | I] <- a warp-fragment accumulator holding the (updated) diagonal tile
__device__ __forceinline__ void potrf_from_acc(double* A, const double (&acc)[2][4][2], int nb, int rb, int cb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int r = rb + 8 * x + g, c = cb + 8 * y + 2 * t + z;
        A[r * ALD + c] = (r < nb && c < nb) ? (c >= r ? acc[x][y][z] : 0.0) : (r == c ? 1.0 : 0.0);
      }
  for (int e = threadIdx.x; e < TB * TB; e += DAG_THREADS) {
    const int r = e >> 6, c = e & (TB - 1);
    A[r * ALD + TB + c] = (r == c) ? 1.0 : 0.0;
  }
}

__device__ __forceinline__ void potrf_core(double* A, int nb, const double* __restrict__ en, double tau,
                                           int32_t* __restrict__ keep) {
  potrf_core_t<TB, DAG_THREADS>(A, nb, en, tau, keep);
}

// Y = R^{-T} (zero-padded) -> Yq: what the bulk's row-panel products need before fin(q, q)
__device__ __forceinline__ void potrf_store_y(const double* A, int nb, double* __restrict__ Yq) {
  const int tid = threadIdx.x, c = tid & (TB - 1), r0 = tid >> 6;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int r = r0 + 4 * u;
    __stcg(Yq + r * TB + c, (r < nb && c < nb) ? A[r * ALD + TB + c] : 0.0);
  }
}
// R (upper, zero below) -> D: read by no task of the factorisation (only by later kernels), so it
// is stored after fin(q, q) is published and drains behind the chain's next products
__device__ __forceinline__ void potrf_store_r(const double* A, double* D, int64_t ld, int nb) {
  const int tid = threadIdx.x, c = tid & (TB - 1), r0 = tid >> 6;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int r = r0 + 4 * u;
    if (r < nb && c < nb) __stcg(D + (int64_t)r * ld + c, c >= r ? A[r * ALD + c] : 0.0);
  }
}

struct CholDag {
  double* G;
  int64_t s;
  int nt;
  const int4* tasks;
  int ntasks;
  int* fin;  // nt x nt: tile (q,c) of R final
  int* ver;  // nt x nt: updates applied to tile (i,c) by the bulk
  int* ticket;
  int* chain_sm;  // 1 + SM of the chain CTA (0 = not yet known)
  int evict;      // the chain CTA's SM partner leaves (no DMMA contention on the chain)
  double* Tb;     // nt x 64 x 64: Y_qq = R_qq^{-T} (row-major), T_qq = Y_qq^T
  const double* en;
  double tau;
  int32_t* keep;
  long long* trace;  // optional (TSVD_DAG_TRACE): per task {type | smid << 8, claimed, ready, done} (ns)
  int zero_lower;    // also zero the strict lower triangle (else it keeps the input's values)
  int cstage;        // strips stage C by cp.async too (needs DAG_SMEM_CSTAGE: one CTA per SM)
  int pipe;          // strips interleave the next tile's copies and the last tile's stores with the MMAs
};

// generic fragment product: acc += sign * A_op B_op with A_op[m][k] = fa(k, m), B_op[k][n] = fb(k, n)
template <bool NEG, class FA, class FB>
__device__ __forceinline__ void mma_gen(double (&acc)[2][4][2], FA fa, FB fb, int rb, int cb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll 4
  for (int kk = 0; kk < TB; kk += 4) {
    double av[2], bv[4];
#pragma unroll
    for (int x = 0; x < 2; ++x) av[x] = NEG ? -fa(kk + t, rb + 8 * x + g) : fa(kk + t, rb + 8 * x + g);
#pragma unroll
    for (int y = 0; y < 4; ++y) bv[y] = fb(kk + t, cb + 8 * y + g);
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) dmma8x8x4(acc[x][y][0], acc[x][y][1], av[x], bv[y]);
  }
}

// acc -> smem [r][c] (pitch TP)
__device__ __forceinline__ void acc_to_smem(const double (&acc)[2][4][2], double* S, int rb, int cb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) S[(rb + 8 * x + g) * TP + cb + 8 * y + 2 * t + z] = acc[x][y][z];
}

__device__ __forceinline__ void zero_tile(double* L, int64_t ld, int nr) {
  for (int e = threadIdx.x; e < nr * TB; e += DAG_THREADS) __stcg(L + (int64_t)(e >> 6) * ld + (e & (TB - 1)), 0.0);
}

// The diagonal chain, run by the CTA holding ticket 0: for j = 0, 1, ..:
//   P(j) in shared memory -> S(j,j+1) = Y_jj^T... (T_jj^T A(j,j+1), T_jj^T = Y_jj read in place)
//   -> A(j+1,j+1) -= R(j,j+1)^T R(j,j+1) straight into the next factorisation's [A | I].
// The bulk's updates of tile (j+1,j+1) / (j,j+1) by panels < j are awaited through ver.
__device__ void chol_chain(const CholDag& a, double* sm) {
  long long tw = 0, tw2 = 0, tp = 0, ts = 0, tu = 0, t0 = 0;  // trace: waits (S / update) / P / S / update (ns)
  long long wthird[3] = {0, 0, 0};
  const bool tr = a.trace != nullptr && threadIdx.x == 0;
#define CT(acc)                   \
  if (tr) {                       \
    const long long t1 = gtimer(); \
    acc += t1 - t0;               \
    t0 = t1;                      \
  }
  if (tr) t0 = gtimer();
  double* F = sm;
  double* Xs = sm + TB * ALD;
  const int warp = threadIdx.x >> 5, rb = (warp >> 1) * 16, cb = (warp & 1) * 32;
  const int64_t s = a.s;
  const int nt = a.nt;
  int nb = tile_n(s);
  // the next step's deflation references, loaded during the update (their latency under its
  // MMAs) instead of at the start of the factorisation on the chain
  __shared__ double en_pre[TB];
  if (threadIdx.x < TB) en_pre[threadIdx.x] = threadIdx.x < nb ? a.en[threadIdx.x] : 1.0;
  potrf_load(F, a.G, s, nb);
  __syncthreads();
  for (int j = 0; j < nt; ++j) {
    double* Djj = a.G + (int64_t)TB * j * s + (int64_t)TB * j;
    potrf_core(F, nb, en_pre, a.tau, a.keep + (int64_t)TB * j);
    potrf_store_y(F, nb, a.Tb + (int64_t)j * TB * TB);
    publish(a.fin + j * nt + j, 1);
    potrf_store_r(F, Djj, s, nb);
    CT(tp);
    if (j + 1 == nt) break;
    const int nc = tile_n(s - (int64_t)TB * (j + 1));
    // S(j, j+1)
    wait_ge(a.ver + j * nt + j + 1, j);
    {
      const long long before = tw;
      CT(tw);
      if (tr) wthird[min(2, 3 * j / nt)] += tw - before;
    }
    double* Bj = Djj + TB;
    {
      Stage<false> st{Xs, Bj, s, TB, nc};
      st.load(0);
      st.store(0);
      st.load(1);
      st.store(1);
    }
    __syncthreads();
    double acc[2][4][2];
    acc_zero(acc);
    mma_gen<false>(acc, [&](int k, int m) { return F[m * ALD + TB + k]; }, [&](int k, int n) { return Xs[k * TP + n]; },
                   rb, cb);
    __syncthreads();
    acc_store(acc, Bj, s, TB, nc, rb, cb);
    acc_to_smem(acc, Xs, rb, cb);
    if (a.zero_lower) zero_tile(a.G + (int64_t)TB * (j + 1) * s + (int64_t)TB * j, s, nc);
    publish(a.fin + j * nt + j + 1, 1);
    CT(ts);
    // A(j+1, j+1) -= R(j,j+1)^T R(j,j+1), the bulk's updates by panels < j first
    wait_ge(a.ver + (j + 1) * nt + j + 1, j);
    {
      const long long before = tw2;
      CT(tw2);
      if (tr) wthird[min(2, 3 * j / nt)] += tw2 - before;
    }
    double* D1 = Djj + (int64_t)TB * s + TB;
    const double en_next = threadIdx.x < nc ? a.en[(int64_t)TB * (j + 1) + threadIdx.x] : 1.0;
    acc_load(acc, D1, s, nc, nc, rb, cb);
    mma64<true>(acc, Xs, Xs, rb, cb);
    if (threadIdx.x < TB) en_pre[threadIdx.x] = en_next;
    potrf_from_acc(F, acc, nc, rb, cb);
    nb = nc;
    __syncthreads();
    CT(tu);
  }
  if (tr) {
    long long* o = a.trace + 4 * (int64_t)a.ntasks;
    o[0] = tw + tw2;
    a.trace[4 * (int64_t)a.ntasks + 4] = tw2;
    a.trace[4 * (int64_t)a.ntasks + 5] = wthird[0];
    a.trace[4 * (int64_t)a.ntasks + 6] = wthird[1];
    a.trace[4 * (int64_t)a.ntasks + 7] = wthird[2];
    o[1] = tp;
    o[2] = ts;
    o[3] = tu;
  }
#undef CT
}

__global__ void __launch_bounds__(DAG_THREADS, 1) chol_dag_kernel(CholDag a) {
  pdl_begin();
  extern __shared__ double sm_dag[];
  double* As = sm_dag;
  double* Bs = sm_dag + TB * TP;
  __shared__ int tk;
  const int warp = threadIdx.x >> 5, rb = (warp >> 1) * 16, cb = (warp & 1) * 32;
  const int64_t s = a.s;
  if (threadIdx.x == 0) tk = atomicAdd(a.ticket, 1);
  for (;;) {
    __syncthreads();
    const int it = tk;
    if (it >= a.ntasks) return;
    TaskTrace tt{a.trace};
    tt.claimed();
    const int4 task = a.tasks[it];
    const int q = task.y, i = task.z, c = task.w;
    const int nri = tile_n(s - (int64_t)TB * i), nrc = tile_n(s - (int64_t)TB * c);
    // the next ticket is claimed now and used after this task (its latency hidden behind the
    // task) — never by the chain, which would hold a ticket for the whole factorisation
    int nxt = a.ntasks;
    if (threadIdx.x == 0 && task.x != T_CHAIN) {
      const int cs = a.evict ? ld_acquire(a.chain_sm) : 0;
      if (cs != (int)smid() + 1) nxt = atomicAdd(a.ticket, 1);
    }
    if (task.x == T_CHAIN) {
      if (threadIdx.x == 0) st_release(a.chain_sm, (int)smid() + 1);
      tt.ready();
      chol_chain(a, sm_dag);
      if (threadIdx.x == 0) {
        const int cs = a.evict ? ld_acquire(a.chain_sm) : 0;
        nxt = (cs == (int)smid() + 1) ? a.ntasks : atomicAdd(a.ticket, 1);
      }
    } else if (task.x == T_S) {
      wait_all(a.fin + q * a.nt + q, 1, a.ver + q * a.nt + c, q);
      tt.ready();
      double* B = a.G + (int64_t)TB * q * s + (int64_t)TB * c;
      stage2<true, false>(As, a.Tb + (int64_t)q * TB * TB, TB, TB, TB, Bs, B, s, TB, nrc);  // T^T = Y
      __syncthreads();
      double acc[2][4][2];
      acc_zero(acc);
      mma64<false>(acc, As, Bs, rb, cb);
      acc_store(acc, B, s, TB, nrc, rb, cb);
      if (a.zero_lower) zero_tile(a.G + (int64_t)TB * c * s + (int64_t)TB * q, s, nrc);  // mirror tile (c, q) := 0
      publish(a.fin + q * a.nt + c, 1);
    } else if (task.x == T_W) {  // A(i, c..c+w) -= R(q,i)^T R(q, c..c+w), R(q,i) staged once
      const int w = min(STRIP, a.nt - c);
      {  // thread 0: fin(q,i); thread 1 + 2u: fin(q, c+u); thread 2 + 2u: ver(i, c+u) >= q
        const int t = threadIdx.x;
        if (t < 1 + 2 * w) {
          const int u = (t - 1) >> 1;
          const int* p = t == 0 ? a.fin + q * a.nt + i : ((t & 1) ? a.fin + q * a.nt + c + u : a.ver + i * a.nt + c + u);
          const int v = (t == 0 || (t & 1)) ? 1 : q;
          while (ld_acquire(p) < v) __nanosleep(32);
        }
        __syncthreads();
      }
      tt.ready();
      if (a.cstage && a.pipe && (s & 1) == 0 && ((uintptr_t)a.G & 15) == 0) {
        // software-pipelined strip: while tile u is multiplied (16 k-steps), every k-step also
        // issues one of this thread's 16 cp.async for tile u+1 (B and C, double-buffered) and,
        // in the first 8, one 16-byte store of tile u-1's result — the LSU work of the copies and
        // write-backs (~2300 cycles per tile when issued in phases of their own) runs under the
        // DMMA pipe's ~4200 cycles.  One barrier per tile; tile u-1 is published after it.
        double* Bb[2] = {Bs, Bs + TB * TP};
        double* Cb[2] = {Bs + 2 * TB * TP, Bs + 3 * TB * TP};
        const double* Rq = a.G + (int64_t)TB * q * s;
        double* Crow = a.G + (int64_t)TB * i * s;
        const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
        tile_async(As, Rq + (int64_t)TB * i, s, TB, nri);
        tile_async(Bb[0], Rq + (int64_t)TB * c, s, TB, tile_n(s - (int64_t)TB * c));
        tile_async(Cb[0], Crow + (int64_t)TB * c, s, nri, tile_n(s - (int64_t)TB * c));
        cp_async_commit_g();
        // this thread's copy chunks: row e / 32, columns 2 (e % 32) + {0, 1}, e = tid + 256 x
        int soff[8];
        int64_t goff[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const int e = threadIdx.x + DAG_THREADS * x, r = e >> 5, c2 = (e & 31) * 2;
          soff[x] = r * TP + c2;
          goff[x] = (int64_t)r * s + c2;
        }
        cp_async_wait_g<0>();
        __syncthreads();
        double acc[2][4][2], prv[2][4][2];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) {
            const double2 v = *reinterpret_cast<const double2*>(Cb[0] + (rb + 8 * x + g) * TP + cb + 8 * y + 2 * t);
            acc[x][y][0] = v.x;
            acc[x][y][1] = v.y;
            prv[x][y][0] = prv[x][y][1] = 0.0;
          }
        for (int u = 0; u < w; ++u) {
          const int cc = c + u, bu = u & 1;
          const bool nxt = u + 1 < w;
          const int n1 = nxt ? tile_n(s - (int64_t)TB * (cc + 1)) : 0;
          const double* nB = Rq + (int64_t)TB * (cc + 1);
          const double* nC = Crow + (int64_t)TB * (cc + 1);
          double* pC = Crow + (int64_t)TB * (cc - 1);  // tile u-1 (u > 0)
          const int npc = u > 0 ? tile_n(s - (int64_t)TB * (cc - 1)) : 0;
          const double* Bsm = Bb[bu];
#pragma unroll
          for (int st = 0; st < TB / 4; ++st) {
            const int kk = 4 * st;
            if (nxt) {  // copy chunk st of tile u+1: B for st < 8, C after
              const int x = st & 7, e = threadIdx.x + DAG_THREADS * x, r = e >> 5, c2 = (e & 31) * 2;
              if (st < 8) {
                const bool ok = c2 < n1;
                cp_async16(Bb[bu ^ 1] + soff[x], ok ? nB + goff[x] : nB, ok);
              } else {
                const bool ok = r < nri && c2 < n1;
                cp_async16(Cb[bu ^ 1] + soff[x], ok ? nC + goff[x] : nC, ok);
              }
            }
            if (u > 0 && st < 8) {  // store chunk st of tile u-1's result
              const int x = st >> 2, y = st & 3, r = rb + 8 * x + g, cl = cb + 8 * y + 2 * t;
              if (r < nri && cl + 1 < npc)
                __stcg(reinterpret_cast<double2*>(pC + (int64_t)r * s + cl), make_double2(prv[x][y][0], prv[x][y][1]));
              else if (r < nri && cl < npc)
                __stcg(pC + (int64_t)r * s + cl, prv[x][y][0]);
            }
            double fa[2], fb[4];
#pragma unroll
            for (int x = 0; x < 2; ++x) fa[x] = -As[(kk + t) * TP + rb + 8 * x + g];
#pragma unroll
            for (int y = 0; y < 4; ++y) fb[y] = Bsm[(kk + t) * TP + cb + 8 * y + g];
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
              for (int y = 0; y < 4; ++y) dmma8x8x4(acc[x][y][0], acc[x][y][1], fa[x], fb[y]);
          }
          if (nxt) cp_async_commit_g();
          cp_async_wait_g<0>();
          __syncthreads();  // tile u+1 landed; every warp is past tile u's reads and u-1's stores
          if (u > 0 && threadIdx.x == 0) st_release(a.ver + i * a.nt + cc - 1, q + 1);
#pragma unroll
          for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) {
              prv[x][y][0] = acc[x][y][0];
              prv[x][y][1] = acc[x][y][1];
              if (nxt) {
                const double2 v =
                    *reinterpret_cast<const double2*>(Cb[bu ^ 1] + (rb + 8 * x + g) * TP + cb + 8 * y + 2 * t);
                acc[x][y][0] = v.x;
                acc[x][y][1] = v.y;
              }
            }
        }
        const int cl = c + w - 1;
        acc_store(prv, Crow + (int64_t)TB * cl, s, nri, tile_n(s - (int64_t)TB * cl), rb, cb);
        __syncthreads();
        if (threadIdx.x == 0) st_release(a.ver + i * a.nt + cl, q + 1);
      } else if (a.cstage && (s & 1) == 0 && ((uintptr_t)a.G & 15) == 0) {
        // everything by cp.async: tile u+1's operand and C stream in while tile u is multiplied
        double* Bb[2] = {Bs, Bs + TB * TP};
        double* Cs = Bs + 2 * TB * TP;
        const double* Rq = a.G + (int64_t)TB * q * s;
        const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
        tile_async(As, Rq + (int64_t)TB * i, s, TB, nri);
        tile_async(Bb[0], Rq + (int64_t)TB * c, s, TB, tile_n(s - (int64_t)TB * c));
        tile_async(Cs, a.G + (int64_t)TB * i * s + (int64_t)TB * c, s, nri, tile_n(s - (int64_t)TB * c));
        cp_async_commit_g();
        long long ph[5] = {0, 0, 0, 0, 0}, pt = a.trace ? clock64() : 0;
#define PH(k)                        \
  if (a.trace) {                     \
    const long long t1_ = clock64(); \
    ph[k] += t1_ - pt;               \
    pt = t1_;                        \
  }
        for (int u = 0; u < w; ++u) {
          const int cc = c + u, ncc = tile_n(s - (int64_t)TB * cc);
          cp_async_wait_g<0>();
          __syncthreads();
          PH(0);
          double acc[2][4][2];
#pragma unroll
          for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) {  // 16-byte reads: conflict-free (8-byte ones were 4-way)
              const double2 v = *reinterpret_cast<const double2*>(Cs + (rb + 8 * x + g) * TP + cb + 8 * y + 2 * t);
              acc[x][y][0] = v.x;
              acc[x][y][1] = v.y;
            }
          __syncthreads();  // Cs consumed
          if (u + 1 < w) {
            const int n1 = tile_n(s - (int64_t)TB * (cc + 1));
            tile_async(Bb[(u + 1) & 1], Rq + (int64_t)TB * (cc + 1), s, TB, n1);
            tile_async(Cs, a.G + (int64_t)TB * i * s + (int64_t)TB * (cc + 1), s, nri, n1);
            cp_async_commit_g();
          }
          PH(1);
          mma64<true>(acc, As, Bb[u & 1], rb, cb);
          PH(2);
          // tile u-1 is published one tile late: its stores were ordered before this
          // iteration's first barrier and have long completed, so the release fence costs
          // nothing (published at once, it stalled warp 0 ~1 us per tile on the store acks,
          // and the CTA with it at the next barrier)
          if (u > 0 && threadIdx.x == 0) st_release(a.ver + i * a.nt + cc - 1, q + 1);
          acc_store(acc, a.G + (int64_t)TB * i * s + (int64_t)TB * cc, s, nri, ncc, rb, cb);
          PH(3);
        }
        __syncthreads();
        if (threadIdx.x == 0) st_release(a.ver + i * a.nt + c + w - 1, q + 1);
        PH(4);
        if (a.trace && threadIdx.x == 0)
          for (int k = 0; k < 5; ++k) atomicAdd((unsigned long long*)a.trace + 4 * (int64_t)a.ntasks + 8 + k, ph[k]);
#undef PH
      } else if ((s & 1) == 0 && ((uintptr_t)a.G & 15) == 0) {
        // R(q,i) once and R(q, c+u) double-buffered by cp.async: tile u+1's operand streams in
        // while tile u is multiplied; C(i, c+u) through registers, loaded after the previous
        // tile's store; each tile published as soon as its stores are issued
        double* Bb[2] = {Bs, Bs + TB * TP};
        const double* Rq = a.G + (int64_t)TB * q * s;
        tile_async(As, Rq + (int64_t)TB * i, s, TB, nri);
        tile_async(Bb[0], Rq + (int64_t)TB * c, s, TB, tile_n(s - (int64_t)TB * c));
        cp_async_commit_g();
        double acc[2][4][2];
        acc_load(acc, a.G + (int64_t)TB * i * s + (int64_t)TB * c, s, nri, tile_n(s - (int64_t)TB * c), rb, cb);
        for (int u = 0; u < w; ++u) {
          const int cc = c + u, ncc = tile_n(s - (int64_t)TB * cc);
          if (u + 1 < w) {
            tile_async(Bb[(u + 1) & 1], Rq + (int64_t)TB * (cc + 1), s, TB, tile_n(s - (int64_t)TB * (cc + 1)));
            cp_async_commit_g();
            cp_async_wait_g<1>();
          } else {
            cp_async_wait_g<0>();
          }
          __syncthreads();
          mma64<true>(acc, As, Bb[u & 1], rb, cb);
          double* C = a.G + (int64_t)TB * i * s + (int64_t)TB * cc;
          acc_store(acc, C, s, nri, ncc, rb, cb);
          __syncthreads();  // stores issued; B[u & 1] free for tile u + 2
          if (threadIdx.x == 0) st_release(a.ver + i * a.nt + cc, q + 1);
          if (u + 1 < w)
            acc_load(acc, C + TB, s, nri, tile_n(s - (int64_t)TB * (cc + 1)), rb, cb);
        }
      } else
      for (int u = 0; u < w; ++u) {
        const int cc = c + u, ncc = tile_n(s - (int64_t)TB * cc);
        double* C = a.G + (int64_t)TB * i * s + (int64_t)TB * cc;
        double acc[2][4][2];
        acc_load(acc, C, s, nri, ncc, rb, cb);
        if (u == 0)
          staged_product<true, false, false>(acc, As, a.G + (int64_t)TB * q * s + (int64_t)TB * i, s, TB, nri, Bs,
                                             a.G + (int64_t)TB * q * s + (int64_t)TB * cc, s, TB, ncc, rb, cb);
        else
          staged_product_b<true>(acc, As, Bs, a.G + (int64_t)TB * q * s + (int64_t)TB * cc, s, TB, ncc, rb, cb);
        acc_store(acc, C, s, nri, ncc, rb, cb);
        publish(a.ver + i * a.nt + cc, q + 1);  // (its barrier also frees Bs for the next tile)
      }
    } else {  // T_U: A(i,c) -= R(q,i)^T R(q,c)
      wait_all(a.fin + q * a.nt + i, 1, a.fin + q * a.nt + c, 1, a.ver + i * a.nt + c, q);
      tt.ready();
      double* C = a.G + (int64_t)TB * i * s + (int64_t)TB * c;
      double acc[2][4][2];
      acc_load(acc, C, s, nri, nrc, rb, cb);
      staged_product<true, false, false>(acc, As, a.G + (int64_t)TB * q * s + (int64_t)TB * i, s, TB, nri, Bs,
                                         a.G + (int64_t)TB * q * s + (int64_t)TB * c, s, TB, nrc, rb, cb);
      acc_store(acc, C, s, nri, nrc, rb, cb);
      publish(a.ver + i * a.nt + c, q + 1);
    }
    tt.done(it, task.x);
    __syncthreads();  // smem reuse; every thread has read tk
    if (threadIdx.x == 0) tk = nxt;
  }
}

struct TrsmDag {
  const double* R;
  int64_t s;
  int nt, nkb, k;
  const double* Tb;
  double* X;
  const int4* tasks;
  int ntasks;
  int* fin;  // nt x nkb: X tile final
  int* ver;  // nt x nkb: bulk updates applied
  int* ticket;
  int* chain_sm;
  int evict;
  long long* trace;
  int pre;  // R holds W(i,j) = T_ii R(i,j) and X holds Y_i = T_ii X_i (trsm_prescale_kernel)
};

// The back-substitution chain (ticket 0): for j = nt-1 .. 0 and every column block b:
//   X_j = T_jj (X_j - R(j,j+1) X_{j+1})   (the bulk's updates from blocks > j+1 awaited via ver)
// fast path (one column block, even s): the operands of step j - 1 (R(j-1, j) and T_{j-1},
// neither of which depends on the chain) stream in by cp.async while step j runs; only X_j waits
__device__ void trsm_chain_pipelined(const TrsmDag& a, double* sm) {
  double* Rb[2] = {sm, sm + TB * RPT};
  double* Tq[2] = {sm + 2 * TB * RPT, sm + 2 * TB * RPT + TB * TP};
  double* Bc = sm + 2 * TB * RPT + 2 * TB * TP;
  const int warp = threadIdx.x >> 5, rb = (warp >> 1) * 16, cb = (warp & 1) * 32;
  const int64_t s = a.s;
  const int nt = a.nt, k = a.k;
  auto prefetch = [&](int j, int buf) {  // T_j and, below the last block, R(j, j+1)
#pragma unroll
    for (int x = 0; x < TB * TB / 2 / DAG_THREADS; ++x) {
      const int e = threadIdx.x + DAG_THREADS * x, r = e >> 5, c = (e & 31) * 2;
      cp_async16(Tq[buf] + r * TP + c, a.Tb + (int64_t)j * TB * TB + r * TB + c, true);
      if (j + 1 < nt) {
        const int nr1 = tile_n(s - (int64_t)TB * (j + 1));
        const bool ok = c < nr1;
        const double* src = a.R + (int64_t)(TB * j + r) * s + (int64_t)TB * (j + 1) + c;
        cp_async16(Rb[buf] + r * RPT + c, ok ? src : a.R, ok);
      }
    }
    cp_async_commit_g();
  };
  prefetch(nt - 1, 0);
  for (int j = nt - 1; j >= 0; --j) {
    const int p = (nt - 1 - j) & 1;
    if (j >= 1) prefetch(j - 1, p ^ 1);
    const int nrj = tile_n(s - (int64_t)TB * j);
    double* Xj = a.X + (int64_t)TB * j * k;
    double acc[2][4][2];
    wait_ge(a.ver + j, nt - 2 - j < 0 ? 0 : nt - 2 - j);
    if (a.pre) {
      // prescaled: X_j = Y_j - W(j,j+1) X_{j+1}, one product on the chain (the bulk updates
      // Y_i -= W(i,j) X_j with the same task code); X_{nt-1} = Y_{nt-1} is final as it stands
      acc_load(acc, Xj, k, nrj, k, rb, cb);
      if (j >= 1) cp_async_wait_g<1>();
      else cp_async_wait_g<0>();
      __syncthreads();
      if (j + 1 < nt) {
        const double* R = Rb[p];
        mma_gen<true>(acc, [&](int kk, int m) { return R[m * RPT + kk]; }, [&](int kk, int n) { return Bc[kk * TP + n]; },
                      rb, cb);
        __syncthreads();
        acc_store(acc, Xj, k, nrj, k, rb, cb);
      }
      acc_to_smem(acc, Bc, rb, cb);
      publish(a.fin + j, 1);
      continue;
    }
    if (j + 1 < nt) {
      acc_load(acc, Xj, k, nrj, k, rb, cb);
      if (j >= 1) cp_async_wait_g<1>();
      else cp_async_wait_g<0>();
      __syncthreads();
      const double* R = Rb[p];
      mma_gen<true>(acc, [&](int kk, int m) { return R[m * RPT + kk]; }, [&](int kk, int n) { return Bc[kk * TP + n]; },
                    rb, cb);
      __syncthreads();
      acc_to_smem(acc, Bc, rb, cb);
    } else {
      Stage<false> st{Bc, Xj, k, nrj, k};
      st.load(0);
      st.store(0);
      st.load(1);
      st.store(1);
      if (j >= 1) cp_async_wait_g<1>();
      else cp_async_wait_g<0>();
    }
    __syncthreads();
    acc_zero(acc);
    mma64<false>(acc, Tq[p], Bc, rb, cb);  // X_j = T_jj (X_j - R(j,j+1) X_{j+1})
    __syncthreads();
    acc_store(acc, Xj, k, nrj, k, rb, cb);
    acc_to_smem(acc, Bc, rb, cb);
    publish(a.fin + j, 1);
  }
}

__device__ void trsm_chain(const TrsmDag& a, double* sm) {
  if (a.nkb == 1 && (a.s & 1) == 0 && ((uintptr_t)a.R & 15) == 0 && ((uintptr_t)a.Tb & 15) == 0) {
    trsm_chain_pipelined(a, sm);
    return;
  }
  double* As = sm;
  double* Bc = sm + TB * TP;
  const int warp = threadIdx.x >> 5, rb = (warp >> 1) * 16, cb = (warp & 1) * 32;
  const int64_t s = a.s;
  const int nt = a.nt, k = a.k;
  for (int j = nt - 1; j >= 0; --j) {
    const int nrj = tile_n(s - (int64_t)TB * j);
    for (int b = 0; b < a.nkb; ++b) {
      const int ncb = min(TB, k - TB * b);
      double* Xj = a.X + (int64_t)TB * j * k + (int64_t)TB * b;
      double acc[2][4][2];
      wait_ge(a.ver + j * a.nkb + b, nt - 2 - j < 0 ? 0 : nt - 2 - j);
      if (j + 1 < nt) {
        const int nr1 = tile_n(s - (int64_t)TB * (j + 1));
        if (a.nkb > 1) {  // X_{j+1, b} (final) from global; with one block it is still in Bc
          Stage<false> st{Bc, a.X + (int64_t)TB * (j + 1) * k + (int64_t)TB * b, k, nr1, ncb};
          st.load(0);
          st.store(0);
          st.load(1);
          st.store(1);
        }
        {
          Stage<true> st{As, a.R + (int64_t)TB * j * s + (int64_t)TB * (j + 1), s, TB, nr1};
          st.load(0);
          st.store(0);
          st.load(1);
          st.store(1);
        }
        acc_load(acc, Xj, k, nrj, ncb, rb, cb);
        __syncthreads();
        mma64<true>(acc, As, Bc, rb, cb);
        __syncthreads();
        acc_to_smem(acc, Bc, rb, cb);
      } else {
        Stage<false> st{Bc, Xj, k, nrj, ncb};
        st.load(0);
        st.store(0);
        st.load(1);
        st.store(1);
      }
      {
        Stage<false> st{As, a.Tb + (int64_t)j * TB * TB, TB, TB, TB};  // T = Y^T
        st.load(0);
        st.store(0);
        st.load(1);
        st.store(1);
      }
      __syncthreads();
      acc_zero(acc);
      mma64<false>(acc, As, Bc, rb, cb);
      __syncthreads();
      acc_store(acc, Xj, k, nrj, ncb, rb, cb);
      acc_to_smem(acc, Bc, rb, cb);
      publish(a.fin + j * a.nkb + b, 1);
    }
  }
}

__global__ void __launch_bounds__(DAG_THREADS, 1) trsm_dag_kernel(TrsmDag a) {
  pdl_begin();
  extern __shared__ double sm_dag[];
  double* As = sm_dag;
  double* Bs = sm_dag + TB * TP;
  __shared__ int tk;
  const int warp = threadIdx.x >> 5, rb = (warp >> 1) * 16, cb = (warp & 1) * 32;
  const int64_t s = a.s;
  if (threadIdx.x == 0) tk = atomicAdd(a.ticket, 1);
  for (;;) {
    __syncthreads();
    const int it = tk;
    if (it >= a.ntasks) return;
    TaskTrace tt{a.trace};
    tt.claimed();
    const int4 task = a.tasks[it];
    const int j = task.y, i = task.z, b = task.w;
    int nxt = a.ntasks;
    if (threadIdx.x == 0 && task.x != T_CHAIN) {
      const int cs = a.evict ? ld_acquire(a.chain_sm) : 0;
      if (cs != (int)smid() + 1) nxt = atomicAdd(a.ticket, 1);
    }
    if (task.x == T_CHAIN) {
      if (threadIdx.x == 0) st_release(a.chain_sm, (int)smid() + 1);
      tt.ready();
      trsm_chain(a, sm_dag);
      if (threadIdx.x == 0) {
        const int cs = a.evict ? ld_acquire(a.chain_sm) : 0;
        nxt = (cs == (int)smid() + 1) ? a.ntasks : atomicAdd(a.ticket, 1);
      }
    } else {  // T_V: X_i -= R(i,j) X_j, j > i + 1
      const int nri = tile_n(s - (int64_t)TB * i), nrj = tile_n(s - (int64_t)TB * j);
      const int ncb = min(TB, a.k - TB * b);
      double* Xi = a.X + (int64_t)TB * i * a.k + (int64_t)TB * b;
      double acc[2][4][2];
      wait_all(a.fin + j * a.nkb + b, 1, a.ver + i * a.nkb + b, a.nt - 1 - j);
      tt.ready();
      stage2<true, false>(As, a.R + (int64_t)TB * i * s + (int64_t)TB * j, s, TB, nrj, Bs,
                          a.X + (int64_t)TB * j * a.k + (int64_t)TB * b, a.k, nrj, ncb);
      acc_load(acc, Xi, a.k, nri, ncb, rb, cb);
      __syncthreads();
      mma64<true>(acc, As, Bs, rb, cb);
      acc_store(acc, Xi, a.k, nri, ncb, rb, cb);
      publish(a.ver + i * a.nkb + b, a.nt - j);
    }
    tt.done(it, task.x);
    __syncthreads();
    if (threadIdx.x == 0) tk = nxt;
  }
}

// ---- task orders.  Ticket 0 is the chain; the bulk follows with look-ahead:
// Cholesky iteration j: (a) S(j, c >= j+2); (b) U(j-1; j+1, c >= j+2); (c) U(j; j+1, c >= j+2);
//   (d) U(j-1; j+2, c >= j+2); (e) U(j; j+2, j+2); (f) U(j-1; i >= j+3, c >= i).
// (U(j; j+1, j+1) is fused into the chain; (e) is the update the chain waits for one step
// later, listed before the bulk (f) so that it is claimed early.  (f) runs as strips T_W of
// STRIP tiles of one tile row.)
// Back substitution iteration j (descending): V(j+1; j-1); V(j+1; i <= j-2).
// Every wait of a bulk task is on the chain or on an earlier ticket, and the chain's waits at
// step j are on tasks of iterations <= j, which only wait on chain output it already published.
std::vector<int4> chol_tasks(int nt) {
  std::vector<int4> v;
  v.push_back(make_int4(T_CHAIN, 0, 0, 0));
  auto U = [&](int q, int i, int c0) {
    for (int c = c0; c < nt; ++c) v.push_back(make_int4(T_U, q, i, c));
  };
  for (int j = 0; j < nt; ++j) {
    for (int c = j + 2; c < nt; ++c) v.push_back(make_int4(T_S, j, j, c));  // (a)
    if (j >= 1 && j + 1 < nt) U(j - 1, j + 1, j + 2);                       // (b)
    if (j + 1 < nt) U(j, j + 1, j + 2);                                     // (c)
    if (j >= 1 && j + 2 < nt) U(j - 1, j + 2, j + 2);                       // (d)
    if (j + 2 < nt) v.push_back(make_int4(T_U, j, j + 2, j + 2));          // (e) the chain's next-but-one diagonal
    if (j >= 1)
      for (int i = j + 3; i < nt; ++i)                                      // (f), in strips
        for (int c = i; c < nt; c += STRIP) v.push_back(make_int4(T_W, j - 1, i, c));
  }
  return v;
}

std::vector<int4> trsm_tasks(int nt, int nkb) {
  std::vector<int4> v;
  v.push_back(make_int4(T_CHAIN, 0, 0, 0));
  for (int j = nt - 1; j >= 0; --j) {
    if (j >= 1 && j + 1 < nt)
      for (int b = 0; b < nkb; ++b) v.push_back(make_int4(T_V, j + 1, j - 1, b));
    if (j + 1 < nt)
      for (int i = j - 2; i >= 0; --i)
        for (int b = 0; b < nkb; ++b) v.push_back(make_int4(T_V, j + 1, i, b));
  }
  return v;
}

// The same orders generated on the device into stream-ordered scratch (no host allocation or
// synchronisation per shape): one CTA per iteration j, its offset from the closed-form sizes.
__host__ __device__ inline int64_t tri(int64_t n) { return n > 0 ? n * (n + 1) / 2 : 0; }
__host__ __device__ inline int64_t chol_iter_size(int nt, int j) {
  const int64_t m = nt - 1 - j, m1 = m > 1 ? m - 1 : 0;
  int64_t n = m1 + m1;                 // (a), (c)
  if (j >= 1) n += m1 + m1;            // (b), (d)
  n += m >= 2 ? 1 : 0;                 // (e)
  if (j >= 1)                          // (f): rows with u = nt - i = 1 .. m - 2 tiles, in strips
    for (int64_t u = 1; u <= m - 2; ++u) n += (u + STRIP - 1) / STRIP;
  return n;
}
__host__ __device__ inline int64_t trsm_iter_size(int nt, int nkb, int j) {
  int64_t n = (j >= 1 && j + 1 < nt) ? 1 : 0;
  if (j + 1 < nt && j >= 2) n += j - 1;
  return n * nkb;
}
int64_t chol_ntasks(int nt) {
  int64_t n = 1;
  for (int j = 0; j < nt; ++j) n += chol_iter_size(nt, j);
  return n;
}
int64_t trsm_ntasks(int nt, int nkb) {
  int64_t n = 1;
  for (int j = 0; j < nt; ++j) n += trsm_iter_size(nt, nkb, j);
  return n;
}

__global__ void gen_chol_tasks(int4* out, int nt) {
  pdl_begin();
  const int j = blockIdx.x;
  __shared__ int64_t off_s;
  if (threadIdx.x == 0) {
    int64_t o = 1;
    for (int q = 0; q < j; ++q) o += chol_iter_size(nt, q);
    off_s = o;
    if (j == 0) out[0] = make_int4(T_CHAIN, 0, 0, 0);
  }
  __syncthreads();
  int4* o = out + off_s;
  const int64_t n = chol_iter_size(nt, j), m = nt - 1 - j, m1 = m > 1 ? m - 1 : 0;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    int64_t x = e;
    int4 t;
    if (x < m1) {
      t = make_int4(T_S, j, j, j + 2 + (int)x);  // (a)
    } else if ((x -= m1), j >= 1 && x < m1) {
      t = make_int4(T_U, j - 1, j + 1, j + 2 + (int)x);  // (b)
    } else {
      if (j >= 1) x -= m1;
      if (x < m1) {
        t = make_int4(T_U, j, j + 1, j + 2 + (int)x);  // (c)
      } else if ((x -= m1), j >= 1 && x < m1) {
        t = make_int4(T_U, j - 1, j + 2, j + 2 + (int)x);  // (d)
      } else {
        if (j >= 1) x -= m1;
        if (m >= 2 && x == 0) {
          t = make_int4(T_U, j, j + 2, j + 2);  // (e)
        } else {
          if (m >= 2) x -= 1;
          int i = j + 3;  // (f): rows i = j+3.., ceil((nt - i) / STRIP) strips each
          while (x >= (nt - i + STRIP - 1) / STRIP) x -= (nt - i++ + STRIP - 1) / STRIP;
          t = make_int4(T_W, j - 1, i, i + (int)x * STRIP);
        }
      }
    }
    o[e] = t;
  }
}

__global__ void gen_trsm_tasks(int4* out, int nt, int nkb) {
  pdl_begin();
  const int j = nt - 1 - (int)blockIdx.x;  // iterations run j = nt-1 .. 0
  __shared__ int64_t off_s;
  if (threadIdx.x == 0) {
    int64_t o = 1;
    for (int q = nt - 1; q > j; --q) o += trsm_iter_size(nt, nkb, q);
    off_s = o;
    if (j == nt - 1) out[0] = make_int4(T_CHAIN, 0, 0, 0);
  }
  __syncthreads();
  int4* o = out + off_s;
  const int64_t n = trsm_iter_size(nt, nkb, j) / nkb;
  const int first = (j >= 1 && j + 1 < nt) ? 1 : 0;
  for (int64_t e = threadIdx.x; e < n * nkb; e += blockDim.x) {
    const int64_t x = e / nkb;
    const int b = (int)(e % nkb);
    o[e] = (first && x == 0) ? make_int4(T_V, j + 1, j - 1, b) : make_int4(T_V, j + 1, j - 2 - (int)(x - first), b);
  }
}

// TSVD_DAG_CHECK=1: compare the device-generated order with the host builders (diagnostics)
void check_tasks(const int4* d, const std::vector<int4>& ref, const char* what) {
  std::vector<int4> h(ref.size());
  cudaDeviceSynchronize();
  cudaMemcpy(h.data(), d, h.size() * sizeof(int4), cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (size_t i = 0; i < h.size(); ++i)
    bad += h[i].x != ref[i].x || h[i].y != ref[i].y || h[i].z != ref[i].z || h[i].w != ref[i].w;
  fprintf(stderr, "[dag %s] task order check: %zu tasks, %zu mismatches\n", what, h.size(), bad);
}
bool check_on() {
  static int on = -1;
  if (on < 0) on = getenv("TSVD_DAG_CHECK") != nullptr;
  return on == 1;
}

int dag_grid() {
  static int n = 0;
  if (!n) {
    int dev = 0, sms = 148, occ = 2;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(chol_dag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DAG_SMEM);
    cudaFuncSetAttribute(trsm_dag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRSM_SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chol_dag_kernel, DAG_THREADS, DAG_SMEM);
    n = sms * std::max(1, std::min(occ, 2));
  }
  return n;
}
int pipe_on() {  // TSVD_DAG_PIPE=0: strips issue copies and stores in phases of their own
  static const int v = !(getenv("TSVD_DAG_PIPE") && atoi(getenv("TSVD_DAG_PIPE")) == 0);
  return v;
}
int cstage_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TSVD_DAG_CSTAGE");  // default on (measured faster at s = 1000..8000)
    v = !(e && atoi(e) == 0);
  }
  return v;
}
int cstage_grid() {
  static int n = 0;
  if (!n) {
    dag_grid();
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(chol_dag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DAG_SMEM_CSTAGE);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chol_dag_kernel, DAG_THREADS, DAG_SMEM_CSTAGE);
    n = sms * std::max(1, occ);
  }
  return n;
}
int trsm_grid() {
  static int n = 0;
  if (!n) {
    dag_grid();
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, trsm_dag_kernel, DAG_THREADS, TRSM_SMEM);
    n = sms * std::max(1, occ);
  }
  return n;
}
}  // namespace

// TSVD_DAG_TRACE=1: per-task device timestamps, summarised on stderr after each DAG launch
// (synchronises; diagnostics only)
long long* trace_alloc(int ntasks) {
  static int on = -1;
  if (on < 0) on = getenv("TSVD_DAG_TRACE") != nullptr;
  if (!on) return nullptr;
  long long* p = nullptr;
  if (cudaMalloc(&p, (size_t)(ntasks + 4) * 4 * sizeof(long long))) return nullptr;
  cudaMemset(p, 0, (size_t)(ntasks + 4) * 4 * sizeof(long long));
  return p;
}
void trace_report(const char* what, long long* d, int ntasks, int nt, cudaStream_t st) {
  if (!d) return;
  std::vector<long long> h((size_t)(ntasks + 4) * 4);
  cudaStreamSynchronize(st);
  cudaMemcpy(h.data(), d, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  long long t0 = h[1], t1 = h[3];
  double wait[5] = {0}, exec[5] = {0}, emax[5] = {0};
  std::vector<long long> pdone;
  int cnt[5] = {0};
  for (int i = 0; i < ntasks; ++i) {
    const long long* r = &h[4 * (size_t)i];
    const int ty = (int)(r[0] & 0xff);
    t0 = std::min(t0, r[1]);
    t1 = std::max(t1, r[3]);
    if (ty < 0 || ty > 4) continue;
    if (ty == T_CHAIN) pdone.push_back(r[3] - r[2]);
    cnt[ty]++;
    wait[ty] += r[2] - r[1];
    exec[ty] += r[3] - r[2];
    emax[ty] = std::max(emax[ty], (double)(r[3] - r[2]));
  }
  fprintf(stderr, "[dag %s] nt %d tasks %d span %.1f us\n", what, nt, ntasks, (t1 - t0) / 1e3);
  const char* nm[5] = {"chain", "S", "U", "Wstrip", "V"};
  for (int ty = 0; ty < 5; ++ty)
    if (cnt[ty])
      fprintf(stderr, "  %s x%-7d wait %8.2f us  exec %7.2f us (max %7.2f)\n", nm[ty], cnt[ty], wait[ty] / cnt[ty] / 1e3,
              exec[ty] / cnt[ty] / 1e3, emax[ty] / 1e3);
  if (!pdone.empty()) fprintf(stderr, "  chain: %.2f us per block step\n", pdone[0] / 1e3 / nt);
  const long long* c = &h[4 * (size_t)ntasks];
  if (c[0] + c[1] + c[2] + c[3] > 0)
    fprintf(stderr, "  chain per step: wait %.2f (before the update %.2f)  P %.2f  S %.2f  update %.2f us\n",
            c[0] / 1e3 / nt, c[4] / 1e3 / nt, c[1] / 1e3 / nt, c[2] / 1e3 / nt, c[3] / 1e3 / nt);
  if (c[0] > 0)
    fprintf(stderr, "  chain waits by thirds of the steps: %.1f / %.1f / %.1f us\n", c[5] / 1e3, c[6] / 1e3, c[7] / 1e3);
  if (cnt[T_W] && c[8] + c[9] + c[10] + c[11] > 0)
    fprintf(stderr, "  strip phases per strip (cycles): operand wait %.0f  C regs %.0f  mma %.0f  store %.0f  tail %.0f\n",
            (double)c[8] / cnt[T_W], (double)c[9] / cnt[T_W], (double)c[10] / cnt[T_W], (double)c[11] / cnt[T_W],
            (double)c[12] / cnt[T_W]);
}

// ---- C-ABI: the order (host) and the device generator's agreement with it
extern "C" int64_t tsvd_dag_order(int32_t kind, int32_t nt, int32_t nkb, int32_t* out, int64_t cap) {
  if (nt <= 0 || nkb <= 0 || (kind != 0 && kind != 1)) return -1;
  const std::vector<int4> v = kind == 0 ? chol_tasks(nt) : trsm_tasks(nt, nkb);
  if (out)
    for (size_t i = 0; i < v.size() && (int64_t)i < cap; ++i) {
      out[4 * i] = v[i].x;
      out[4 * i + 1] = v[i].y;
      out[4 * i + 2] = v[i].z;
      out[4 * i + 3] = v[i].w;
    }
  return (int64_t)v.size();
}

extern "C" int64_t tsvd_dag_check(int32_t kind, int32_t nt, int32_t nkb) {
  if (nt <= 0 || nkb <= 0 || (kind != 0 && kind != 1)) return -1;
  const std::vector<int4> ref = kind == 0 ? chol_tasks(nt) : trsm_tasks(nt, nkb);
  const int64_t n = kind == 0 ? chol_ntasks(nt) : trsm_ntasks(nt, nkb);
  if (n != (int64_t)ref.size()) return n > (int64_t)ref.size() ? n : (int64_t)ref.size();
  int4* d = nullptr;
  if (cudaMalloc(&d, n * sizeof(int4))) return -1;
  if (kind == 0) gen_chol_tasks<<<nt, 256>>>(d, nt);
  else gen_trsm_tasks<<<nt, 256>>>(d, nt, nkb);
  std::vector<int4> h(n);
  const cudaError_t e = cudaMemcpy(h.data(), d, n * sizeof(int4), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e) return -1;
  int64_t bad = 0;
  for (int64_t i = 0; i < n; ++i)
    bad += h[i].x != ref[i].x || h[i].y != ref[i].y || h[i].z != ref[i].z || h[i].w != ref[i].w;
  return bad;
}

// TSVD_DAG_EVICT=0 keeps a bulk CTA on the chain's SM
int evict_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TSVD_DAG_EVICT");
    v = !(e && std::string(e) == "0");
  }
  return v;
}

// TSVD_CHOL=panel selects the launch-per-panel path of dense.cu (A/B measurements)
bool dag_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TSVD_CHOL");
    v = !(e && std::string(e) == "panel");
  }
  return v == 1;
}

cudaError_t chol_dag(cudaStream_t st, double* G, int64_t s, const double* enorm2, double tau, int32_t* keep,
                     double* Tb, bool zero_lower) {
  if (s <= 0) return cudaSuccess;
  const int nt = (int)((s + TB - 1) / TB);
  cudaError_t e = cudaSuccess;
  const int ntasks = (int)chol_ntasks(nt);
  int4* tasks = nullptr;
  if ((e = cudaMallocAsync(&tasks, (size_t)ntasks * sizeof(int4), st))) return e;
  launch_k(gen_chol_tasks, nt, 256, 0, st, tasks, nt);
  if (check_on()) check_tasks(tasks, chol_tasks(nt), "chol");
  const int grid = std::min(dag_grid(), ntasks);
  int* flags = nullptr;
  const size_t nflag = 2 * (size_t)nt * nt + 2;
  if ((e = cudaMallocAsync(&flags, nflag * sizeof(int), st))) return e;
  if ((e = cudaMemsetAsync(flags, 0, nflag * sizeof(int), st))) return e;
  long long* tr = trace_alloc(ntasks);
  int* ctl = flags + 2 * (size_t)nt * nt;
  const int cst = cstage_on();
  CholDag a{G, s, nt, tasks, ntasks, flags, flags + (size_t)nt * nt, ctl, ctl + 1, evict_on(), Tb, enorm2, tau, keep, tr,
            zero_lower ? 1 : 0, cst, pipe_on()};
  {
    KScope sc(KC_PANEL, (double)s * s * s / 3.0, 8.0 * (double)s * s * 1.5);
    ++g_launches;
    if (cst) launch_k(chol_dag_kernel, std::min(grid, cstage_grid()), DAG_THREADS, DAG_SMEM_CSTAGE, st, a);
    else launch_k(chol_dag_kernel, grid, DAG_THREADS, DAG_SMEM, st, a);
  }
  if ((e = cudaGetLastError())) return e;
  if (tr) fprintf(stderr, "[dag chol] s %lld (%s), G %% 16 = %d, cstage %d\n", (long long)s, (s & 1) ? "odd" : "even",
                  (int)((uintptr_t)G & 15), cst);
  trace_report("chol", tr, ntasks, nt, st);
  if ((e = cudaFreeAsync(tasks, st))) return e;
  return cudaFreeAsync(flags, st);
}

// W(i,j) = T_ii R(i,j) for the tiles j > i (x = j), and Y_i = T_ii X_i in place (x = nt); T_ii =
// Y_ii^T from Tb, staged [k][m] as the chain does.  One 64^3 DMMA product per CTA.
__global__ void __launch_bounds__(DAG_THREADS) trsm_prescale_kernel(const double* __restrict__ R, int64_t s, int nt,
                                                                   const double* __restrict__ Tb, double* X, int k,
                                                                   double* __restrict__ W) {
  pdl_begin();
  extern __shared__ double sm_dag[];
  double* As = sm_dag;
  double* Bs = sm_dag + TB * TP;
  const int j = blockIdx.x, i = blockIdx.y;
  if (j < nt && j <= i) return;
  const int warp = threadIdx.x >> 5, rb = (warp >> 1) * 16, cb = (warp & 1) * 32;
  const int nri = tile_n(s - (int64_t)TB * i);
  const bool xb = j == nt;
  const int ncj = xb ? k : tile_n(s - (int64_t)TB * j);
  const double* src = xb ? X + (int64_t)TB * i * k : R + (int64_t)TB * i * s + (int64_t)TB * j;
  const int64_t ld = xb ? k : s;
  stage2<false, false>(As, Tb + (int64_t)i * TB * TB, TB, TB, TB, Bs, src, ld, nri, ncj);
  __syncthreads();
  double acc[2][4][2];
  acc_zero(acc);
  mma64<false>(acc, As, Bs, rb, cb);
  double* dst = xb ? X + (int64_t)TB * i * k : W + (int64_t)TB * i * s + (int64_t)TB * j;
  acc_store(acc, dst, ld, nri, ncj, rb, cb);
}

int trsm_pre_on() {  // TSVD_TRSM_PRE=0: the chain applies T_jj itself (two products per step)
  static const int v = !(getenv("TSVD_TRSM_PRE") && atoi(getenv("TSVD_TRSM_PRE")) == 0);
  return v;
}

cudaError_t trsm_dag(cudaStream_t st, const double* R, int64_t s, const double* Tb, double* X, int k) {
  if (s <= 0 || k <= 0) return cudaSuccess;
  const int nt = (int)((s + TB - 1) / TB), nkb = (k + TB - 1) / TB;
  cudaError_t e = cudaSuccess;
  const int ntasks = (int)trsm_ntasks(nt, nkb);
  int4* tasks = nullptr;
  if ((e = cudaMallocAsync(&tasks, (size_t)ntasks * sizeof(int4), st))) return e;
  launch_k(gen_trsm_tasks, nt, 256, 0, st, tasks, nt, nkb);
  if (check_on()) check_tasks(tasks, trsm_tasks(nt, nkb), "trsm");
  const int grid = std::min(trsm_grid(), ntasks);
  int* flags = nullptr;
  const size_t nflag = 2 * (size_t)nt * nkb + 2;
  if ((e = cudaMallocAsync(&flags, nflag * sizeof(int), st))) return e;
  if ((e = cudaMemsetAsync(flags, 0, nflag * sizeof(int), st))) return e;
  long long* tr = trace_alloc(ntasks);
  int* ctl = flags + 2 * (size_t)nt * nkb;
  // prescaled form when the chain takes its fast path (one column block, 16-byte rows)
  const bool pre = trsm_pre_on() && nkb == 1 && (s & 1) == 0 && ((uintptr_t)R & 15) == 0 && ((uintptr_t)Tb & 15) == 0 &&
                   ((uintptr_t)X & 15) == 0 && (k & 1) == 0;
  double* W = nullptr;
  if (pre) {
    if ((e = cudaMallocAsync(&W, (size_t)s * s * sizeof(double), st))) return e;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(trsm_prescale_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * TB * TP * 8));
      attr = true;
    }
    ++g_launches;
    launch_k(trsm_prescale_kernel, dim3(nt + 1, nt), DAG_THREADS, (size_t)2 * TB * TP * sizeof(double), st, R, s, nt, Tb,
             X, k, W);
  }
  TrsmDag a{pre ? W : R, s, nt, nkb, k, Tb, X, tasks, ntasks, flags, flags + (size_t)nt * nkb, ctl, ctl + 1, evict_on(),
            tr, pre ? 1 : 0};
  {
    KScope sc(KC_PANEL, (double)s * s * k, 8.0 * ((double)s * s / 2.0 + 2.0 * s * k));
    ++g_launches;
    launch_k(trsm_dag_kernel, grid, DAG_THREADS, TRSM_SMEM, st, a);
  }
  if ((e = cudaGetLastError())) return e;
  trace_report("trsm", tr, ntasks, nt, st);
  if (W && (e = cudaFreeAsync(W, st))) return e;
  if ((e = cudaFreeAsync(tasks, st))) return e;
  return cudaFreeAsync(flags, st);
}

}  // namespace tsvd
