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
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "ops.h"

namespace tsvd {

namespace {
constexpr int TB = 64;         // tile
constexpr int TP = TB + 8;     // smem pitch of [k][m] operands (== 8 mod 16: conflict-free fragments)
constexpr int SUB = 16;        // sub-panel of the diagonal factorisation
constexpr int DAG_THREADS = 256;
constexpr size_t DAG_SMEM = 2 * (size_t)TB * TP * sizeof(double);  // >= TB * (2 TB + 4) doubles

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

enum : int { T_P = 0, T_S = 1, T_U = 2, T_F = 3, T_V = 4 };

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
__device__ __forceinline__ void publish(int* p, int v) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release(p, v);
  }
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

// acc (warp's 16 x 32 block: rows rb + 8a + g, cols cb + 8b + 2t{,+1}) += sign * As^T Bs,
// As, Bs in [k][m] layout.
template <bool NEG>
__device__ __forceinline__ void mma64(double (&acc)[2][4][2], const double* As, const double* Bs, int rb, int cb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll 4
  for (int kk = 0; kk < TB; kk += 4) {
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

// acc <-> global 64 x 64 block (row-major, ld), rows < nr, cols < nc
__device__ __forceinline__ void acc_load(double (&acc)[2][4][2], const double* C, int64_t ld, int nr, int nc, int rb,
                                         int cb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
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

__device__ void tile_potrf_inv(double* sm, double* D, int64_t ld, int nb, const double* __restrict__ en,
                               double tau, int32_t* __restrict__ keep, double* __restrict__ Yq) {
  double* A = sm;
  __shared__ double rinv[TB], en_s[TB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
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
  if (tid < TB) en_s[tid] = tid < nb ? en[tid] : 1.0;
  __syncthreads();
  for (int j0 = 0; j0 < TB; j0 += SUB) {
    const int j1 = j0 + SUB;
    if (warp == 0) {
      const int c = lane & 15, p = lane >> 4;
      double a[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = A[(j0 + 2 * m + p) * ALD + j0 + c];
#pragma unroll
      for (int i = 0; i < SUB; ++i) {
        const int src = (i & 1) * 16;
        const double d = __shfl_sync(0xffffffffu, a[i >> 1], src + i);
        const int gi = j0 + i;
        const bool real = gi < nb;
        const double e = en_s[gi];
        const bool kp = real && !(e == 0.0 || d <= tau * e);
        const double y = kp ? rsqrt(d) : (real ? 0.0 : 1.0);
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
        if (lane == 0) {
          rinv[gi] = y;
          if (real) keep[gi] = kp;
        }
      }
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int rr = 2 * m + p;
        if (c >= rr) A[(j0 + rr) * ALD + j0 + c] = a[m];
      }
    }
    __syncthreads();
    // row block: rows j0..j1 of the columns j1..63 of A and 64..64+j1 of [I] (64 columns)
    if (tid < TB) {
      const int col = tid < TB - j1 ? j1 + tid : TB + (tid - (TB - j1));
      double x[SUB];
#pragma unroll
      for (int q = 0; q < SUB; ++q) {
        double v = A[(j0 + q) * ALD + col];
#pragma unroll
        for (int u = 0; u < q; ++u) v = fma(-A[(j0 + u) * ALD + j0 + q], x[u], v);
        x[q] = v * rinv[j0 + q];
        A[(j0 + q) * ALD + col] = x[q];
      }
    }
    __syncthreads();
    if (j1 < TB) {
      // trailing: A[j1:, j1:] (upper tiles) and the right block rows j1.., columns < j1
      const int ntl = (TB - j1) / 8, nup = ntl * ntl, nright = ntl * (j1 / 8);
      for (int tile = warp; tile < nup + nright; tile += DAG_THREADS / 32) {
        int r0, c0;
        if (tile < nup) {
          const int tr = tile / ntl, tc = tile % ntl;
          if (tr > tc) continue;
          r0 = j1 + tr * 8;
          c0 = j1 + tc * 8;
        } else {
          const int x = tile - nup, nc = j1 / 8;
          r0 = j1 + (x / nc) * 8;
          c0 = TB + (x % nc) * 8;
        }
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < SUB; kk += 4)
          dmma8x8x4(a0, a1, A[(j0 + kk + t) * ALD + r0 + g], A[(j0 + kk + t) * ALD + c0 + g]);
        const int r = r0 + g, c = c0 + 2 * t;
        if (c0 >= TB || r <= c) A[r * ALD + c] -= a0;
        if (c0 >= TB || r <= c + 1) A[r * ALD + c + 1] -= a1;
      }
      __syncthreads();
    }
  }
  {
    const int c = tid & (TB - 1), r0 = tid >> 6;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int r = r0 + 4 * u;
      if (r < nb && c < nb) __stcg(D + (int64_t)r * ld + c, c >= r ? A[r * ALD + c] : 0.0);
      __stcg(Yq + r * TB + c, (r < nb && c < nb) ? A[r * ALD + TB + c] : 0.0);
    }
  }
}

struct CholDag {
  double* G;
  int64_t s;
  int nt;
  const int4* tasks;
  int ntasks;
  int* fin;  // nt x nt: tile (q,c) of R final
  int* ver;  // nt x nt: updates applied to tile (i,c)
  int* ticket;
  double* Tb;  // nt x 64 x 64: Y_qq = R_qq^{-T} (row-major), T_qq = Y_qq^T
  const double* en;
  double tau;
  int32_t* keep;
  long long* trace;  // optional (TSVD_DAG_TRACE): per task {type | smid << 8, claimed, ready, done} (ns)
};

__global__ void __launch_bounds__(DAG_THREADS, 2) chol_dag_kernel(CholDag a) {
  extern __shared__ double sm_dag[];
  double* As = sm_dag;
  double* Bs = sm_dag + TB * TP;
  __shared__ int tk;
  const int warp = threadIdx.x >> 5, rb = (warp >> 1) * 16, cb = (warp & 1) * 32;
  const int64_t s = a.s;
  for (;;) {
    if (threadIdx.x == 0) tk = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int it = tk;
    if (it >= a.ntasks) return;
    TaskTrace tt{a.trace};
    tt.claimed();
    const int4 task = a.tasks[it];
    const int q = task.y, i = task.z, c = task.w;
    const int nri = tile_n(s - (int64_t)TB * i), nrc = tile_n(s - (int64_t)TB * c);
    if (task.x == T_P) {
      wait_ge(a.ver + q * a.nt + q, q);
      tt.ready();
      double* D = a.G + (int64_t)TB * q * s + (int64_t)TB * q;
      tile_potrf_inv(sm_dag, D, s, nrc, a.en + (int64_t)TB * q, a.tau, a.keep + (int64_t)TB * q,
                     a.Tb + (int64_t)q * TB * TB);
      publish(a.fin + q * a.nt + q, 1);
    } else if (task.x == T_S) {
      wait_ge(a.fin + q * a.nt + q, 1);
      wait_ge(a.ver + q * a.nt + c, q);
      tt.ready();
      double* B = a.G + (int64_t)TB * q * s + (int64_t)TB * c;
      stage2<true, false>(As, a.Tb + (int64_t)q * TB * TB, TB, TB, TB, Bs, B, s, TB, nrc);  // T^T = Y
      __syncthreads();
      double acc[2][4][2];
      acc_zero(acc);
      mma64<false>(acc, As, Bs, rb, cb);
      acc_store(acc, B, s, TB, nrc, rb, cb);
      // mirror tile (c, q) of the lower triangle := 0
      double* L = a.G + (int64_t)TB * c * s + (int64_t)TB * q;
      for (int e = threadIdx.x; e < nrc * TB; e += DAG_THREADS) __stcg(L + (int64_t)(e >> 6) * s + (e & (TB - 1)), 0.0);
      publish(a.fin + q * a.nt + c, 1);
    } else {  // T_U: A(i,c) -= R(q,i)^T R(q,c)
      wait_ge(a.fin + q * a.nt + i, 1);
      wait_ge(a.fin + q * a.nt + c, 1);
      wait_ge(a.ver + i * a.nt + c, q);
      tt.ready();
      stage2<false, false>(As, a.G + (int64_t)TB * q * s + (int64_t)TB * i, s, TB, nri, Bs,
                           a.G + (int64_t)TB * q * s + (int64_t)TB * c, s, TB, nrc);
      double* C = a.G + (int64_t)TB * i * s + (int64_t)TB * c;
      double acc[2][4][2];
      acc_load(acc, C, s, nri, nrc, rb, cb);
      __syncthreads();
      mma64<true>(acc, As, Bs, rb, cb);
      acc_store(acc, C, s, nri, nrc, rb, cb);
      publish(a.ver + i * a.nt + c, q + 1);
    }
    tt.done(it, task.x);
    __syncthreads();  // smem and tk reuse
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
  int* ver;  // nt x nkb: updates applied
  int* ticket;
  long long* trace;
};

__global__ void __launch_bounds__(DAG_THREADS, 2) trsm_dag_kernel(TrsmDag a) {
  extern __shared__ double sm_dag[];
  double* As = sm_dag;
  double* Bs = sm_dag + TB * TP;
  __shared__ int tk;
  const int warp = threadIdx.x >> 5, rb = (warp >> 1) * 16, cb = (warp & 1) * 32;
  const int64_t s = a.s;
  for (;;) {
    if (threadIdx.x == 0) tk = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int it = tk;
    if (it >= a.ntasks) return;
    TaskTrace tt{a.trace};
    tt.claimed();
    const int4 task = a.tasks[it];
    const int j = task.y, i = task.z, b = task.w;  // F: j == i
    const int nri = tile_n(s - (int64_t)TB * i), nrj = tile_n(s - (int64_t)TB * j);
    const int ncb = min(TB, a.k - TB * b);
    double* Xi = a.X + (int64_t)TB * i * a.k + (int64_t)TB * b;
    double acc[2][4][2];
    if (task.x == T_F) {  // X_i = T_ii X_i
      wait_ge(a.ver + i * a.nkb + b, a.nt - 1 - i);
      tt.ready();
      stage2<false, false>(As, a.Tb + (int64_t)i * TB * TB, TB, TB, TB, Bs, Xi, a.k, nri, ncb);  // T = Y^T
      __syncthreads();
      acc_zero(acc);
      mma64<false>(acc, As, Bs, rb, cb);
      acc_store(acc, Xi, a.k, nri, ncb, rb, cb);
      publish(a.fin + i * a.nkb + b, 1);
    } else {  // T_V: X_i -= R(i,j) X_j, j > i
      wait_ge(a.fin + j * a.nkb + b, 1);
      wait_ge(a.ver + i * a.nkb + b, a.nt - 1 - j);
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
  }
}

// ---- task lists (built once per shape on the host, cached on the device)
std::vector<int4> chol_tasks(int nt) {
  std::vector<int4> v;
  auto U = [&](int q, int i) {
    for (int c = i; c < nt; ++c) v.push_back(make_int4(T_U, q, i, c));
  };
  for (int j = 0; j < nt; ++j) {
    v.push_back(make_int4(T_P, j, j, j));
    for (int c = j + 1; c < nt; ++c) v.push_back(make_int4(T_S, j, j, c));
    if (j + 1 < nt) {
      if (j >= 1) U(j - 1, j + 1);  // tile row j+1 by panel j-1, then by panel j (look-ahead)
      U(j, j + 1);
    }
    if (j >= 1)
      for (int i = j + 2; i < nt; ++i) U(j - 1, i);  // bulk of panel j-1
  }
  return v;
}

std::vector<int4> trsm_tasks(int nt, int nkb) {
  std::vector<int4> v;
  auto V = [&](int j, int i) {
    for (int b = 0; b < nkb; ++b) v.push_back(make_int4(T_V, j, i, b));
  };
  for (int j = nt - 1; j >= 0; --j) {
    for (int b = 0; b < nkb; ++b) v.push_back(make_int4(T_F, j, j, b));
    if (j >= 1) {
      if (j + 1 < nt) V(j + 1, j - 1);
      V(j, j - 1);
    }
    if (j + 1 < nt)
      for (int i = j - 2; i >= 0; --i) V(j + 1, i);
  }
  return v;
}

// The same orders generated on the device into stream-ordered scratch (no host allocation or
// synchronisation per shape): one CTA per iteration j, its offset from the closed-form sizes.
__host__ __device__ inline int64_t tri(int64_t n) { return n > 0 ? n * (n + 1) / 2 : 0; }
__host__ __device__ inline int64_t chol_iter_size(int nt, int j) {
  const int64_t m = nt - 1 - j;
  return 1 + m * (j >= 1 ? 3 : 2) + (j >= 1 ? tri(nt - j - 2) : 0);
}
__host__ __device__ inline int64_t trsm_iter_size(int nt, int nkb, int j) {
  int64_t n = 1;
  if (j >= 1) n += (j + 1 < nt) + 1;
  if (j + 1 < nt && j >= 2) n += j - 1;
  return n * nkb;
}
int64_t chol_ntasks(int nt) {
  int64_t n = 0;
  for (int j = 0; j < nt; ++j) n += chol_iter_size(nt, j);
  return n;
}
int64_t trsm_ntasks(int nt, int nkb) {
  int64_t n = 0;
  for (int j = 0; j < nt; ++j) n += trsm_iter_size(nt, nkb, j);
  return n;
}

__global__ void gen_chol_tasks(int4* out, int nt) {
  const int j = blockIdx.x;
  __shared__ int64_t off_s;
  if (threadIdx.x == 0) {
    int64_t o = 0;
    for (int q = 0; q < j; ++q) o += chol_iter_size(nt, q);
    off_s = o;
  }
  __syncthreads();
  int4* o = out + off_s;
  const int64_t n = chol_iter_size(nt, j), m = nt - 1 - j;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    int64_t x = e;
    int4 t;
    if (x == 0) {
      t = make_int4(T_P, j, j, j);
    } else if ((x -= 1) < m) {
      t = make_int4(T_S, j, j, j + 1 + (int)x);
    } else if ((x -= m), j >= 1 && x < m) {
      t = make_int4(T_U, j - 1, j + 1, j + 1 + (int)x);
    } else {
      if (j >= 1) x -= m;
      if (x < m) {
        t = make_int4(T_U, j, j + 1, j + 1 + (int)x);
      } else {
        x -= m;  // bulk of panel j-1: rows i = j+2.., nt - i entries each
        int i = j + 2;
        while (x >= nt - i) x -= nt - i++;
        t = make_int4(T_U, j - 1, i, i + (int)x);
      }
    }
    o[e] = t;
  }
}

__global__ void gen_trsm_tasks(int4* out, int nt, int nkb) {
  const int j = nt - 1 - (int)blockIdx.x;  // iterations run j = nt-1 .. 0
  __shared__ int64_t off_s;
  if (threadIdx.x == 0) {
    int64_t o = 0;
    for (int q = nt - 1; q > j; --q) o += trsm_iter_size(nt, nkb, q);
    off_s = o;
  }
  __syncthreads();
  int4* o = out + off_s;
  const int64_t n = trsm_iter_size(nt, nkb, j) / nkb;
  for (int64_t e = threadIdx.x; e < n * nkb; e += blockDim.x) {
    int64_t x = e / nkb;
    const int b = (int)(e % nkb);
    int4 t;
    if (x == 0) {
      t = make_int4(T_F, j, j, b);
    } else {
      x -= 1;
      const int hasnext = (j >= 1 && j + 1 < nt);
      if (hasnext && x == 0) t = make_int4(T_V, j + 1, j - 1, b);
      else if (j >= 1 && x == hasnext) t = make_int4(T_V, j, j - 1, b);
      else t = make_int4(T_V, j + 1, j - 2 - (int)(x - hasnext - 1), b);
    }
    o[e] = t;
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
    cudaFuncSetAttribute(trsm_dag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DAG_SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chol_dag_kernel, DAG_THREADS, DAG_SMEM);
    n = sms * std::max(1, std::min(occ, 2));
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
  if (cudaMalloc(&p, (size_t)ntasks * 4 * sizeof(long long))) return nullptr;
  return p;
}
void trace_report(const char* what, long long* d, int ntasks, int nt, cudaStream_t st) {
  if (!d) return;
  std::vector<long long> h((size_t)ntasks * 4);
  cudaStreamSynchronize(st);
  cudaMemcpy(h.data(), d, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  long long t0 = h[1], t1 = h[3];
  double wait[5] = {0}, exec[5] = {0}, emax[5] = {0};
  int cnt[5] = {0};
  std::vector<long long> pdone;
  for (int i = 0; i < ntasks; ++i) {
    const long long* r = &h[4 * (size_t)i];
    const int ty = (int)(r[0] & 0xff);
    t0 = std::min(t0, r[1]);
    t1 = std::max(t1, r[3]);
    if (ty < 0 || ty > 4) continue;
    cnt[ty]++;
    wait[ty] += r[2] - r[1];
    exec[ty] += r[3] - r[2];
    emax[ty] = std::max(emax[ty], (double)(r[3] - r[2]));
    if (ty == T_P || ty == T_F) pdone.push_back(r[3]);
  }
  fprintf(stderr, "[dag %s] nt %d tasks %d span %.1f us\n", what, nt, ntasks, (t1 - t0) / 1e3);
  const char* nm[5] = {"P", "S", "U", "F", "V"};
  for (int ty = 0; ty < 5; ++ty)
    if (cnt[ty])
      fprintf(stderr, "  %s x%-7d wait %8.2f us  exec %7.2f us (max %7.2f)\n", nm[ty], cnt[ty], wait[ty] / cnt[ty] / 1e3,
              exec[ty] / cnt[ty] / 1e3, emax[ty] / 1e3);
  std::sort(pdone.begin(), pdone.end());
  if (pdone.size() > 1)
    fprintf(stderr, "  panel interval: mean %.2f us (first %.2f, last %.2f)\n",
            (pdone.back() - pdone.front()) / 1e3 / (pdone.size() - 1), (pdone[1] - pdone[0]) / 1e3,
            (pdone[pdone.size() - 1] - pdone[pdone.size() - 2]) / 1e3);
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
                     double* Tb) {
  if (s <= 0) return cudaSuccess;
  const int nt = (int)((s + TB - 1) / TB);
  cudaError_t e = cudaSuccess;
  const int ntasks = (int)chol_ntasks(nt);
  int4* tasks = nullptr;
  if ((e = cudaMallocAsync(&tasks, (size_t)ntasks * sizeof(int4), st))) return e;
  gen_chol_tasks<<<nt, 256, 0, st>>>(tasks, nt);
  if (check_on()) check_tasks(tasks, chol_tasks(nt), "chol");
  const int grid = std::min(dag_grid(), ntasks);
  int* flags = nullptr;
  const size_t nflag = 2 * (size_t)nt * nt + 1;
  if ((e = cudaMallocAsync(&flags, nflag * sizeof(int), st))) return e;
  if ((e = cudaMemsetAsync(flags, 0, nflag * sizeof(int), st))) return e;
  long long* tr = trace_alloc(ntasks);
  CholDag a{G, s, nt, tasks, ntasks, flags, flags + (size_t)nt * nt, flags + 2 * (size_t)nt * nt, Tb, enorm2, tau, keep,
            tr};
  {
    KScope sc(KC_PANEL, (double)s * s * s / 3.0, 8.0 * (double)s * s * 1.5);
    ++g_launches;
    chol_dag_kernel<<<grid, DAG_THREADS, DAG_SMEM, st>>>(a);
  }
  if ((e = cudaGetLastError())) return e;
  trace_report("chol", tr, ntasks, nt, st);
  if ((e = cudaFreeAsync(tasks, st))) return e;
  return cudaFreeAsync(flags, st);
}

cudaError_t trsm_dag(cudaStream_t st, const double* R, int64_t s, const double* Tb, double* X, int k) {
  if (s <= 0 || k <= 0) return cudaSuccess;
  const int nt = (int)((s + TB - 1) / TB), nkb = (k + TB - 1) / TB;
  cudaError_t e = cudaSuccess;
  const int ntasks = (int)trsm_ntasks(nt, nkb);
  int4* tasks = nullptr;
  if ((e = cudaMallocAsync(&tasks, (size_t)ntasks * sizeof(int4), st))) return e;
  gen_trsm_tasks<<<nt, 256, 0, st>>>(tasks, nt, nkb);
  if (check_on()) check_tasks(tasks, trsm_tasks(nt, nkb), "trsm");
  const int grid = std::min(dag_grid(), ntasks);
  int* flags = nullptr;
  const size_t nflag = 2 * (size_t)nt * nkb + 1;
  if ((e = cudaMallocAsync(&flags, nflag * sizeof(int), st))) return e;
  if ((e = cudaMemsetAsync(flags, 0, nflag * sizeof(int), st))) return e;
  long long* tr = trace_alloc(ntasks);
  TrsmDag a{R, s, nt, nkb, k, Tb, X, tasks, ntasks, flags, flags + (size_t)nt * nkb, flags + 2 * (size_t)nt * nkb, tr};
  {
    KScope sc(KC_PANEL, (double)s * s * k, 8.0 * ((double)s * s / 2.0 + 2.0 * s * k));
    ++g_launches;
    trsm_dag_kernel<<<grid, DAG_THREADS, DAG_SMEM, st>>>(a);
  }
  if ((e = cudaGetLastError())) return e;
  trace_report("trsm", tr, ntasks, nt, st);
  if ((e = cudaFreeAsync(tasks, st))) return e;
  return cudaFreeAsync(flags, st);
}

}  // namespace tsvd
