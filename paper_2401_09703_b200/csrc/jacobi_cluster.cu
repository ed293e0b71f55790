// jacobi_cluster.cu — K9: one-sided Jacobi of a core 128 < n <= 512 wide, resident in ONE
// thread-block cluster (SVD_k of the core: Alg 3 line 2 P:364, Alg 4 line 3 P:381, Alg 9
// line 2 P:1192; BASELINE.json north_star step 3 "a one-sided Jacobi kernel resident in one
// CTA cluster").
//
// Hestenes' method (the same rotation, tolerance and sweep rule as the one-CTA K7 of
// jacobi.cu): the columns of A (m x n, m <= 512) are orthogonalised by plane rotations; the
// converged column norms are the singular values and the normalised columns the left
// singular vectors.  A round of the round-robin ("circle") tournament rotates N/2 disjoint
// column pairs at once; N - 1 rounds make a sweep.
//
// Distribution over a cluster of C CTAs (C = 16, non-portable; 8 when 16 cannot be
// scheduled): global pair g = c P + i (P = N / 2C pairs per CTA) lives in CTA c, warp i; its
// two columns in CTA c's shared memory.  Between rounds the tournament moves every column one
// place along the circle  top_1 -> .. -> top_{N/2-1} -> bot_{N/2-1} -> .. -> bot_0 -> top_1
// (top_0 fixed).  Inside a CTA that move is a relabelling: the slots form conveyors whose
// buffers are used as rings (slot position j at global round R -> ring buffer (j - R) mod L),
// so no column is copied locally; only the conveyor exits cross CTAs — at most two columns per
// CTA per round, written by the rotating warp straight from its registers into the
// neighbour's inbox (DSMEM), then, after the cluster barrier, copied into the ring buffer the
// exit just vacated.  Per round: one cluster barrier and one CTA barrier, no kernel launches,
// no host round trips (the multi-launch K8 synchronised with the host once per sweep).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "ops.h"

namespace cg = cooperative_groups;

namespace tsvd {

namespace {

constexpr int K9_SWEEPS = 40;
constexpr int K9_MAXN = 512;

struct K9Geom {
  int C, c, P, N;
};

// conveyor position -> local ring buffer; the slot's position at round R
// c == 0 (C > 1):  top[0] fixed (buffer 0); ring of L = 2P - 1 over buffers 1..2P-1:
//                  j = P-1-i for bot[i], j = P-1+i for top[i >= 1]
// c == C-1:        ring of L = 2P over buffers 0..2P-1: j = i for top[i], j = 2P-1-i for bot[i]
// otherwise:       ring A (top[i], j = i) over buffers 0..P-1, ring B (bot[i], j = P-1-i) over P..2P-1
// ring position j at ring phase ph = R mod L (0 <= j, ph < L): no division on the round's path
__device__ __forceinline__ int ring_buf(int base, int L, int j, int ph) {
  const int x = j - ph;
  return base + (x < 0 ? x + L : x);
}
// the rings' lengths of this CTA: (LA, LB); c == 0: one ring 2P-1 (LA); c == C-1: one ring 2P (LA)
struct K9Phase {
  int a, b;  // R mod LA, R mod LB
};
__device__ __forceinline__ int slot_buf(const K9Geom& g, bool top, int i, const K9Phase& ph) {
  const int P = g.P;
  if (g.c == 0 && g.C > 1) {
    if (top && i == 0) return 0;
    return ring_buf(1, 2 * P - 1, top ? P - 1 + i : P - 1 - i, ph.a);
  }
  if (g.c == g.C - 1) return ring_buf(0, 2 * P, top ? i : 2 * P - 1 - i, ph.a);
  return top ? ring_buf(0, P, i, ph.a) : ring_buf(P, P, P - 1 - i, ph.b);
}
__device__ __forceinline__ void k9_advance(const K9Geom& g, K9Phase& ph) {
  const int LA = (g.c == 0 && g.C > 1) ? 2 * g.P - 1 : (g.c == g.C - 1 ? 2 * g.P : g.P);
  if (++ph.a == LA) ph.a = 0;
  if (++ph.b == g.P) ph.b = 0;
}

template <int NU>
__global__ void __launch_bounds__(512) jacobi_cluster_kernel(const double* __restrict__ A, int64_t lda, int m, int n,
                                                              int kk, double tol, double* __restrict__ theta,
                                                              double* __restrict__ F, int64_t ldf,
                                                              int* __restrict__ info, double* __restrict__ tiny_out) {
  pdl_begin();
  cg::cluster_group cl = cg::this_cluster();
  constexpr int LDM = 32 * NU;  // rows per buffer (zero padded)
  extern __shared__ __align__(16) double sm[];
  K9Geom geo;
  geo.C = (int)cl.num_blocks();
  geo.c = (int)cl.block_rank();
  geo.N = ((n + 2 * geo.C - 1) / (2 * geo.C)) * (2 * geo.C);
  geo.P = geo.N / (2 * geo.C);
  const int P = geo.P, N = geo.N, c = geo.c, C = geo.C;
  const int nbuf = 2 * P + 4;
  double* buf = sm;                                  // nbuf x LDM
  double* nrm2 = buf + (size_t)nbuf * LDM;           // nbuf
  double* alln = nrm2 + nbuf;                        // K9_MAXN: final norms by column id
  int* cid = reinterpret_cast<int*>(alln + K9_MAXN);  // nbuf
  __shared__ int rot_local;
  __shared__ int totals[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;

  // ---- load: global pair g = c P + i holds columns g (top) and N-1-g (bottom) at R = 0
  for (int i = 0; i < P; ++i) {
    for (int side = 0; side < 2; ++side) {
      const int g = c * P + i;
      const int col = side == 0 ? g : N - 1 - g;
      const int b = slot_buf(geo, side == 0, i, K9Phase{0, 0});
      for (int r = tid; r < LDM; r += nthr) buf[(size_t)b * LDM + r] = (col < n && r < m) ? A[(int64_t)col * lda + r] : 0.0;
      if (tid == 0) cid[b] = col;
    }
  }
  if (tid == 0) {
    rot_local = 0;
    totals[0] = totals[1] = 0;
  }
  cl.sync();

  const bool is_warp_pair = warp < P;
  long long R = 0;
  K9Phase ph{0, 0};
  int sweep = 0;
  bool conv = false;
  for (; sweep < K9_SWEEPS; ++sweep) {
    // exact squared norms at the sweep start (carried through the rotations within it)
    if (is_warp_pair) {
      for (int side = 0; side < 2; ++side) {
        const int b = slot_buf(geo, side == 0, warp, ph);
        double a = 0.0;
#pragma unroll
        for (int x = 0; x < NU; ++x) {
          const double v = buf[(size_t)b * LDM + lane + 32 * x];
          a = fma(v, v, a);
        }
        a = warp_sum(a);
        if (lane == 0) nrm2[b] = a;
      }
    }
    if (c == 0 && tid == 0) totals[(sweep + 1) & 1] = 0;
    __syncthreads();
    int local = 0;
    for (int step = 0; step < N - 1; ++step, ++R) {
      const int par = (int)(R & 1);
      if (is_warp_pair) {
        const int i = warp;
        const int bt = slot_buf(geo, true, i, ph), bb = slot_buf(geo, false, i, ph);
        // orientation by column id (the same pair always rotates the same way round)
        const bool tfirst = cid[bt] < cid[bb];
        const int bp = tfirst ? bt : bb, bq = tfirst ? bb : bt;
        double u[NU], v[NU];
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int x = 0; x < NU; ++x) {
          u[x] = buf[(size_t)bp * LDM + lane + 32 * x];
          v[x] = buf[(size_t)bq * LDM + lane + 32 * x];
          if (x & 1) c1 = fma(u[x], v[x], c1);
          else c0 = fma(u[x], v[x], c0);
        }
        const double cc = warp_sum(c0 + c1);
        const double a = nrm2[bp], b = nrm2[bq];
        double na = a, nb = b;
        const bool rot = a > 0.0 && b > 0.0 && cc * cc > (tol * tol) * (a * b);
        if (rot) {
          const double c2 = 2.0 * cc, h = b - a, g2 = h >= 0 ? c2 : -c2;
          const double D = fabs(h) + sqrt(fma(h, h, c2 * c2));
          const double qn = rsqrt(fma(D, D, c2 * c2));
          const double cs = D * qn, sn = g2 * qn;
#pragma unroll
          for (int x = 0; x < NU; ++x) {
            const double uu = u[x], vv = v[x];
            u[x] = cs * uu - sn * vv;
            v[x] = sn * uu + cs * vv;
          }
          const double t = g2 / D;
          na = fma(-t, cc, a);
          nb = fma(t, cc, b);
          ++local;
        }
        // exits: top[P-1] of every CTA but the last goes right (the neighbour's top entry),
        // bot[0] of every CTA but the first goes left (the neighbour's bottom entry)
        const bool top_exit = (i == P - 1) && (c < C - 1);
        const bool bot_exit = (i == 0) && (c > 0);
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          const bool is_top = (side == 0) == tfirst;  // u belongs to bp
          const int bsel = side == 0 ? bp : bq;
          const double nn = side == 0 ? na : nb;
          const bool ex = is_top ? top_exit : bot_exit;
          if (ex) {
            const int dst_rank = is_top ? c + 1 : c - 1;
            const int ib = 2 * P + par * 2 + (is_top ? 0 : 1);
            double* rb = cl.map_shared_rank(buf, dst_rank) + (size_t)ib * LDM;
#pragma unroll
            for (int x = 0; x < NU; ++x) rb[lane + 32 * x] = side == 0 ? u[x] : v[x];
            if (lane == 0) {
              *cl.map_shared_rank(nrm2 + ib, dst_rank) = nn;
              *cl.map_shared_rank(cid + ib, dst_rank) = cid[bsel];
            }
          } else if (rot) {
#pragma unroll
            for (int x = 0; x < NU; ++x) buf[(size_t)bsel * LDM + lane + 32 * x] = side == 0 ? u[x] : v[x];
            if (lane == 0) nrm2[bsel] = nn;
          }
        }
      }
      cl.sync();  // the exits have landed in the neighbours' inboxes; every read of this round is done
      // entries: the inbox of this round -> the ring buffer the exit vacated (entry position at R + 1)
      k9_advance(geo, ph);
      if (c > 0) {  // top entry (from the left)
        const int ib = 2 * P + par * 2 + 0;
        const int b = (c == C - 1) ? ring_buf(0, 2 * P, 0, ph.a) : ring_buf(0, P, 0, ph.a);
        for (int r = tid; r < LDM; r += nthr) buf[(size_t)b * LDM + r] = buf[(size_t)ib * LDM + r];
        if (tid == 0) {
          nrm2[b] = nrm2[ib];
          cid[b] = cid[ib];
        }
      }
      if (c < C - 1) {  // bottom entry (from the right)
        const int ib = 2 * P + par * 2 + 1;
        const int b = (c == 0) ? ring_buf(1, 2 * P - 1, 0, ph.a) : ring_buf(P, P, 0, ph.b);
        for (int r = tid; r < LDM; r += nthr) buf[(size_t)b * LDM + r] = buf[(size_t)ib * LDM + r];
        if (tid == 0) {
          nrm2[b] = nrm2[ib];
          cid[b] = cid[ib];
        }
      }
      __syncthreads();
    }
    // sweep end: the cluster-wide rotation count
    if (lane == 0 && local) atomicAdd(&rot_local, local);
    __syncthreads();
    if (tid == 0) {
      atomicAdd(cl.map_shared_rank(&totals[sweep & 1], 0), rot_local);
      rot_local = 0;
    }
    cl.sync();
    const int tot = *cl.map_shared_rank(&totals[sweep & 1], 0);
    if (tot == 0) {
      conv = true;
      break;
    }
  }
  // ---- final norms, by column id, broadcast to every CTA of the cluster
  if (is_warp_pair) {
    for (int side = 0; side < 2; ++side) {
      const int b = slot_buf(geo, side == 0, warp, ph);
      double a = 0.0;
#pragma unroll
      for (int x = 0; x < NU; ++x) {
        const double v = buf[(size_t)b * LDM + lane + 32 * x];
        a = fma(v, v, a);
      }
      a = warp_sum(a);
      const int id = cid[b];
      if (lane < C) *cl.map_shared_rank(alln + id, lane) = sqrt(a);
      if (lane == 0) nrm2[b] = sqrt(a);
    }
  }
  cl.sync();
  double fro = 0.0;
  for (int j = 0; j < n; ++j) fro = fma(alln[j], alln[j], fro);
  const double tiny = 1e-14 * sqrt(fro) + 1e-300;
  if (is_warp_pair) {
    for (int side = 0; side < 2; ++side) {
      const int b = slot_buf(geo, side == 0, warp, ph);
      const int id = cid[b];
      if (id >= n) continue;
      const double v = nrm2[b];
      int r = 0;
      for (int l = lane; l < n; l += 32) r += (alln[l] > v) || (alln[l] == v && l < id);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
      if (lane == 0) theta[r] = v;
      if (r < kk) {
        const double inv = v > tiny ? 1.0 / v : 0.0;
        for (int x = 0; x < NU; ++x) {
          const int row = lane + 32 * x;
          if (row < m) F[(int64_t)r * ldf + row] = buf[(size_t)b * LDM + row] * inv;
        }
      }
    }
  }
  if (c == 0 && tid == 0 && info) {
    info[0] = sweep + (conv ? 1 : 0);
    info[1] = conv ? 1 : 0;
    *tiny_out = tiny;
  }
  cl.sync();  // no CTA exits while others may still read its shared memory
}

// ---------------------------------------------------------------- K9 (blocked ordering)
// The same rotations in a two-level ("block-cyclic") tournament order: the N columns form 2C
// blocks of w = N / 2C; CTA c holds two of them (X, the top row of the block circle, and Y, the
// bottom row).  An outer round pairs every column of X with every column of Y in w inner rounds
// (warp i rotates X_i with Y_{(i+t) mod w} in inner round t: w disjoint pairs); the first outer
// round of a sweep also runs the pairs inside X and inside Y (a round robin within each block,
// w - 1 inner rounds).  Then the blocks move one place around the block circle (2C - 1 outer
// rounds per sweep cover every block pair once, so every column pair is rotated once per sweep:
// N - 1 inner rounds, as in the scalar order).  Inner rounds synchronise the CTA only; the
// cluster synchronises at the block moves: 3 (2C - 1) cluster barriers per sweep instead of
// N - 1.  Moves are pulls over DSMEM through a third block buffer:
//   phase 1: CTA c >= 1 pulls its next X (CTA c-1's X; CTA 0's Y for c = 1) into its spare S;
//   cluster barrier (every X has been read: each CTA's old X buffer is free);
//   phase 2: CTA c <= C-2 pulls its next Y (CTA c+1's Y) into its old X buffer (CTA 0: into its
//            Y buffer, read in phase 1; CTA 0's X, block position 0 of the circle, never moves);
//            CTA C-1's next Y is its own old X (a relabelling);
//   cluster barrier; relabel (X, Y, S) <- (S, old X, old Y) on every CTA but CTA 0.
// (A cluster barrier also precedes phase 1: a neighbour may still be rotating its blocks.)
__device__ __forceinline__ int bk_pos(int slot, int step, int w) {  // round robin within a block
  if (slot == 0) return 0;
  int x = slot - 1 + step;
  if (x >= w - 1) x -= w - 1;
  return 1 + x;
}

template <int NU>
__device__ __forceinline__ void k9_rotate(double* xp, double* xq, double* np_, double* nq_, double tol, int lane,
                                          int& local) {
  double u[NU], v[NU];
  double c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int x = 0; x < NU; ++x) {
    u[x] = xp[lane + 32 * x];
    v[x] = xq[lane + 32 * x];
    if (x & 1) c1 = fma(u[x], v[x], c1);
    else c0 = fma(u[x], v[x], c0);
  }
  const double cc = warp_sum(c0 + c1);
  const double a = *np_, b = *nq_;
  if (a > 0.0 && b > 0.0 && cc * cc > (tol * tol) * (a * b)) {
    const double c2 = 2.0 * cc, h = b - a, g2 = h >= 0 ? c2 : -c2;
    const double D = fabs(h) + sqrt(fma(h, h, c2 * c2));
    const double qn = rsqrt(fma(D, D, c2 * c2));
    const double cs = D * qn, sn = g2 * qn;
#pragma unroll
    for (int x = 0; x < NU; ++x) {
      xp[lane + 32 * x] = cs * u[x] - sn * v[x];
      xq[lane + 32 * x] = sn * u[x] + cs * v[x];
    }
    if (lane == 0) {
      const double t = g2 / D;
      *np_ = fma(-t, cc, a);
      *nq_ = fma(t, cc, b);
    }
    ++local;
  }
}

// Copy n double2 from another CTA's shared memory (DSMEM) into this CTA's: U remote loads in
// flight per thread before their stores (the plain loop waits for each remote load before the
// next: ~20 % of K9's time).  U = 4 for the blocks of up to 256 rows (n = 128: 1.36 -> 1.20 ms,
// C4's Ritz problem 1.27 -> 1.14 ms); the 384 / 512-row kernels stay at U = 1: at their
// 128-register budget the staging spilled and the inner rounds slowed more than the pulls gained)
template <int U>
__device__ __forceinline__ void dsmem_pull(double2* __restrict__ ds, const double2* __restrict__ rs, int n, int tid,
                                           int nthr) {
  for (int e0 = tid; e0 < n; e0 += U * nthr) {
    double2 t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * nthr;
      if (e < n) t[u] = rs[e];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * nthr;
      if (e < n) ds[e] = t[u];
    }
  }
}

template <int NU>
__global__ void __launch_bounds__(512) jacobi_cblock_kernel(const double* __restrict__ A, int64_t lda, int m, int n,
                                                             int kk, double tol, double* __restrict__ theta,
                                                             double* __restrict__ F, int64_t ldf,
                                                             int* __restrict__ info, double* __restrict__ tiny_out,
                                                             int kt) {
  pdl_begin();
  cg::cluster_group cl = cg::this_cluster();
  constexpr int LDM = 32 * NU;
  extern __shared__ __align__(16) double sm[];
  const int C = (int)cl.num_blocks(), c = (int)cl.block_rank();
  const int N = ((n + 4 * C - 1) / (4 * C)) * (4 * C);
  const int w = N / (2 * C);
  double* blk = sm;                                  // 3 x w x LDM
  double* nrm = blk + (size_t)3 * w * LDM;           // 3 x w (carried squared norms)
  double* alln = nrm + 3 * w;                        // K9_MAXN: final norms by column id
  int* cid = reinterpret_cast<int*>(alln + K9_MAXN);  // 3 x w
  int* topf = cid + 3 * w;                           // K9_MAXN: column id in the leading kt this sweep
  __shared__ int rot_local;
  __shared__ int totals[2];
  __shared__ int useskip;
  __shared__ double red_s[2][16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
  auto col = [&](int b, int j) { return blk + ((size_t)b * w + j) * LDM; };
  if (tid == 0) useskip = 0;
  int ix = 0, iy = 1, is = 2;
  // block positions of the circle: CTA c holds top block c and bottom block 2C-1-c
  for (int b = 0; b < 2; ++b) {
    const int bl = b == 0 ? c : 2 * C - 1 - c;
    for (int j = 0; j < w; ++j) {
      const int id = bl * w + j;
      double* d = col(b, j);
      for (int r = tid; r < LDM; r += nthr) d[r] = (id < n && r < m) ? A[(int64_t)id * lda + r] : 0.0;
      if (tid == 0) cid[b * w + j] = id;
    }
  }
  if (tid == 0) {
    rot_local = 0;
    totals[0] = totals[1] = 0;
  }
  cl.sync();
  // (ix, iy, is) of CTAs c >= 1 after q relabellings: (0,1,2) -> (2,0,1) -> (1,2,0) -> ..
  auto idx_of = [](int q, int which) {  // which 0: X, 1: Y
    const int r = q % 3;
    const int x = (3 - r) % 3;   // X buffer: 0, 2, 1, ..
    return which == 0 ? x : (x + 1) % 3;
  };
  int sweep = 0, q = 0;
  bool conv = false;
  for (; sweep < K9_SWEEPS; ++sweep) {
    if (warp < w) {  // exact squared norms at the sweep start
      for (int b = 0; b < 2; ++b) {
        const int bi = b == 0 ? ix : iy;
        const double* d = col(bi, warp);
        double a = 0.0;
#pragma unroll
        for (int x = 0; x < NU; ++x) a = fma(d[lane + 32 * x], d[lane + 32 * x], a);
        a = warp_sum(a);
        if (lane == 0) nrm[bi * w + warp] = a;
      }
    }
    if (c == 0 && tid == 0) totals[(sweep + 1) & 1] = 0;
    // Leading set (kt > 0: the caller needs only the kt largest triplets, e.g. SVD_k of a core
    // plus θ_{k+1}): the columns whose norm ranks below kt this sweep.  Once the rest (the tail)
    // has Frobenius norm below half the kt-th column norm, pairs of two tail columns are not
    // rotated: the leading columns are still made orthogonal to every column, so at convergence
    // A V = [A_1 A_2] with A_1 orthogonal to A_2 and A_1^T A_1 diagonal — an invariant split —
    // and ||A_2||_2 <= ||A_2||_F < θ_kt / 2 keeps A_1's norms the kt largest singular values.
    // Only the tail's internal orthogonalisation (about half the sweeps on the configs[3]
    // weight-update cores) is skipped; its values (theta beyond kt) are then column norms only.
    if (kt > 0 && kt < n) {
      __syncthreads();
      if (warp < w) {
        for (int b = 0; b < 2; ++b) {
          const int bi = b == 0 ? ix : iy;
          const int id = cid[bi * w + warp];
          if (lane < C) *cl.map_shared_rank(alln + id, lane) = nrm[bi * w + warp];
        }
      }
      cl.sync();
      double tail = 0.0, thk = 0.0;
      for (int j = tid; j < n; j += nthr) {
        const double v = alln[j];
        int r = 0;
        for (int l = 0; l < n; ++l) r += (alln[l] > v) || (alln[l] == v && l < j);
        topf[j] = r < kt;
        if (r >= kt) tail += v;
        if (r == kt - 1) thk = v;
      }
      tail = warp_sum(tail);
      thk = warp_max(thk);
      if (lane == 0) {
        red_s[0][warp] = tail;
        red_s[1][warp] = thk;
      }
      __syncthreads();
      if (tid == 0) {
        double ts = 0.0, tk = 0.0;
        for (int q2 = 0; q2 < nthr / 32; ++q2) {
          ts += red_s[0][q2];
          tk = fmax(tk, red_s[1][q2]);
        }
        useskip = ts < 0.25 * tk;   // squared norms: ||A_2||_F < θ_kt / 2
      }
      cl.sync();  // (every CTA has read alln before anyone writes it again)
    }
    __syncthreads();
    const bool skip_tail = useskip != 0;
    int local = 0;
    for (int o = 0; o < 2 * C - 1; ++o) {
      if (o == 0) {  // pairs inside X and inside Y
        for (int t = 0; t < w - 1; ++t) {
          if (warp < w) {
            const int half = w / 2, i = warp % half, bi = warp < half ? ix : iy;
            int p = bk_pos(i, t, w), qq = bk_pos(w - 1 - i, t, w);
            if (cid[bi * w + qq] < cid[bi * w + p]) { const int tt = p; p = qq; qq = tt; }
            if (!(skip_tail && !topf[cid[bi * w + p]] && !topf[cid[bi * w + qq]]))
              k9_rotate<NU>(col(bi, p), col(bi, qq), nrm + bi * w + p, nrm + bi * w + qq, tol, lane, local);
          }
          __syncthreads();
        }
      }
      // every X column with every Y column: warp i keeps X_i (and its carried norm) in
      // registers for the w inner rounds; only the visiting Y columns go through shared memory
      // (half the shared-memory traffic of a round, 16-byte accesses)
      {
        const int i = warp < w ? warp : 0;
        double2 xr[NU / 2];
        double2* xs = reinterpret_cast<double2*>(col(ix, i));
#pragma unroll
        for (int x = 0; x < NU / 2; ++x) xr[x] = xs[lane + 32 * x];
        double xa = nrm[ix * w + i];
        const int xid = cid[ix * w + i];
        const bool xtail = skip_tail && !topf[xid];
        for (int t = 0; t < w; ++t) {
          int j = i + t;
          if (j >= w) j -= w;
          if (warp < w && !(xtail && !topf[cid[iy * w + j]])) {
            double2* ys = reinterpret_cast<double2*>(col(iy, j));
            double2 yr[NU / 2];
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int x = 0; x < NU / 2; ++x) {
              yr[x] = ys[lane + 32 * x];
              c0 = fma(xr[x].x, yr[x].x, c0);
              c1 = fma(xr[x].y, yr[x].y, c1);
            }
            const double cc = warp_sum(c0 + c1);
            const double ya = nrm[iy * w + j];
            const bool xf = xid < cid[iy * w + j];  // orientation: p = the smaller column id
            const double a = xf ? xa : ya, b = xf ? ya : xa;
            if (a > 0.0 && b > 0.0 && cc * cc > (tol * tol) * (a * b)) {
              const double c2 = 2.0 * cc, h = b - a, g2 = h >= 0 ? c2 : -c2;
              const double D = fabs(h) + sqrt(fma(h, h, c2 * c2));
              const double qn = rsqrt(fma(D, D, c2 * c2));
              const double cs = D * qn, sn = g2 * qn;
              // p' = cs p - sn q, q' = sn p + cs q  with (p, q) = (x, y) or (y, x)
              const double sx = xf ? -sn : sn;   // x' = cs x + sx y
              const double sy = xf ? sn : -sn;   // y' = sy x + cs y
#pragma unroll
              for (int x = 0; x < NU / 2; ++x) {
                const double2 u = xr[x], v = yr[x];
                xr[x] = make_double2(fma(cs, u.x, sx * v.x), fma(cs, u.y, sx * v.y));
                ys[lane + 32 * x] = make_double2(fma(sy, u.x, cs * v.x), fma(sy, u.y, cs * v.y));
              }
              const double tt = g2 / D;
              const double na = fma(-tt, cc, a), nb = fma(tt, cc, b);
              xa = xf ? na : nb;
              if (lane == 0) nrm[iy * w + j] = xf ? nb : na;
              ++local;
            }
          }
          __syncthreads();
        }
        if (warp < w) {
#pragma unroll
          for (int x = 0; x < NU / 2; ++x) xs[lane + 32 * x] = xr[x];
          if (lane == 0) nrm[ix * w + i] = xa;
        }
      }
      // ---- block move (two pull phases; every CTA has finished this outer round's rotations)
      cl.sync();
      if (c >= 1) {
        const int src = c - 1;
        const int sb = (c == 1) ? 1 : idx_of(q, 0);  // CTA 0 keeps X in buffer 0, Y in 1
        const double2* rs = reinterpret_cast<const double2*>(cl.map_shared_rank(blk, src) + (size_t)sb * w * LDM);
        double2* ds = reinterpret_cast<double2*>(blk + (size_t)is * w * LDM);
        dsmem_pull<(NU <= 8 ? 4 : 1)>(ds, rs, w * LDM / 2, tid, nthr);
        if (tid < w) {
          nrm[is * w + tid] = *cl.map_shared_rank(nrm + sb * w + tid, src);
          cid[is * w + tid] = *cl.map_shared_rank(cid + sb * w + tid, src);
        }
      }
      cl.sync();
      if (c <= C - 2) {
        const int src = c + 1;
        const int sb = idx_of(q, 1);  // CTA c+1 >= 1: Y buffer of the common sequence
        const int db = (c == 0) ? 1 : ix;
        const double2* rs = reinterpret_cast<const double2*>(cl.map_shared_rank(blk, src) + (size_t)sb * w * LDM);
        double2* ds = reinterpret_cast<double2*>(blk + (size_t)db * w * LDM);
        dsmem_pull<(NU <= 8 ? 4 : 1)>(ds, rs, w * LDM / 2, tid, nthr);
        if (tid < w) {
          nrm[db * w + tid] = *cl.map_shared_rank(nrm + sb * w + tid, src);
          cid[db * w + tid] = *cl.map_shared_rank(cid + sb * w + tid, src);
        }
      }
      cl.sync();
      ++q;
      if (c >= 1) {
        const int ox = ix, oy = iy;
        ix = is;
        iy = ox;
        is = oy;
      }
    }
    if (lane == 0 && local) atomicAdd(&rot_local, local);
    __syncthreads();
    if (tid == 0) {
      atomicAdd(cl.map_shared_rank(&totals[sweep & 1], 0), rot_local);
      rot_local = 0;
    }
    cl.sync();
    const int tot = *cl.map_shared_rank(&totals[sweep & 1], 0);
    if (tot == 0) {
      conv = true;
      break;
    }
  }
  // ---- final norms, by column id, broadcast to every CTA of the cluster
  if (warp < w) {
    for (int b = 0; b < 2; ++b) {
      const int bi = b == 0 ? ix : iy;
      const double* d = col(bi, warp);
      double a = 0.0;
#pragma unroll
      for (int x = 0; x < NU; ++x) a = fma(d[lane + 32 * x], d[lane + 32 * x], a);
      a = warp_sum(a);
      const int id = cid[bi * w + warp];
      if (lane < C) *cl.map_shared_rank(alln + id, lane) = sqrt(a);
      if (lane == 0) nrm[bi * w + warp] = sqrt(a);
    }
  }
  cl.sync();
  double fro = 0.0;
  for (int j = 0; j < n; ++j) fro = fma(alln[j], alln[j], fro);
  const double tiny = 1e-14 * sqrt(fro) + 1e-300;
  if (warp < w) {
    for (int b = 0; b < 2; ++b) {
      const int bi = b == 0 ? ix : iy;
      const int id = cid[bi * w + warp];
      if (id >= n) continue;
      const double v = nrm[bi * w + warp];
      int r = 0;
      for (int l = lane; l < n; l += 32) r += (alln[l] > v) || (alln[l] == v && l < id);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
      if (lane == 0) theta[r] = v;
      if (r < kk) {
        const double inv = v > tiny ? 1.0 / v : 0.0;
        const double* d = col(bi, warp);
        for (int x = 0; x < NU; ++x) {
          const int row = lane + 32 * x;
          if (row < m) F[(int64_t)r * ldf + row] = d[row] * inv;
        }
      }
    }
  }
  if (c == 0 && tid == 0 && info) {
    info[0] = sweep + (conv ? 1 : 0);
    info[1] = conv ? 1 : 0;
    *tiny_out = tiny;
  }
  cl.sync();
}

template <int NU>
size_t k9b_smem(int w) {
  return ((size_t)3 * w * 32 * NU + 3 * w + K9_MAXN) * sizeof(double) + (3 * w + K9_MAXN) * sizeof(int) + 16;
}

template <int NU>
cudaError_t launch_k9b(cudaStream_t st, int C, const double* A, int64_t lda, int m, int n, int kk, double tol,
                       double* theta, double* F, int64_t ldf, int* info, double* tiny, int kt) {
  const int N = ((n + 4 * C - 1) / (4 * C)) * (4 * C);
  const int w = N / (2 * C);
  const size_t smem = k9b_smem<NU>(w);
  if (smem > 227 * 1024 || w > 16 || w < 2) return cudaErrorInvalidValue;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(jacobi_cblock_kernel<NU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
    return e;
  if ((e = cudaFuncSetAttribute(jacobi_cblock_kernel<NU>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1))) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(32 * std::max(w, 4));
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
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, jacobi_cblock_kernel<NU>, &cfg) != cudaSuccess || ncl < 1) {
    cudaGetLastError();
    return cudaErrorInvalidConfiguration;
  }
  return cudaLaunchKernelEx(&cfg, jacobi_cblock_kernel<NU>, A, lda, m, n, kk, tol, theta, F, ldf, info, tiny, kt);
}

template <int NU>
size_t k9_smem(int P) {
  return ((size_t)(2 * P + 4) * 32 * NU + (2 * P + 4) + K9_MAXN) * sizeof(double) + (2 * P + 4) * sizeof(int) + 16;
}

template <int NU>
cudaError_t launch_k9(cudaStream_t st, int C, const double* A, int64_t lda, int m, int n, int kk, double tol,
                      double* theta, double* F, int64_t ldf, int* info, double* tiny) {
  const int N = ((n + 2 * C - 1) / (2 * C)) * (2 * C);
  const int P = N / (2 * C);
  const size_t smem = k9_smem<NU>(P);
  if (smem > 227 * 1024 || P > 16 || P < 2) return cudaErrorInvalidValue;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(jacobi_cluster_kernel<NU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
    return e;
  if ((e = cudaFuncSetAttribute(jacobi_cluster_kernel<NU>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1))) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(32 * std::max(P, 4));
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
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, jacobi_cluster_kernel<NU>, &cfg) != cudaSuccess || ncl < 1) {
    cudaGetLastError();
    return cudaErrorInvalidConfiguration;
  }
  return cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel<NU>, A, lda, m, n, kk, tol, theta, F, ldf, info, tiny);
}

}  // namespace

bool k9_supported(int64_t m, int64_t n) { return n > 0 && m >= n && m <= K9_MAXN && n <= K9_MAXN; }

// K9 launch: the same outputs as K7 (theta: n values descending; F: m x kk normalised leading
// columns; info = {sweeps, converged}; tiny = 1e-14 ||A||_F).  Cluster of 16 CTAs, else 8.
cudaError_t jacobi_cluster(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, int kk, double tol,
                           double* theta, double* F, int64_t ldf, int* info, double* tiny, int kt) {
  if (!k9_supported(m, n)) return cudaErrorInvalidValue;
  cudaError_t e = cudaErrorInvalidConfiguration;
  static const bool scalar = getenv("TSVD_K9_SCALAR") && atoi(getenv("TSVD_K9_SCALAR")) == 1;
  // cluster size: the smallest of 4 / 8 / 16 CTAs whose blocks hold at most 12 columns (C2's
  // 96-column Ritz problems on 4 CTAs, C1's 116-column core and C4's 192 on 8, 384 and 512 on
  // 16 — fewer CTAs, fewer outer rounds and cluster barriers per sweep; measured per config,
  // profiles/r2_k9_cluster_sweep.log); TSVD_K9_C overrides (tuning)
  static const int c_env = getenv("TSVD_K9_C") ? atoi(getenv("TSVD_K9_C")) : 0;
  int c_pick = 16;
  for (int C : {4, 8}) {
    const int64_t N = (n + 4 * C - 1) / (4 * C) * (4 * C);
    if (N / (2 * C) <= 12) {
      c_pick = C;
      break;
    }
  }
  if (!scalar) {
    for (int C : {c_env > 0 ? c_env : c_pick, 16, 8}) {
      if (m <= 192) e = launch_k9b<6>(st, C, A, lda, (int)m, (int)n, kk, tol, theta, F, ldf, info, tiny, kt);
      else if (m <= 256) e = launch_k9b<8>(st, C, A, lda, (int)m, (int)n, kk, tol, theta, F, ldf, info, tiny, kt);
      else if (m <= 384) e = launch_k9b<12>(st, C, A, lda, (int)m, (int)n, kk, tol, theta, F, ldf, info, tiny, kt);
      else e = launch_k9b<16>(st, C, A, lda, (int)m, (int)n, kk, tol, theta, F, ldf, info, tiny, kt);
      if (e == cudaSuccess) return e;
      cudaGetLastError();
    }
  }
  for (int C : {16, 8}) {
    if (m <= 192) e = launch_k9<6>(st, C, A, lda, (int)m, (int)n, kk, tol, theta, F, ldf, info, tiny);
    else if (m <= 256) e = launch_k9<8>(st, C, A, lda, (int)m, (int)n, kk, tol, theta, F, ldf, info, tiny);
    else if (m <= 384) e = launch_k9<12>(st, C, A, lda, (int)m, (int)n, kk, tol, theta, F, ldf, info, tiny);
    else e = launch_k9<16>(st, C, A, lda, (int)m, (int)n, kk, tol, theta, F, ldf, info, tiny);
    if (e == cudaSuccess) break;
    cudaGetLastError();
  }
  return e;
}

}  // namespace tsvd
