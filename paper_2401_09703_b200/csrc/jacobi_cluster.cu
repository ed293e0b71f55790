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
__device__ __forceinline__ int ring_buf(int base, int L, int j, long long R) {
  const long long x = ((long long)j - R) % L;
  return base + (int)(x < 0 ? x + L : x);
}
__device__ __forceinline__ int slot_buf(const K9Geom& g, bool top, int i, long long R) {
  const int P = g.P;
  if (g.c == 0 && g.C > 1) {
    if (top && i == 0) return 0;
    return ring_buf(1, 2 * P - 1, top ? P - 1 + i : P - 1 - i, R);
  }
  if (g.c == g.C - 1) return ring_buf(0, 2 * P, top ? i : 2 * P - 1 - i, R);
  return top ? ring_buf(0, P, i, R) : ring_buf(P, P, P - 1 - i, R);
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
      const int b = slot_buf(geo, side == 0, i, 0);
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
  int sweep = 0;
  bool conv = false;
  for (; sweep < K9_SWEEPS; ++sweep) {
    // exact squared norms at the sweep start (carried through the rotations within it)
    if (is_warp_pair) {
      for (int side = 0; side < 2; ++side) {
        const int b = slot_buf(geo, side == 0, warp, R);
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
        const int bt = slot_buf(geo, true, i, R), bb = slot_buf(geo, false, i, R);
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
      if (c > 0) {  // top entry (from the left)
        const int ib = 2 * P + par * 2 + 0;
        const int b = (c == C - 1) ? ring_buf(0, 2 * P, 0, R + 1) : ring_buf(0, P, 0, R + 1);
        for (int r = tid; r < LDM; r += nthr) buf[(size_t)b * LDM + r] = buf[(size_t)ib * LDM + r];
        if (tid == 0) {
          nrm2[b] = nrm2[ib];
          cid[b] = cid[ib];
        }
      }
      if (c < C - 1) {  // bottom entry (from the right)
        const int ib = 2 * P + par * 2 + 1;
        const int b = (c == 0) ? ring_buf(1, 2 * P - 1, 0, R + 1) : ring_buf(P, P, 0, R + 1);
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
      const int b = slot_buf(geo, side == 0, warp, R);
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
      const int b = slot_buf(geo, side == 0, warp, R);
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
                           double* theta, double* F, int64_t ldf, int* info, double* tiny) {
  if (!k9_supported(m, n)) return cudaErrorInvalidValue;
  cudaError_t e = cudaErrorInvalidConfiguration;
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
