// sparse.cu — the nnz-proportional kernels of the update (HBM / L2 bound).
//
//   K1 build_csc    batch ingest: E (CSR over the s update vectors) -> CSC over the
//                   lift-side rows it touches, plus the touched list J.
//   K2 gather_spmm  Lemma 1: W = E X', reading only the X' rows E
//                   touches; warp per update vector, 128-bit row loads.
//   K3 sparse_gram  Lemma 2 inner products of the sparse parts: E E^T,
//                   warp per output row, accumulator in shared memory.
//   K10 scatter_add the "sparse matrix addition" of PAPER.md:307 / Alg 9 line 7
//                   (P:1200): X'[j] += sum_i E_ij Z[i], warp per touched row j of X'
//                   (CSC), no atomics on X'.
#include <algorithm>
#include <cstdlib>
#include <cfloat>
#include <climits>
#include <cstdint>


#include "ops.h"

namespace tsvd {

// ------------------------------------------------------------------ validation
namespace {
// Input validation in two flat passes (a warp per row was one warp's walk over a 2e5-nonzero
// power-law row: 0.7 ms on configs[4] batches).  Rows: the row_ptr range and monotonicity;
// nonzeros: column range, finite value, and columns ascending inside a row — a descent
// ci[p-1] >= ci[p] is legal only at a row start, found by a binary search of row_ptr.
__global__ void validate_rows_kernel(int64_t s, int64_t nnz, const int64_t* __restrict__ rp, int* flag) {
  pdl_begin();
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < s; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = rp[w], e = rp[w + 1];
    // the row_ptr endpoints are checked on the host after this kernel
    if (b < 0 || e > nnz || e < b) atomicOr(flag, 1);
  }
}
__global__ void validate_kernel(int64_t s, int64_t dim, int64_t nnz, const int64_t* __restrict__ rp,
                                const int32_t* __restrict__ ci, const double* __restrict__ v, int* flag) {
  pdl_begin();
  int bad = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int c = ci[p];
    if (c < 0 || c >= dim) bad |= 1;
    if (!isfinite(v[p])) bad |= 2;
    if (p > 0 && ci[p - 1] >= c) {  // legal only if p starts a row
      int64_t lo = 0, hi = s;        // the first row w with rp[w] >= p
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (rp[mid] < p) lo = mid + 1;
        else hi = mid;
      }
      if (lo > s || rp[lo] != p) bad |= 1;
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicOr(flag, bad);
}

// ------------------------------------------------------------------ exclusive scan (int64)
constexpr int SCAN_T = 1024, SCAN_I = 4, SCAN_TILE = SCAN_T * SCAN_I;

__global__ void __launch_bounds__(SCAN_T) scan_tile_kernel(const int64_t* __restrict__ in, int64_t* __restrict__ out,
                                                           int64_t n, int64_t* __restrict__ tile_tot) {
  pdl_begin();
  __shared__ int64_t wsum[32];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_I;
  int64_t x[SCAN_I], loc = 0;
#pragma unroll
  for (int i = 0; i < SCAN_I; ++i) {
    x[i] = (base + i < n) ? in[base + i] : 0;
    loc += x[i];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    int64_t ws = wsum[lane], wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    wsum[lane] = wi - ws;  // exclusive warp offsets
    if (lane == 31 && tile_tot) tile_tot[blockIdx.x] = wi;
  }
  __syncthreads();
  int64_t run = wsum[w] + inc - loc;
#pragma unroll
  for (int i = 0; i < SCAN_I; ++i) {
    if (base + i < n) out[base + i] = run;
    run += x[i];
  }
}

__global__ void scan_add_kernel(int64_t* out, int64_t n, const int64_t* __restrict__ tile_off) {
  pdl_begin();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += tile_off[i / SCAN_TILE];
}

cudaError_t scan_exclusive(cudaStream_t st, const int64_t* in, int64_t* out, int64_t n, Scratch& ws) {
  if (n <= 0) return cudaSuccess;
  const unsigned tiles = cdiv(n, SCAN_TILE);
  if (tiles == 1) {
    ++g_launches;
    launch_k(scan_tile_kernel, 1, SCAN_T, 0, st, in, out, n, nullptr);
    return cudaGetLastError();
  }
  int64_t* tot = ws.alloc<int64_t>(tiles);
  int64_t* off = ws.alloc<int64_t>(tiles);
  if (ws.err) return ws.err;
  g_launches += 2;
  launch_k(scan_tile_kernel, tiles, SCAN_T, 0, st, in, out, n, tot);
  cudaError_t e = scan_exclusive(st, tot, off, tiles, ws);
  if (e != cudaSuccess) return e;
  launch_k(scan_add_kernel, cdiv(n, 256), 256, 0, st, out, n, off);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K1 CSR -> CSC
__global__ void col_hist_kernel(int64_t nnz, const int32_t* __restrict__ ci, unsigned long long* cnt) {
  pdl_begin();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[ci[p]], 1ull);
}

__global__ void touched_flag_kernel(int64_t dim, const int64_t* __restrict__ cnt, int64_t* __restrict__ flag) {
  pdl_begin();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < dim) flag[j] = cnt[j] > 0 ? 1 : 0;
}

__global__ void compact_J_kernel(int64_t dim, const int64_t* __restrict__ cnt, const int64_t* __restrict__ pos,
                                 int32_t* __restrict__ J) {
  pdl_begin();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < dim && cnt[j] > 0) J[pos[j]] = (int32_t)j;
}

// CSC order by one radix sort of (column << 32 | row) keys: deterministic (rows ascending
// within every column, hub columns included) and O(nnz) regardless of column degree.
// per entry of a CSR: its column (the sort key) and its row
__global__ void csc_rows_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                uint32_t* __restrict__ key, int32_t* __restrict__ row) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s) return;
  for (int64_t p = rp[w] + lane; p < rp[w + 1]; p += 32) {
    key[p] = (uint32_t)ci[p];
    row[p] = (int32_t)w;
  }
}

// CSC entries through the sort permutation
__global__ void csc_gather_kernel(int64_t nnz, const int32_t* __restrict__ perm, const int32_t* __restrict__ rowof,
                                  const double* __restrict__ val, int32_t* __restrict__ row, double* __restrict__ cval) {
  pdl_begin();
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = perm[q];
    row[q] = rowof[p];
    cval[q] = val[p];
  }
}

constexpr int kLongRow = 32;   // longer rows: a CTA of LONG_WARPS warps each (cold gathers are latency bound)
// rows of 128-256-wide gathers stay on one warp up to 128 nonzeros: a CTA spends ~2 us per row
// whatever its length below ~100 (one gather latency, its reductions and barrier), so with
// configs[4]'s mean degree of 45 the 296 long-row CTAs served ~90k rows one at a time (1.2 ms
// per gather); a warp per row keeps the whole GPU's warps busy (the U = 4 loads in flight of
// 2 KB rows cover the latency)
__host__ __device__ constexpr int long_row_threshold(int K) { return K >= 128 ? 128 : kLongRow; }
constexpr int LONG_WARPS = 32;
// acc += sum over p = begin, begin + step, .. < end of val[p] * X[idx[p], lane slice], four
// nonzeros' loads in flight per iteration, the FMAs applied in p order (the same sum as one
// nonzero at a time; the loops are otherwise bound by one dependent load pair per nonzero)
template <int LANES, int VEC, bool STREAM>
__device__ __forceinline__ void accum_rows(double2 (&acc)[VEC], int64_t begin, int64_t end, int64_t step,
                                           const int32_t* __restrict__ idx, const double* __restrict__ val,
                                           const double* __restrict__ X, int li, int64_t ldx = 2 * LANES * VEC) {
  constexpr int U = 4;
  int64_t p = begin;
  for (; p + (U - 1) * step < end; p += U * step) {
    int c[U];
    double vv[U];
    double2 a[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = STREAM ? ld_stream_i32(idx + p + u * step) : idx[p + u * step];
      vv[u] = STREAM ? ld_stream_f64(val + p + u * step) : val[p + u * step];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double2* x0 = reinterpret_cast<const double2*>(X + (int64_t)c[u] * ldx) + li;
#pragma unroll
      for (int q = 0; q < VEC; ++q) a[u][q] = x0[q * LANES];
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        acc[q].x = fma(vv[u], a[u][q].x, acc[q].x);
        acc[q].y = fma(vv[u], a[u][q].y, acc[q].y);
      }
  }
  for (; p < end; p += step) {
    const int c0 = STREAM ? ld_stream_i32(idx + p) : idx[p];
    const double v0 = STREAM ? ld_stream_f64(val + p) : val[p];
    const double2* x0 = reinterpret_cast<const double2*>(X + (int64_t)c0 * ldx) + li;
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      const double2 a = x0[q * LANES];
      acc[q].x = fma(v0, a.x, acc[q].x);
      acc[q].y = fma(v0, a.y, acc[q].y);
    }
  }
}
// ------------------------------------------------------------------ K2 gather-SpMM
// Rows longer than kLongRow (power-law hubs: up to thousands of nonzeros in one update vector)
// get a whole CTA of LONG_WARPS warps: (32 / LANES) groups per warp stride over the row's
// nonzeros, four loads in flight each; the partial rows are combined in a fixed order
// (shuffles within a warp, then shared memory across warps) — deterministic, no atomics.
// The long rows are listed first (long_list_kernel); the CTAs loop over the list.
__global__ void long_list_kernel(int64_t n, const int32_t* __restrict__ rowid, const int64_t* __restrict__ ptr,
                                 int32_t* __restrict__ list, int* __restrict__ cnt, int thr) {
  pdl_begin();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t row = rowid ? rowid[r] : r;
  if (ptr[row + 1] - ptr[row] > thr) list[atomicAdd(cnt, 1)] = (int32_t)r;
}

template <int LANES, int VEC>
struct LongCfg {  // warps per long-row CTA: the partial rows must fit 48 KB of static shared memory
  static constexpr int K = 2 * LANES * VEC;
  static constexpr int WARPS = (K / 2) * 16 * LONG_WARPS <= 48 * 1024 ? LONG_WARPS : (48 * 1024) / ((K / 2) * 16);
};
// Rows longer than kChunk nonzeros (the heaviest power-law rows: configs[4] batches hold rows
// of 1e5 nonzeros, 200 MB of gathers, which one CTA streams at ~100 GB/s) are cut into chunks
// of kChunk, one work item each: the long-row CTAs loop over the items, a one-chunk row is
// written as before, a multi-chunk row's chunks write partial rows that chunk_reduce_kernel sums
// in chunk order — deterministic, no atomics.
constexpr int kChunk = 4096;
struct LongPlan {
  int32_t* list = nullptr;  // long rows (positions in the row set), cnt of them
  int* cnt = nullptr;
  int64_t* nch = nullptr;   // chunks per listed row (n + 1, zero past cnt)
  int64_t* base = nullptr;  // exclusive scan of nch: first item of the row
  int64_t* base2 = nullptr; // exclusive scan of the multi-chunk rows' chunk counts: first partial row
  int2* items = nullptr;    // (list position, chunk)
  double* part = nullptr;   // partial rows of the multi-chunk rows' items
  int64_t max_items = 0;
};
__global__ void long_nch_kernel(int64_t n, const int32_t* __restrict__ list, const int* __restrict__ cnt,
                                const int32_t* __restrict__ rowid, const int64_t* __restrict__ ptr,
                                int64_t* __restrict__ nch, int64_t* __restrict__ nch2) {
  pdl_begin();
  const int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (h > n) return;
  int64_t c = 0;
  if (h < *cnt) {
    const int64_t r = list[h];
    const int64_t row = rowid ? rowid[r] : r;
    c = (ptr[row + 1] - ptr[row] + kChunk - 1) / kChunk;
  }
  nch[h] = c;
  nch2[h] = c > 1 ? c : 0;   // the partial rows only multi-chunk rows write
}
__global__ void long_items_kernel(int64_t n, const int* __restrict__ cnt, const int64_t* __restrict__ nch,
                                  const int64_t* __restrict__ base, int2* __restrict__ items) {
  pdl_begin();
  const int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= *cnt) return;
  for (int64_t c = 0; c < nch[h]; ++c) items[base[h] + c] = make_int2((int)h, (int)c);
}
template <bool CSC>
__global__ void chunk_reduce_kernel(const int32_t* __restrict__ list, const int* __restrict__ cnt,
                                    const int32_t* __restrict__ rowid, const int64_t* __restrict__ nch,
                                    const int64_t* __restrict__ base2, const double* __restrict__ part, int K,
                                    double* __restrict__ out, int64_t ldo) {
  pdl_begin();
  const int nl = *cnt;
  for (int h = blockIdx.x; h < nl; h += gridDim.x) {
    const int64_t nc = nch[h];
    if (nc < 2) continue;
    const int64_t r = list[h];
    const int64_t row = CSC ? rowid[r] : r;
    for (int t = threadIdx.x; t < K; t += blockDim.x) {
      double a = 0.0;
      for (int64_t c = 0; c < nc; ++c) a += part[(base2[h] + c) * K + t];
      if (CSC) out[row * ldo + t] += a;
      else out[row * ldo + t] = a;
    }
  }
}

template <int LANES, int VEC, bool CSC>
__global__ void __launch_bounds__(32 * LongCfg<LANES, VEC>::WARPS) rowsum_long_kernel(const int32_t* __restrict__ list,
                                                                      const int* __restrict__ cnt,
                                                                      const int32_t* __restrict__ rowid,
                                                                      const int64_t* __restrict__ ptr,
                                                                      const int32_t* __restrict__ idx,
                                                                      const double* __restrict__ v,
                                                                      const double* __restrict__ X,
                                                                      double* __restrict__ out, int64_t ldx,
                                                                      int64_t ldo, const int2* __restrict__ items,
                                                                      const int64_t* __restrict__ nch,
                                                                      const int64_t* __restrict__ base,
                                                                      const int64_t* __restrict__ base2,
                                                                      double* __restrict__ part) {
  pdl_begin();
  constexpr int K = 2 * LANES * VEC;
  constexpr int G = 32 / LANES;
  constexpr int NWL = LongCfg<LANES, VEC>::WARPS;
  __shared__ double2 red[NWL][K / 2];
  const int nl = items ? (int)base[*cnt] : *cnt;
  for (int it = blockIdx.x; it < nl; it += gridDim.x) {
  const int h = items ? items[it].x : it;
  const int64_t r = list[h];
  const int64_t row = CSC ? rowid[r] : r;  // CSC: the touched column J[r] of X
  int64_t b = ptr[row], e = ptr[row + 1];
  const bool chunked = items && nch[h] > 1;
  if (items) {
    b += (int64_t)items[it].y * kChunk;
    e = min(e, b + kChunk);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, grp = lane / LANES, li = lane % LANES;
  double2 acc[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) acc[q] = make_double2(0.0, 0.0);
  accum_rows<LANES, VEC, false>(acc, b + warp * G + grp, e, NWL * G, idx, v, X, li, ldx);
#pragma unroll
  for (int o = LANES; o < 32; o <<= 1)
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      acc[q].x += __shfl_xor_sync(0xffffffffu, acc[q].x, o);
      acc[q].y += __shfl_xor_sync(0xffffffffu, acc[q].y, o);
    }
  if (grp == 0)
#pragma unroll
    for (int q = 0; q < VEC; ++q) red[warp][q * LANES + li] = acc[q];
  __syncthreads();
  for (int c = threadIdx.x; c < K / 2; c += blockDim.x) {
    double2 t = red[0][c];
    for (int w = 1; w < NWL; ++w) {
      t.x += red[w][c].x;
      t.y += red[w][c].y;
    }
    if (chunked) {
      reinterpret_cast<double2*>(part + (base2[h] + items[it].y) * K)[c] = t;
      continue;
    }
    double2* o = reinterpret_cast<double2*>(out + row * ldo) + c;
    if (CSC) {
      double2 x = *o;
      x.x += t.x;
      x.y += t.y;
      *o = x;
    } else {
      *o = t;
    }
  }
  __syncthreads();  // red reused by the next row
  }
}

// LANES lanes per nonzero, each owning VEC double2 of the k-row; 32/LANES nonzeros in flight.
template <int LANES, int VEC>
__global__ void __launch_bounds__(256) gather_spmm_kernel(int64_t s, const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ ci, const double* __restrict__ v,
                                                          const double* __restrict__ X, double* __restrict__ W,
                                                          int64_t ldx = 2 * LANES * VEC, int64_t ldw = 2 * LANES * VEC) {
  pdl_begin();
  constexpr int K = 2 * LANES * VEC;
  constexpr int G = 32 / LANES;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= s) return;
  const int lane = threadIdx.x & 31, grp = lane / LANES, li = lane % LANES;
  double2 acc[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) acc[q] = make_double2(0.0, 0.0);
  const int64_t b = rp[w], e = rp[w + 1];
  if (e - b > long_row_threshold(K)) return;  // rowsum_long_kernel takes it
  accum_rows<LANES, VEC, true>(acc, b + grp, e, G, ci, v, X, li, ldx);
#pragma unroll
  for (int o = LANES; o < 32; o <<= 1)
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      acc[q].x += __shfl_xor_sync(0xffffffffu, acc[q].x, o);
      acc[q].y += __shfl_xor_sync(0xffffffffu, acc[q].y, o);
    }
  if (grp == 0) {
    double2* out = reinterpret_cast<double2*>(W + w * ldw) + li;
#pragma unroll
    for (int q = 0; q < VEC; ++q) out[q * LANES] = acc[q];
  }
}

// generic k: lanes stride over the row
__global__ void gather_spmm_generic(int64_t s, int k, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                    const double* __restrict__ v, const double* __restrict__ X, double* __restrict__ W) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= s) return;
  const int lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < k; c0 += 32) {
    const int c = c0 + lane;
    double acc = 0.0;
    for (int64_t p = rp[w]; p < rp[w + 1]; ++p)
      if (c < k) acc = fma(v[p], X[(int64_t)ci[p] * k + c], acc);
    if (c < k) W[w * k + c] = acc;
  }
}

// ------------------------------------------------------------------ K3 sparse Gram
// G = E E^T, upper triangle (i <= r: what the SYRK, the Cholesky and copy_diag read), computed
// row by row as G[i, r] = sum over the nonzeros (i, j) of row i, in row order, of v_ij v_rj.
// The s rows of G are cut into NB blocks of B columns; for each touched column J[jj] the table
// off[jj][b] (b = 0..NB) holds the absolute CSC position of its first entry with row >= b B
// (rows ascend inside a CSC column), so the entries of column j that land in blocks [b0, b1) are
// the contiguous range off[jj][b0] .. off[jj][b1].  A task (i, b0, b1) computes G[i, b0 B .. b1 B)
// by one warp: row i's nonzeros are walked 32 at a time, the products v_ij v_rj of the chunk are
// enumerated as one flat list (a warp scan of the range lengths maps flat index -> (nonzero,
// entry)), 32 products per step, and added to G[i, r] leader by leader in lane (= row-nonzero)
// order — every G entry is summed in the same order whatever the task split: deterministic.
// Row i's tasks partition the blocks b >= i / B (the strictly lower blocks are not computed) in
// pieces of about max(GRAM_TASK, 2 nnz_i) products, so a heavy row (a power user, a hub) is
// spread over many warps without partial rows to merge.  Hot columns (more than `hot` entries)
// have an empty range here: their products come from the dense SYRK (sparse_gram).
constexpr int64_t GRAM_TASK = 2048;

// off[jj * (NB + 1) + b] for the touched columns, warp per column (a lane per b, binary search)
__global__ void gram_colblk_kernel(int64_t nJ, const int32_t* __restrict__ J, const int64_t* __restrict__ colptr,
                                   const int32_t* __restrict__ crow, int NB, int64_t B, int64_t hot,
                                   int64_t* __restrict__ off) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nJ) return;
  const int j = J[w];
  const int64_t c0 = colptr[j], c1 = colptr[j + 1];
  const bool is_hot = c1 - c0 > hot;
  for (int b = lane; b <= NB; b += 32) {
    int64_t lo = c0, hi = c1;  // first position with row >= b B
    const int64_t key = (int64_t)b * B;
    if (is_hot) lo = c0;
    else
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)crow[mid] < key) lo = mid + 1;
        else hi = mid;
      }
    off[w * (NB + 1) + b] = lo;
  }
}

// per row: jjp[p] = compact column index of nonzero p; ntask[i] = the number of tasks of row i
__global__ void gram_plan_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const int64_t* __restrict__ jpos, const int64_t* __restrict__ off, int NB, int64_t B,
                                 int32_t* __restrict__ jjp, int64_t* __restrict__ ntask) {
  pdl_begin();
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= s) return;
  const int bi = (int)(i / B);
  int64_t W = 0;
  for (int64_t p = rp[i] + lane; p < rp[i + 1]; p += 32) {
    const int64_t jj = jpos[ci[p]];
    jjp[p] = (int32_t)jj;
    W += off[jj * (NB + 1) + NB] - off[jj * (NB + 1) + bi];
  }
  for (int o = 16; o > 0; o >>= 1) W += __shfl_xor_sync(0xffffffffu, W, o);
  if (lane == 0) {
    const int64_t per = max(GRAM_TASK, 2 * (rp[i + 1] - rp[i]));
    const int64_t nt = (W + per - 1) / per;
    ntask[i] = max((int64_t)1, min(nt, (int64_t)(NB - bi)));
  }
}

__global__ void __launch_bounds__(256) sparse_gram_kernel(int64_t s, const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ jjp,
                                                          const double* __restrict__ v,
                                                          const int64_t* __restrict__ off, int NB, int64_t B,
                                                          const int32_t* __restrict__ crow,
                                                          const double* __restrict__ cval,
                                                          const int64_t* __restrict__ tbase,
                                                          double* __restrict__ G) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  const int64_t ntasks = tbase[s];
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t task = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; task < ntasks; task += nw) {
    int64_t lo = 0, hi = s - 1;  // row: the last i with tbase[i] <= task
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (tbase[mid] <= task) lo = mid;
      else hi = mid - 1;
    }
    const int64_t i = lo;
    const int t = (int)(task - tbase[i]), nt = (int)(tbase[i + 1] - tbase[i]);
    const int bi = (int)(i / B), nbl = NB - bi;
    const int b0 = bi + (int)((int64_t)t * nbl / nt), b1 = bi + (int)((int64_t)(t + 1) * nbl / nt);
    double* acc = G + i * s;
    const int64_t r1 = min(s, (int64_t)b1 * B);
    for (int64_t r = (int64_t)b0 * B + lane; r < r1; r += 32) acc[r] = 0.0;
    __syncwarp();
    const int64_t pe = rp[i + 1];
    for (int64_t p0 = rp[i]; p0 < pe; p0 += 32) {
      const int np = (int)(pe - p0 < 32 ? pe - p0 : 32);
      double vij = 0.0;
      int64_t cb = 0;
      int dg = 0;
      if (lane < np) {
        const int64_t jj = jjp[p0 + lane];
        vij = v[p0 + lane];
        cb = off[jj * (NB + 1) + b0];
        dg = (int)(off[jj * (NB + 1) + b1] - cb);
      }
      int incl = dg;  // inclusive scan of the range lengths over the lanes
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(FULL, incl, 31);
      for (int t0 = 0; t0 < total; t0 += 32) {
        const int tt = t0 + lane;
        const bool live = tt < total;
        int l = 0, h = 31;  // nonzero of flat index tt: the first lane c with incl[c] > tt
#pragma unroll
        for (int it = 0; it < 5; ++it) {
          const int mid = (l + h) >> 1;
          const int im = __shfl_sync(FULL, incl, mid);
          if (im > tt) h = mid;
          else l = mid + 1;
        }
        const int c = l;
        const int ic = __shfl_sync(FULL, incl, c), dc = __shfl_sync(FULL, dg, c);
        const int64_t cbc = __shfl_sync(FULL, cb, c);
        const double vc = __shfl_sync(FULL, vij, c);
        int r = 0;
        double prod = 0.0;
        if (live) {
          const int64_t q = cbc + (tt - (ic - dc));
          r = crow[q];
          prod = vc * cval[q];
        }
        unsigned pending = __ballot_sync(FULL, live);
        while (pending) {
          const unsigned grp = __match_any_sync(FULL, live && ((pending >> lane) & 1) ? r : -1 - lane);
          const bool mine = ((pending >> lane) & 1) && (__ffs(grp & pending) - 1) == lane;
          if (mine) acc[r] += prod;
          pending &= ~__ballot_sync(FULL, mine);
          __syncwarp();
        }
      }
    }
    __syncwarp();
  }
}

// K3 cold part by expand-sort-reduce: every off-diagonal product of a cold column, v_aj v_bj
// for the entry pairs a < b of column j, is written with the key (a, b) in (column, a, b)
// order; a stable radix sort by key groups the products of each G[a, b] in column order, and
// the head of each run of equal keys adds its run in that order.  No dependent global loads
// outside a run, every step a streaming pass over the product list: balanced whatever the row
// and column degrees (hub rows and power users were single-warp latency chains in the row
// walk).  The diagonal G[a, a] (a run as long as row a) is the cold part of the row norm,
// summed by a warp per row (hot_dense_kernel).
// pairs of the cold columns: c (c - 1) / 2, else 0
__global__ void gram_colpairs_kernel(int64_t nJ, const int32_t* __restrict__ J, const int64_t* __restrict__ colptr,
                                     int64_t hot, int64_t* __restrict__ np) {
  pdl_begin();
  const int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (jj < nJ) {
    const int64_t c = colptr[J[jj] + 1] - colptr[J[jj]];
    np[jj] = c > hot ? 0 : c * (c - 1) / 2;
  }
  if (jj == nJ) np[nJ] = 0;
}

// product t of the pair list: its column (the last jj with poff[jj] <= t), then the pair (x, y),
// x < y, of the column's entries in row-major strict-upper order (row x starts at
// x (2c - x - 1) / 2)
template <typename KeyT>
__global__ void gram_expand_kernel(int64_t P, int64_t nJ, const int64_t* __restrict__ poff,
                                   const int32_t* __restrict__ J, const int64_t* __restrict__ colptr,
                                   const int32_t* __restrict__ crow, const double* __restrict__ cval, int64_t s,
                                   KeyT* __restrict__ key, int32_t* __restrict__ perm, double* __restrict__ prod) {
  pdl_begin();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < P; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nJ - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (poff[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    const int64_t c0 = colptr[J[lo]], c = colptr[J[lo] + 1] - c0, u = t - poff[lo];
    const double b2 = 2.0 * (double)c - 1.0;
    int64_t x = (int64_t)((b2 - sqrt(fmax(b2 * b2 - 8.0 * (double)u, 0.0))) * 0.5);
    x = max((int64_t)0, min(x, c - 2));
    while (x > 0 && x * (2 * c - x - 1) / 2 > u) --x;
    while (x + 2 < c && (x + 1) * (2 * c - x - 2) / 2 <= u) ++x;
    const int64_t y = x + 1 + (u - x * (2 * c - x - 1) / 2);
    const int64_t a = crow[c0 + x], b = crow[c0 + y];
    key[t] = (KeyT)(a * s + b);
    perm[t] = (int32_t)t;
    prod[t] = cval[c0 + x] * cval[c0 + y];
  }
}

// run heads of the sorted keys add their run (sorted = column order) into G[a, b]; the run is
// read 8 entries per round trip
template <typename KeyT>
__global__ void gram_reduce_kernel(int64_t P, const KeyT* __restrict__ key, const int32_t* __restrict__ perm,
                                   const double* __restrict__ prod, int64_t s, double* __restrict__ G) {
  pdl_begin();
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < P; k += (int64_t)gridDim.x * blockDim.x) {
    const KeyT kk = key[k];
    if (k > 0 && key[k - 1] == kk) continue;
    double a = 0.0;
    for (int64_t m = k;; m += 8) {
      KeyT kq[8];
      double pq[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) kq[q] = m + q < P ? key[m + q] : (KeyT)(kk + 1);
#pragma unroll
      for (int q = 0; q < 8; ++q) pq[q] = kq[q] == kk ? prod[perm[m + q]] : 0.0;
      bool more = true;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        more = more && kq[q] == kk;
        if (more) a += pq[q];
      }
      if (!more) break;
    }
    const int64_t r = (int64_t)(kk / (KeyT)s), c = (int64_t)(kk % (KeyT)s);
    G[r * s + c] += a;
  }
}

// G's upper triangle (row-major s x s) = 0
__global__ void zero_upper_kernel(int64_t s, double* __restrict__ G) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s) return;
  for (int64_t c = w + lane; c < s; c += 32) G[w * s + c] = 0.0;
}

// ------------------------------------------------------------------ K10 scatter-add
template <int LANES, int VEC>
__global__ void __launch_bounds__(256) scatter_add_kernel(int64_t nJ, const int32_t* __restrict__ J,
                                                          const int64_t* __restrict__ colptr,
                                                          const int32_t* __restrict__ crow,
                                                          const double* __restrict__ cval, const double* __restrict__ Z,
                                                          double* __restrict__ X) {
  pdl_begin();
  constexpr int K = 2 * LANES * VEC;
  constexpr int G = 32 / LANES;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nJ) return;
  const int lane = threadIdx.x & 31, grp = lane / LANES, li = lane % LANES;
  const int j = J[w];
  if (colptr[j + 1] - colptr[j] > long_row_threshold(K)) return;  // rowsum_long_kernel<..., true> takes it
  double2 acc[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) acc[q] = make_double2(0.0, 0.0);
  accum_rows<LANES, VEC, false>(acc, colptr[j] + grp, colptr[j + 1], G, crow, cval, Z, li);
#pragma unroll
  for (int o = LANES; o < 32; o <<= 1)
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      acc[q].x += __shfl_xor_sync(0xffffffffu, acc[q].x, o);
      acc[q].y += __shfl_xor_sync(0xffffffffu, acc[q].y, o);
    }
  if (grp == 0) {
    double2* x = reinterpret_cast<double2*>(X + (int64_t)j * K) + li;
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
      double2 o = x[q * LANES];
      o.x += acc[q].x;
      o.y += acc[q].y;
      x[q * LANES] = o;
    }
  }
}

__global__ void scatter_add_generic(int64_t nJ, int k, const int32_t* __restrict__ J, const int64_t* __restrict__ colptr,
                                    const int32_t* __restrict__ crow, const double* __restrict__ cval,
                                    const double* __restrict__ Z, double* __restrict__ X) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nJ) return;
  const int lane = threadIdx.x & 31;
  const int j = J[w];
  for (int c0 = 0; c0 < k; c0 += 32) {
    const int c = c0 + lane;
    double acc = 0.0;
    for (int64_t p = colptr[j]; p < colptr[j + 1]; ++p)
      if (c < k) acc = fma(cval[p], Z[(int64_t)crow[p] * k + c], acc);
    if (c < k) X[(int64_t)j * k + c] += acc;
  }
}

__global__ void row_sqnorm_kernel(int64_t s, const int64_t* __restrict__ rp, const double* __restrict__ v,
                                  double* __restrict__ out) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= s) return;
  const int lane = threadIdx.x & 31;
  double a = 0.0;
  for (int64_t p = rp[w] + lane; p < rp[w + 1]; p += 32) a = fma(v[p], v[p], a);
  a = warp_sum(a);
  if (lane == 0) out[w] = a;
}

// flag[i] = 1 if row i of A (and of B, when given) is nonempty
__global__ void nonempty_kernel(int64_t s, const int64_t* __restrict__ rpa, const int64_t* __restrict__ rpb,
                                int64_t* __restrict__ flag) {
  pdl_begin();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > s) return;
  if (i == s) { flag[s] = 0; return; }
  bool ne = rpa[i + 1] > rpa[i];
  if (rpb) ne = ne && (rpb[i + 1] > rpb[i]);
  flag[i] = ne ? 1 : 0;
}

// len[pos] = row length of the selected rows (input of the row_ptr scan)
__global__ void sel_len_kernel(int64_t s, const int64_t* __restrict__ rp, const int64_t* __restrict__ flag,
                               const int64_t* __restrict__ pos, int64_t* __restrict__ len, int64_t s_eff) {
  pdl_begin();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < s && flag[i]) len[pos[i]] = rp[i + 1] - rp[i];
  if (i == 0) len[s_eff] = 0;
}

// rows-only selection (no partner side): the kept rows are exactly the nonempty ones, so the
// compacted CSR shares col_idx / val with the input; its row pointers are the input's at the
// kept rows (rpn[pos[i]] = rp[i]) and rpn[s_eff] = nnz
__global__ void sel_rowptr_kernel(int64_t s, const int64_t* __restrict__ rp, const int64_t* __restrict__ flag,
                                  const int64_t* __restrict__ pos, int64_t* __restrict__ rpn, int64_t s_eff) {
  pdl_begin();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < s && flag[i]) rpn[pos[i]] = rp[i];
  if (i == 0) rpn[s_eff] = rp[s];
}

// copy the selected rows (warp per input row)
__global__ void sel_copy_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ v, const int64_t* __restrict__ flag,
                                const int64_t* __restrict__ pos, const int64_t* __restrict__ rpn,
                                int32_t* __restrict__ cin, double* __restrict__ vn) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s || !flag[w]) return;
  const int64_t b = rp[w], o = rpn[pos[w]];
  for (int64_t p = lane; p < rp[w + 1] - b; p += 32) {
    cin[o + p] = ci[b + p];
    vn[o + p] = v[b + p];
  }
}

// dst (s x k) = src rows pos[i] where flag[i], else 0
__global__ void expand_sel_kernel(const double* __restrict__ src, const int64_t* __restrict__ flag,
                                  const int64_t* __restrict__ pos, const int64_t* __restrict__ map,
                                  const double* __restrict__ scl, int64_t s, int k, double* __restrict__ dst) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < s * k; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i, c;
    divmod_idx(e, k, i, c);
    if (map) {  // merged duplicates: the representative's row, scaled by 1 / sqrt(multiplicity)
      const int64_t q = map[i];
      dst[e] = q >= 0 ? scl[i] * src[q * k + c] : 0.0;
    } else {
      dst[e] = flag[i] ? src[pos[i] * k + c] : 0.0;
    }
  }
}

// ---- duplicate update vectors (exact rows / columns updates)
// A group of w identical update vectors e contributes w e^T e to every Gram the update forms,
// which is what one vector sqrt(w) e contributes: the group is replaced by that one vector
// (exact reformulation), and the new factor's rows of the group are the
// representative's row divided by sqrt(w).  Found by a 64-bit content hash, a stable sort by
// hash and an element-wise comparison with the first row of the hash run (a hash collision
// only costs a missed merge).
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__global__ void row_hash_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ v, unsigned long long* __restrict__ key,
                                int32_t* __restrict__ idx) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s) return;
  const int64_t b = rp[w], e = rp[w + 1];
  unsigned long long h = 0;
  for (int64_t p = b + lane; p < e; p += 32)
    h += mix64(((unsigned long long)(unsigned)ci[p] << 32) ^ mix64((unsigned long long)__double_as_longlong(v[p])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if (lane == 0) {
    h = mix64(h ^ (unsigned long long)(e - b));
    key[w] = (e == b) ? ~0ull : (h == ~0ull ? h - 1 : h);
    idx[w] = (int32_t)w;
  }
}
__global__ void dup_group_kernel(int64_t s, const unsigned long long* __restrict__ key, const int32_t* __restrict__ idx,
                                 const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const double* __restrict__ v, int32_t* __restrict__ repr) {
  pdl_begin();
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= s) return;
  const int32_t row = idx[p];
  if (key[p] == ~0ull) {  // empty
    repr[row] = -1;
    return;
  }
  int64_t h = p;
  while (h > 0 && key[h - 1] == key[p]) --h;  // first row of the hash run (smallest index: stable sort)
  const int32_t head = idx[h];
  bool same = head != row && rp[row + 1] - rp[row] == rp[head + 1] - rp[head];
  for (int64_t a = rp[row], b = rp[head]; same && a < rp[row + 1]; ++a, ++b)
    same = ci[a] == ci[b] && v[a] == v[b];
  repr[row] = same ? head : row;
}
__global__ void dup_count_kernel(int64_t s, const int32_t* __restrict__ repr, int* __restrict__ mult,
                                 int64_t* __restrict__ flag) {
  pdl_begin();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > s) return;
  if (i == s) {
    flag[s] = 0;
    return;
  }
  const int32_t r = repr[i];
  flag[i] = (r == i) ? 1 : 0;
  if (r >= 0) atomicAdd(&mult[r], 1);
}
__global__ void dup_map_kernel(int64_t s, const int32_t* __restrict__ repr, const int* __restrict__ mult,
                               const int64_t* __restrict__ pos, int64_t* __restrict__ map, double* __restrict__ scl) {
  pdl_begin();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s) return;
  const int32_t r = repr[i];
  map[i] = r >= 0 ? pos[r] : -1;
  scl[i] = r >= 0 ? rsqrt((double)mult[r]) : 0.0;
}
// copy the representatives' rows, values scaled by sqrt(multiplicity) (warp per input row)
__global__ void dup_copy_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ v, const int64_t* __restrict__ flag,
                                const int64_t* __restrict__ pos, const int* __restrict__ mult,
                                const int64_t* __restrict__ rpn, int32_t* __restrict__ cin, double* __restrict__ vn) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s || !flag[w]) return;
  const double f = sqrt((double)mult[w]);
  const int64_t o = rpn[pos[w]] - rp[w];
  for (int64_t p = rp[w] + lane; p < rp[w + 1]; p += 32) {
    cin[p + o] = ci[p];
    vn[p + o] = f * v[p];
  }
}
}  // namespace

cudaError_t select_nonempty(cudaStream_t st, const DevCSR& A, const DevCSR* B, DevCSR& Aout, DevCSR* Bout,
                            RowSel& sel, Scratch& ws, int64_t* h_scratch) {
  const int64_t s = A.s;
  sel.s = s;
  sel.flag = ws.alloc<int64_t>(s + 1);
  sel.pos = ws.alloc<int64_t>(s + 1);
  if (ws.err) return ws.err;
  ++g_launches;
  launch_k(nonempty_kernel, cdiv(s + 1, 256), 256, 0, st, s, A.row_ptr, B ? B->row_ptr : nullptr, sel.flag);
  cudaError_t e = scan_exclusive(st, sel.flag, sel.pos, s + 1, ws);
  if (e) return e;
  if ((e = cudaMemcpyAsync(h_scratch, sel.pos + s, sizeof(int64_t), cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;
  sel.s_eff = *h_scratch;
  auto one = [&](const DevCSR& X, DevCSR& Y) -> cudaError_t {
    Y = X;
    Y.s = sel.s_eff;
    if (sel.s_eff == s) return cudaSuccess;  // nothing to drop: borrow X
    if (!B) {  // empty rows only: same nonzeros, no copy and no count to read back
      int64_t* rpn = ws.alloc<int64_t>(sel.s_eff + 1);
      if (ws.err) return ws.err;
      g_launches += 1;
      launch_k(sel_rowptr_kernel, cdiv(std::max<int64_t>(s, 1), 256), 256, 0, st, s, X.row_ptr, sel.flag, sel.pos, rpn,
                                                                            sel.s_eff);
      Y.row_ptr = rpn;
      return cudaGetLastError();
    }
    int64_t* len = ws.alloc<int64_t>(sel.s_eff + 1);
    int64_t* rpn = ws.alloc<int64_t>(sel.s_eff + 1);
    if (ws.err) return ws.err;
    g_launches += 1;
    launch_k(sel_len_kernel, cdiv(std::max<int64_t>(s, 1), 256), 256, 0, st, s, X.row_ptr, sel.flag, sel.pos, len, sel.s_eff);
    cudaError_t e2 = scan_exclusive(st, len, rpn, sel.s_eff + 1, ws);
    if (e2) return e2;
    if ((e2 = cudaMemcpyAsync(h_scratch, rpn + sel.s_eff, sizeof(int64_t), cudaMemcpyDeviceToHost, st))) return e2;
    if ((e2 = cudaStreamSynchronize(st))) return e2;
    Y.nnz = *h_scratch;
    int32_t* cin = ws.alloc<int32_t>(std::max<int64_t>(Y.nnz, 1));
    double* vn = ws.alloc<double>(std::max<int64_t>(Y.nnz, 1));
    if (ws.err) return ws.err;
    if (s > 0) {
      g_launches += 1;
      launch_k(sel_copy_kernel, cdiv(s * 32, 256), 256, 0, st, s, X.row_ptr, X.col_idx, X.val, sel.flag, sel.pos, rpn, cin,
                                                        vn);
    }
    Y.row_ptr = rpn;
    Y.col_idx = cin;
    Y.val = vn;
    return cudaGetLastError();
  };
  if ((e = one(A, Aout))) return e;
  if (B && (e = one(*B, *Bout))) return e;
  return cudaSuccess;
}

// ------------------------------------------------------------------ K1's stable counting sort
// LSD radix sort of (key, index) pairs, 8-bit digits, hand-written (no library sort on the path):
// per pass a per-tile digit histogram (tiles of 2048 items, digit-major so that one exclusive
// scan yields every (digit, tile)'s output offset), then a stable scatter in which each warp
// ranks 32 consecutive items at a time with __match_any_sync (peers with the same digit) and
// per-warp digit counters in shared memory.  Input order is preserved among equal keys, so
// the CSC of a row-ordered CSR comes out with rows ascending inside every column — the
// deterministic summation order of K3 / K10 — and duplicate groups keep their first row.
constexpr int RS_THREADS = 256, RS_ITEMS = 8, RS_TILE = RS_THREADS * RS_ITEMS;

template <typename KeyT>
__global__ void __launch_bounds__(RS_THREADS) radix_hist_kernel(int64_t n, const KeyT* __restrict__ keys, int shift,
                                                                int64_t ntiles, int64_t* __restrict__ hist) {
  pdl_begin();
  __shared__ int cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * RS_TILE;
  for (int j = threadIdx.x; j < RS_TILE; j += RS_THREADS) {
    const int64_t i = t0 + j;
    if (i < n) atomicAdd(&cnt[(int)((keys[i] >> shift) & 0xff)], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

template <typename KeyT>
__global__ void __launch_bounds__(RS_THREADS) radix_scatter_kernel(int64_t n, const KeyT* __restrict__ kin,
                                                                   const int32_t* __restrict__ vin, int shift,
                                                                   int64_t ntiles, const int64_t* __restrict__ offs,
                                                                   KeyT* __restrict__ kout, int32_t* __restrict__ vout) {
  pdl_begin();
  __shared__ int wcnt[RS_THREADS / 32][256];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int d = lane; d < 256; d += 32) wcnt[w][d] = 0;
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE + (int64_t)w * (32 * RS_ITEMS);
  KeyT key[RS_ITEMS];
  int32_t val[RS_ITEMS];
  int dig[RS_ITEMS], rank[RS_ITEMS];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int q = 0; q < RS_ITEMS; ++q) {
    const int64_t i = base + 32 * q + lane;
    const bool ok = i < n;
    key[q] = ok ? kin[i] : KeyT(0);
    val[q] = ok ? vin[i] : 0;
    const int d = ok ? (int)((key[q] >> shift) & 0xff) : 256 + lane;  // invalid lanes: unique tags
    dig[q] = d;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    int r = 0;
    if (ok) r = wcnt[w][d] + __popc(peers & lt);
    __syncwarp();
    if (ok && (__ffs(peers) - 1) == lane) wcnt[w][d] += __popc(peers);
    __syncwarp();
    rank[q] = r;
  }
  __syncthreads();
  {  // counts of each digit in the warps before w (the tile is in warp order)
    const int d = tid;
    int run = 0;
#pragma unroll
    for (int ww = 0; ww < RS_THREADS / 32; ++ww) {
      const int c = wcnt[ww][d];
      wcnt[ww][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < RS_ITEMS; ++q) {
    const int64_t i = base + 32 * q + lane;
    if (i >= n) continue;
    const int d = dig[q];
    const int64_t pos = offs[(int64_t)d * ntiles + blockIdx.x] + wcnt[w][d] + rank[q];
    kout[pos] = key[q];
    vout[pos] = val[q];
  }
}

__global__ void iota_kernel(int64_t n, int32_t* __restrict__ v) {
  pdl_begin();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

// stable sort of (key, val) by the bits [0, end_bit) of key; the result is in (k0, v0) or
// (k1, v1) as *which says (0 / 1)
template <typename KeyT>
cudaError_t radix_sort_pairs(cudaStream_t st, int64_t n, KeyT* k0, int32_t* v0, KeyT* k1, int32_t* v1, int end_bit,
                             int* which, Scratch& ws) {
  *which = 0;
  if (n <= 1) return cudaSuccess;
  const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
  int64_t* hist = ws.alloc<int64_t>((size_t)256 * ntiles + 1);
  int64_t* offs = ws.alloc<int64_t>((size_t)256 * ntiles + 1);
  if (ws.err) return ws.err;
  cudaError_t e;
  KeyT* ka = k0;
  KeyT* kb = k1;
  int32_t* va = v0;
  int32_t* vb = v1;
  for (int shift = 0; shift < end_bit; shift += 8) {
    g_launches += 2;
    launch_k(radix_hist_kernel<KeyT>, (unsigned)ntiles, RS_THREADS, 0, st, n, ka, shift, ntiles, hist);
    if ((e = cudaMemsetAsync(hist + (size_t)256 * ntiles, 0, sizeof(int64_t), st))) return e;
    if ((e = scan_exclusive(st, hist, offs, (int64_t)256 * ntiles + 1, ws))) return e;
    launch_k(radix_scatter_kernel<KeyT>, (unsigned)ntiles, RS_THREADS, 0, st, n, ka, va, shift, ntiles, offs, kb, vb);
    std::swap(ka, kb);
    std::swap(va, vb);
    *which ^= 1;
  }
  return cudaGetLastError();
}

cudaError_t select_unique(cudaStream_t st, const DevCSR& A, DevCSR& Aout, RowSel& sel, Scratch& ws,
                          int64_t* h_scratch) {
  const int64_t s = A.s;
  sel.s = s;
  sel.flag = ws.alloc<int64_t>(s + 1);
  sel.pos = ws.alloc<int64_t>(s + 1);
  unsigned long long* key = ws.alloc<unsigned long long>(s);
  unsigned long long* key2 = ws.alloc<unsigned long long>(s);
  int32_t* idx = ws.alloc<int32_t>(s);
  int32_t* idx2 = ws.alloc<int32_t>(s);
  int32_t* repr = ws.alloc<int32_t>(s);
  int* mult = ws.alloc<int>(s);
  sel.map = ws.alloc<int64_t>(s);
  sel.scl = ws.alloc<double>(s);
  if (ws.err) return ws.err;
  cudaError_t e;
  if ((e = cudaMemsetAsync(mult, 0, s * sizeof(int), st))) return e;
  g_launches += 4;
  launch_k(row_hash_kernel, cdiv(s * 32, 256), 256, 0, st, s, A.row_ptr, A.col_idx, A.val, key, idx);
  int which = 0;
  if ((e = radix_sort_pairs<unsigned long long>(st, s, key, idx, key2, idx2, 64, &which, ws))) return e;
  if (which == 0) {  // (an even pass count leaves the result in the input buffers)
    std::swap(key, key2);
    std::swap(idx, idx2);
  }
  launch_k(dup_group_kernel, cdiv(s, 256), 256, 0, st, s, key2, idx2, A.row_ptr, A.col_idx, A.val, repr);
  launch_k(dup_count_kernel, cdiv(s + 1, 256), 256, 0, st, s, repr, mult, sel.flag);
  if ((e = scan_exclusive(st, sel.flag, sel.pos, s + 1, ws))) return e;
  ++g_launches;
  launch_k(dup_map_kernel, cdiv(s, 256), 256, 0, st, s, repr, mult, sel.pos, sel.map, sel.scl);
  if ((e = cudaMemcpyAsync(h_scratch, sel.pos + s, sizeof(int64_t), cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;
  sel.s_eff = *h_scratch;
  Aout = A;
  Aout.s = sel.s_eff;
  if (sel.s_eff == s) {  // nothing empty, nothing merged: borrow A
    sel.map = nullptr;
    return cudaSuccess;
  }
  int64_t* len = ws.alloc<int64_t>(sel.s_eff + 1);
  int64_t* rpn = ws.alloc<int64_t>(sel.s_eff + 1);
  if (ws.err) return ws.err;
  ++g_launches;
  launch_k(sel_len_kernel, cdiv(std::max<int64_t>(s, 1), 256), 256, 0, st, s, A.row_ptr, sel.flag, sel.pos, len, sel.s_eff);
  if ((e = scan_exclusive(st, len, rpn, sel.s_eff + 1, ws))) return e;
  if ((e = cudaMemcpyAsync(h_scratch, rpn + sel.s_eff, sizeof(int64_t), cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;
  Aout.nnz = *h_scratch;
  int32_t* cin = ws.alloc<int32_t>(std::max<int64_t>(Aout.nnz, 1));
  double* vn = ws.alloc<double>(std::max<int64_t>(Aout.nnz, 1));
  if (ws.err) return ws.err;
  ++g_launches;
  launch_k(dup_copy_kernel, cdiv(s * 32, 256), 256, 0, st, s, A.row_ptr, A.col_idx, A.val, sel.flag, sel.pos, mult, rpn, cin,
                                                     vn);
  Aout.row_ptr = rpn;
  Aout.col_idx = cin;
  Aout.val = vn;
  return cudaGetLastError();
}

// One empty update vector appended to E (row pointer s + 2 long, the last repeating nnz).
// The exact path pads an odd s this way: its Gram row and column are zero, so the pivot is
// deflated ((E E^T)_ii = 0, R8) and changes nothing, while every s x s operand gets
// an even leading dimension (16-byte rows: the cp.async / double2 paths of the tile DAG).
cudaError_t pad_even_rows(cudaStream_t st, DevCSR& E, Scratch& ws) {
  if ((E.s & 1) == 0) return cudaSuccess;
  int64_t* rp = ws.alloc<int64_t>(E.s + 2);
  if (ws.err) return ws.err;
  cudaError_t e;
  if ((e = cudaMemcpyAsync(rp, E.row_ptr, (size_t)(E.s + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st))) return e;
  if ((e = cudaMemcpyAsync(rp + E.s + 1, E.row_ptr + E.s, sizeof(int64_t), cudaMemcpyDeviceToDevice, st))) return e;
  E.row_ptr = rp;
  E.s += 1;
  return cudaSuccess;
}

cudaError_t expand_selected(cudaStream_t st, const RowSel& sel, const double* src, int k, double* dst) {
  if (sel.s * k == 0) return cudaSuccess;
  ++g_launches;
  launch_k(expand_sel_kernel, (unsigned)std::min<int64_t>(cdiv(sel.s * k, 256), 148 * 16), 256, 0, st, 
      src, sel.flag, sel.pos, sel.map, sel.scl, sel.s, k, dst);
  return cudaGetLastError();
}

cudaError_t scan_exclusive_i64(cudaStream_t st, const int64_t* in, int64_t* out, int64_t n, Scratch& ws) {
  return scan_exclusive(st, in, out, n, ws);
}

cudaError_t validate_csr(cudaStream_t st, const DevCSR& E, int* d_flag) {
  if (E.s == 0) return cudaSuccess;
  g_launches += E.nnz ? 2 : 1;
  launch_k(validate_rows_kernel, (unsigned)std::min<int64_t>(cdiv(E.s, 256), 148 * 8), 256, 0, st, E.s, E.nnz,
           E.row_ptr, d_flag);
  if (E.nnz)
    launch_k(validate_kernel, (unsigned)std::min<int64_t>(cdiv(E.nnz, 256), 148 * 16), 256, 0, st, E.s, E.dim, E.nnz,
             E.row_ptr, E.col_idx, E.val, d_flag);
  return cudaGetLastError();
}

cudaError_t build_csc(cudaStream_t st, const DevCSR& E, DevCSC& out, Scratch& ws, int64_t* h_nJ) {
  const int64_t dim = E.dim, nnz = E.nnz;
  int64_t* cnt = ws.alloc<int64_t>(dim + 1);
  out.colptr = ws.alloc<int64_t>(dim + 1);
  int64_t* flag = ws.alloc<int64_t>(dim + 1);
  int64_t* pos = ws.alloc<int64_t>(dim + 1);
  out.row = ws.alloc<int32_t>(nnz);
  out.val = ws.alloc<double>(nnz);
  if (ws.err) return ws.err;
  cudaError_t e;
  if ((e = cudaMemsetAsync(cnt, 0, (dim + 1) * sizeof(int64_t), st))) return e;
  if (nnz > 0) {
    const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(nnz, 256), 148 * 16);
    ++g_launches;
    launch_k(col_hist_kernel, blocks, 256, 0, st, nnz, E.col_idx, reinterpret_cast<unsigned long long*>(cnt));
  }
  if ((e = scan_exclusive(st, cnt, out.colptr, dim + 1, ws))) return e;
  ++g_launches;
  launch_k(touched_flag_kernel, cdiv(dim + 1, 256), 256, 0, st, dim, cnt, flag);
  if ((e = cudaMemsetAsync(flag + dim, 0, sizeof(int64_t), st))) return e;
  if ((e = scan_exclusive(st, flag, pos, dim + 1, ws))) return e;
  // |J| = pos[dim]
  if ((e = cudaMemcpyAsync(h_nJ, pos + dim, sizeof(int64_t), cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;
  out.nJ = *h_nJ;
  out.jpos = pos;
  out.J = ws.alloc<int32_t>(out.nJ);
  if (ws.err) return ws.err;
  ++g_launches;
  launch_k(compact_J_kernel, cdiv(dim, 256), 256, 0, st, dim, cnt, pos, out.J);
  if (nnz > 0) {
    const Scratch::Mark sort_mark = ws.mark();  // the sort's keys and temporary storage are
    struct Rew {                                // returned once the CSC is unpacked
      Scratch& w;
      Scratch::Mark mk;
      ~Rew() { w.rewind(mk); }
    } rew{ws, sort_mark};
    // stable counting sort of the entries by column (input order: rows ascending), then the
    // rows and values gathered through the permutation
    uint32_t* kin = ws.alloc<uint32_t>(nnz);
    uint32_t* kout = ws.alloc<uint32_t>(nnz);
    int32_t* pin = ws.alloc<int32_t>(nnz);
    int32_t* pout = ws.alloc<int32_t>(nnz);
    int32_t* rowof = ws.alloc<int32_t>(nnz);
    if (ws.err) return ws.err;
    int end_bit = 8;
    while (end_bit < 32 && (1ll << end_bit) < dim) end_bit += 8;
    const unsigned gb = (unsigned)std::min<int64_t>(cdiv(nnz, 256), 148 * 8);
    g_launches += 2;
    launch_k(csc_rows_kernel, cdiv(E.s * 32, 256), 256, 0, st, E.s, E.row_ptr, E.col_idx, kin, rowof);
    launch_k(iota_kernel, gb, 256, 0, st, nnz, pin);
    int which = 0;
    if ((e = radix_sort_pairs<uint32_t>(st, nnz, kin, pin, kout, pout, end_bit, &which, ws))) return e;
    ++g_launches;
    launch_k(csc_gather_kernel, gb, 256, 0, st, nnz, which ? pout : pin, rowof, E.val, out.row, out.val);
  }
  return cudaGetLastError();
}

// The long-row work list of a CSR (rowid = null) or CSC-over-J (rowid = J) row set: rows above
// kLongRow nonzeros, rows above kChunk cut into chunks (LongPlan).  Small sets (nnz below 2^20)
// skip the chunking (items = null: one CTA per long row, as before).
cudaError_t long_plan(cudaStream_t st, int64_t n, const int32_t* rowid, const int64_t* ptr, int64_t nnz, int K,
                      int Kthr, LongPlan& lp, Scratch& ws) {
  lp.list = ws.alloc<int32_t>(n + 1);
  if (ws.err) return ws.err;
  lp.cnt = reinterpret_cast<int*>(lp.list + n);
  cudaError_t e;
  if ((e = cudaMemsetAsync(lp.cnt, 0, sizeof(int), st))) return e;
  ++g_launches;
  launch_k(long_list_kernel, cdiv(n, 256), 256, 0, st, n, rowid, ptr, lp.list, lp.cnt, long_row_threshold(Kthr));
  if (nnz < ((int64_t)1 << 20)) return cudaSuccess;
  lp.nch = ws.alloc<int64_t>(n + 1);
  int64_t* nch2 = ws.alloc<int64_t>(n + 1);
  lp.base = ws.alloc<int64_t>(n + 1);
  lp.base2 = ws.alloc<int64_t>(n + 1);
  lp.max_items = n + nnz / kChunk + 1;
  lp.items = ws.alloc<int2>(lp.max_items);
  lp.part = ws.alloc<double>((size_t)(2 * (nnz / kChunk) + 16) * K);
  if (ws.err) return ws.err;
  g_launches += 2;
  launch_k(long_nch_kernel, cdiv(n + 1, 256), 256, 0, st, n, lp.list, lp.cnt, rowid, ptr, lp.nch, nch2);
  if ((e = scan_exclusive(st, lp.nch, lp.base, n + 1, ws))) return e;
  if ((e = scan_exclusive(st, nch2, lp.base2, n + 1, ws))) return e;
  launch_k(long_items_kernel, cdiv(n, 256), 256, 0, st, n, lp.cnt, lp.nch, lp.base, lp.items);
  return cudaGetLastError();
}

// W (s x width, leading dimension ldw) = E X (X: dim x width, leading dimension ldx), width a sum
// of the fast widths: panels of 256 / 128 / 64 / 32 / 16 columns (e.g. the 288-wide randomized
// range finder of k = 256)
cudaError_t gather_spmm_ld(cudaStream_t st, const DevCSR& E, const double* X, int64_t ldx, int width, double* W,
                           int64_t ldw) {
  if (E.s == 0 || width == 0) return cudaSuccess;
  if (width % 16) return cudaErrorInvalidValue;
  Scratch ws(st);
  const unsigned grid = cdiv(E.s * 32, 256);
  LongPlan lp;
  int plan_thr = -1;
  for (int c0 = 0; c0 < width;) {
    const int rest = width - c0;
    const int pw = rest >= 256 ? 256 : rest >= 128 ? 128 : rest >= 64 ? 64 : rest >= 32 ? 32 : 16;
    if (long_row_threshold(pw) != plan_thr) {  // the long-row list of this panel width
      lp = LongPlan();
      cudaError_t e0 = long_plan(st, E.s, nullptr, E.row_ptr, E.nnz, 256, pw, lp, ws);
      if (e0) return e0;
      plan_thr = long_row_threshold(pw);
    }
    const double* Xp = X + c0;
    double* Wp = W + c0;
    g_launches += lp.items ? 3 : 2;
    switch (pw) {
#define GSL(L, V)                                                                                                     \
  launch_k(gather_spmm_kernel<L, V>, grid, 256, 0, st, E.s, E.row_ptr, E.col_idx, E.val, Xp, Wp, ldx, ldw);          \
  launch_k(rowsum_long_kernel<L, V, false>, 296, 32 * LongCfg<L, V>::WARPS, 0, st, lp.list, lp.cnt, nullptr, E.row_ptr, \
           E.col_idx, E.val, Xp, Wp, ldx, ldw, lp.items, lp.nch, lp.base, lp.base2, lp.part);                          \
  break;
      case 16: GSL(8, 1)
      case 32: GSL(16, 1)
      case 64: GSL(32, 1)
      case 128: GSL(32, 2)
      default: GSL(32, 4)
#undef GSL
    }
    if (lp.items)
      launch_k(chunk_reduce_kernel<false>, 148, 256, 0, st, lp.list, lp.cnt, nullptr, lp.nch, lp.base2, lp.part, pw, Wp,
               ldw);
    c0 += pw;
  }
  return cudaGetLastError();
}

cudaError_t gather_spmm(cudaStream_t st, const DevCSR& E, const double* X, int k, double* W) {
  if (E.s == 0) return cudaSuccess;
  if (k == 16 || k == 32 || k == 64 || k == 128 || k == 256) return gather_spmm_ld(st, E, X, k, k, W, k);
  const unsigned grid = cdiv(E.s * 32, 256);
  ++g_launches;
  launch_k(gather_spmm_generic, grid, 256, 0, st, E.s, k, E.row_ptr, E.col_idx, E.val, X, W);
  return cudaGetLastError();
}

namespace {
// the scalar products of the upper triangle of the sparse Gram: sum over the touched columns
// of c_j (c_j + 1) / 2 — the algorithmic flops (2 per product) of the profiling pass's accounting
__global__ void gram_products_kernel(int64_t nJ, const int32_t* __restrict__ J, const int64_t* __restrict__ colptr,
                                     unsigned long long* total) {
  const int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long a = 0;
  if (jj < nJ) {
    const unsigned long long c = (unsigned long long)(colptr[J[jj] + 1] - colptr[J[jj]]);
    a = c * (c + 1) / 2;
  }
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0 && a) atomicAdd(total, a);
}

// hot/cold split candidates: for T = kHotT[t] (the last slot: tf, a forced threshold), the
// number of columns with more than T entries and the strict-upper products c (c - 1) / 2 of
// the others (the pair-list length; integer sums: order-free)
constexpr int kNT = 10;
__constant__ int64_t kHotT[kNT - 1] = {16, 32, 64, 128, 256, 512, 1024, 4096, INT64_MAX};
__global__ void gram_cost_kernel(int64_t nJ, const int32_t* __restrict__ J, const int64_t* __restrict__ colptr,
                                 int64_t tf, unsigned long long* __restrict__ out) {
  pdl_begin();
  unsigned long long hc[kNT], pc[kNT];
#pragma unroll
  for (int t = 0; t < kNT; ++t) hc[t] = pc[t] = 0;
  for (int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; jj < nJ; jj += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = colptr[J[jj] + 1] - colptr[J[jj]];
#pragma unroll
    for (int t = 0; t < kNT; ++t) {
      if (c > (t < kNT - 1 ? kHotT[t] : tf)) ++hc[t];
      else pc[t] += (unsigned long long)(c * (c - 1) / 2);
    }
  }
#pragma unroll
  for (int t = 0; t < kNT; ++t)
    for (int o = 16; o > 0; o >>= 1) {
      hc[t] += __shfl_xor_sync(0xffffffffu, hc[t], o);
      pc[t] += __shfl_xor_sync(0xffffffffu, pc[t], o);
    }
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int t = 0; t < kNT; ++t) {
      if (hc[t]) atomicAdd(&out[t], hc[t]);
      if (pc[t]) atomicAdd(&out[kNT + t], pc[t]);
    }
}

__global__ void hot_flag_kernel(int64_t nJ, const int32_t* __restrict__ J, const int64_t* __restrict__ colptr,
                                int64_t hot, int64_t* __restrict__ flag) {
  pdl_begin();
  const int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (jj < nJ) flag[jj] = (colptr[J[jj] + 1] - colptr[J[jj]] > hot) ? 1 : 0;
  if (jj == nJ) flag[nJ] = 0;
}
// D[i, hidx(j)] = v_ij for the nonzeros of the hot columns (D zeroed, s x h row-major; D may be
// null when there are none) and dcold[i] = the squares of row i's entries in the cold columns
// (the diagonal of their Gram; warp per row, fixed tree)
__global__ void hot_dense_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const double* __restrict__ v, const int64_t* __restrict__ jpos,
                                 const int64_t* __restrict__ hpos, const int64_t* __restrict__ colptr, int64_t hot,
                                 int64_t h, double* __restrict__ D, double* __restrict__ dcold) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s) return;
  double a = 0.0;
  for (int64_t p = rp[w] + lane; p < rp[w + 1]; p += 32) {
    const int j = ci[p];
    if (colptr[j + 1] - colptr[j] > hot) D[w * h + hpos[jpos[j]]] = v[p];
    else a = fma(v[p], v[p], a);
  }
  a = warp_sum(a);
  if (lane == 0) dcold[w] = a;
}

__global__ void diag_add_kernel(int64_t s, const double* __restrict__ d, double* __restrict__ G) {
  pdl_begin();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < s) G[i * s + i] += d[i];
}
}  // namespace

double sparse_gram_products(cudaStream_t st, const DevCSR& E, const DevCSC& C) {
  if (E.s == 0 || C.nJ == 0) return 0.0;
  unsigned long long* d = nullptr;
  unsigned long long h = 0;
  if (cudaMallocAsync(&d, sizeof(unsigned long long), st) != cudaSuccess) return 0.0;
  cudaMemsetAsync(d, 0, sizeof(unsigned long long), st);
  gram_products_kernel<<<(unsigned)cdiv(C.nJ, 256), 256, 0, st>>>(C.nJ, C.J, C.colptr, d);
  cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  cudaStreamSynchronize(st);
  return (double)h;
}

template <typename KeyT>
cudaError_t gram_esc(cudaStream_t st, const DevCSC& C, int64_t s, int64_t hot, int64_t P, double* G, Scratch& ws) {
  int64_t* np = ws.alloc<int64_t>(C.nJ + 1);
  int64_t* poff = ws.alloc<int64_t>(C.nJ + 1);
  KeyT* k0 = ws.alloc<KeyT>(P);
  KeyT* k1 = ws.alloc<KeyT>(P);
  int32_t* p0 = ws.alloc<int32_t>(P);
  int32_t* p1 = ws.alloc<int32_t>(P);
  double* prod = ws.alloc<double>(P);
  if (ws.err) return ws.err;
  cudaError_t e;
  g_launches += 3;
  launch_k(gram_colpairs_kernel, cdiv(C.nJ + 1, 256), 256, 0, st, C.nJ, C.J, C.colptr, hot, np);
  if ((e = scan_exclusive(st, np, poff, C.nJ + 1, ws))) return e;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(P, 256), 148 * 16);
  launch_k(gram_expand_kernel<KeyT>, grid, 256, 0, st, P, C.nJ, poff, C.J, C.colptr, C.row, C.val, s, k0, p0, prod);
  int end_bit = 8;
  while (end_bit < (int)(8 * sizeof(KeyT)) && ((unsigned long long)s * s - 1) >> end_bit) end_bit += 8;
  int which = 0;
  if ((e = radix_sort_pairs<KeyT>(st, P, k0, p0, k1, p1, end_bit, &which, ws))) return e;
  launch_k(gram_reduce_kernel<KeyT>, grid, 256, 0, st, P, which ? k1 : k0, which ? p1 : p0, prod, s, G);
  return cudaGetLastError();
}

// K3: the hot columns (Zipf-popular items, graph hubs: a few hundred columns that carry most
// of sum_j c_j^2) as a dense s x h block whose SYRK D D^T the DMMA GEMM writes to the upper
// triangle (beta = 0: no separate zero fill); the products of the cold columns then added by
// expand-sort-reduce (gram_esc).  The threshold is the candidate of least modelled time
// cold products / rate_cold + s^2 h / rate_syrk from one pass over the column counts (one
// host synchronisation, which also sizes the product list).  Above kEscCap cold products the
// row-walk kernel (sparse_gram_cold) takes the cold part, before the SYRK adds (beta = 1).
cudaError_t sparse_gram(cudaStream_t st, const DevCSR& E, const DevCSC& C, double* G, Scratch& ws) {
  const int64_t s = E.s;
  if (s == 0) return cudaSuccess;
  // tuning knobs: TSVD_GRAM_HOT > 0 forces the threshold, < 0 turns the dense part off;
  // TSVD_GRAM_ESC=0 uses the row walk for the cold part
  static const int64_t hot_env = getenv("TSVD_GRAM_HOT") ? atoll(getenv("TSVD_GRAM_HOT")) : 0;
  static const bool esc_on = !(getenv("TSVD_GRAM_ESC") && atoi(getenv("TSVD_GRAM_ESC")) == 0);
  static const double rate_cold = getenv("TSVD_GRAM_COLD_RATE") ? atof(getenv("TSVD_GRAM_COLD_RATE")) : 2.0e10;
  static const double rate_syrk = getenv("TSVD_GRAM_SYRK_RATE") ? atof(getenv("TSVD_GRAM_SYRK_RATE")) : 2.5e13;
  constexpr int64_t kEscCap = (int64_t)1 << 25;
  cudaError_t e;
  const unsigned zgrid = (unsigned)cdiv(s * 32, 256);
  if (C.nJ == 0) {
    ++g_launches;
    launch_k(zero_upper_kernel, zgrid, 256, 0, st, s, G);
    return cudaGetLastError();
  }
  static thread_local unsigned long long* h_cost = nullptr;
  if (!h_cost && cudaMallocHost(&h_cost, 2 * kNT * sizeof(unsigned long long)) != cudaSuccess)
    return cudaErrorMemoryAllocation;
  unsigned long long* d_cost = ws.alloc<unsigned long long>(2 * kNT);
  if (ws.err) return ws.err;
  if ((e = cudaMemsetAsync(d_cost, 0, 2 * kNT * sizeof(unsigned long long), st))) return e;
  ++g_launches;
  launch_k(gram_cost_kernel, (unsigned)std::min<int64_t>(cdiv(C.nJ, 256), 148 * 4), 256, 0, st, C.nJ, C.J, C.colptr,
           hot_env > 0 ? hot_env : INT64_MAX, d_cost);
  if ((e = cudaMemcpyAsync(h_cost, d_cost, 2 * kNT * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;
  static const int64_t T[kNT] = {16, 32, 64, 128, 256, 512, 1024, 4096, INT64_MAX, INT64_MAX};
  int tb = kNT - 2;  // all cold
  if (hot_env > 0) {
    tb = kNT - 1;
  } else if (hot_env == 0) {
    double best = 1e300;
    for (int t = 0; t < kNT - 1; ++t) {
      const double H = (double)h_cost[t], Pc = (double)h_cost[kNT + t];
      if (esc_on && Pc > (double)kEscCap && t != kNT - 2) continue;
      const double cost = Pc / rate_cold + (H > 0 ? (double)s * s * H / rate_syrk + 2e-5 : 0.0);
      if (cost < best) {
        best = cost;
        tb = t;
      }
    }
  }
  const int64_t hot = hot_env > 0 ? hot_env : T[tb];
  const int64_t h = (int64_t)h_cost[tb], P = (int64_t)h_cost[kNT + tb];
  const bool esc = esc_on && P <= kEscCap;
  double* D = nullptr;
  int64_t* hpos = nullptr;
  double* dcold = ws.alloc<double>(s);
  if (h > 0) {
    int64_t* hflag = ws.alloc<int64_t>(C.nJ + 1);
    hpos = ws.alloc<int64_t>(C.nJ + 1);
    D = ws.alloc<double>((size_t)s * h);
    if (ws.err) return ws.err;
    ++g_launches;
    launch_k(hot_flag_kernel, cdiv(C.nJ + 1, 256), 256, 0, st, C.nJ, C.J, C.colptr, hot, hflag);
    if ((e = scan_exclusive(st, hflag, hpos, C.nJ + 1, ws))) return e;
    if ((e = cudaMemsetAsync(D, 0, (size_t)s * h * sizeof(double), st))) return e;
  }
  if (ws.err) return ws.err;
  if (h > 0 || esc) {
    ++g_launches;
    launch_k(hot_dense_kernel, zgrid, 256, 0, st, s, E.row_ptr, E.col_idx, E.val, C.jpos, hpos, C.colptr,
             h > 0 ? hot : INT64_MAX, h, D, dcold);
  }
  if (!esc) {  // row walk (writes its ranges), then the SYRK adds
    if ((e = sparse_gram_cold(st, E, C, G, ws, h > 0 ? hot : INT64_MAX))) return e;
    return h > 0 ? dgemm(st, s, s, h, 1.0, CMat{D, h, 1}, CMat{D, 1, h}, 1.0, Mat{G, s, 1}, 1) : cudaSuccess;
  }
  if (h > 0) {
    if ((e = dgemm(st, s, s, h, 1.0, CMat{D, h, 1}, CMat{D, 1, h}, 0.0, Mat{G, s, 1}, 1))) return e;
  } else {
    ++g_launches;
    launch_k(zero_upper_kernel, zgrid, 256, 0, st, s, G);
  }
  ++g_launches;
  launch_k(diag_add_kernel, cdiv(s, 256), 256, 0, st, s, dcold, G);
  if (P == 0) return cudaGetLastError();
  if ((unsigned long long)s * s <= 0xffffffffull) return gram_esc<uint32_t>(st, C, s, hot, P, G, ws);
  return gram_esc<unsigned long long>(st, C, s, hot, P, G, ws);
}

cudaError_t sparse_gram_cold(cudaStream_t st, const DevCSR& E, const DevCSC& C, double* G, Scratch& ws, int64_t hot) {
  const int64_t s = E.s;
  if (s == 0) return cudaSuccess;
  // row blocks of G: about 128 columns each, at most 64, the table within 64 MB
  int64_t NB = std::min<int64_t>(64, cdiv(s, 128));
  if (C.nJ > 0) NB = std::max<int64_t>(1, std::min<int64_t>(NB, ((int64_t)8 << 20) / C.nJ - 1));
  const int64_t B = cdiv(s, NB);
  int64_t* off = ws.alloc<int64_t>((size_t)std::max<int64_t>(C.nJ, 1) * (NB + 1));
  int32_t* jjp = ws.alloc<int32_t>(std::max<int64_t>(E.nnz, 1));
  int64_t* ntask = ws.alloc<int64_t>(s + 1);
  int64_t* tbase = ws.alloc<int64_t>(s + 1);
  if (ws.err) return ws.err;
  cudaError_t e;
  if ((e = cudaMemsetAsync(ntask + s, 0, sizeof(int64_t), st))) return e;
  g_launches += 3;
  if (C.nJ > 0)
    launch_k(gram_colblk_kernel, cdiv(C.nJ * 32, 256), 256, 0, st, C.nJ, C.J, C.colptr, C.row, (int)NB, B, hot, off);
  else
    --g_launches;
  launch_k(gram_plan_kernel, cdiv(s * 32, 256), 256, 0, st, s, E.row_ptr, E.col_idx, C.jpos, off, (int)NB, B, jjp,
           ntask);
  if ((e = scan_exclusive(st, ntask, tbase, s + 1, ws))) return e;
  static const int gram_grid = getenv("TSVD_GRAM_GRID") ? atoi(getenv("TSVD_GRAM_GRID")) : 148 * 8;  // tuning
  launch_k(sparse_gram_kernel, gram_grid, 256, 0, st, s, E.row_ptr, jjp, E.val, off, (int)NB, B, C.row, C.val, tbase, G);
  return cudaGetLastError();
}

cudaError_t scatter_add(cudaStream_t st, const DevCSC& C, int64_t nnz, const double* Z, int k, double* X) {
  if (C.nJ == 0) return cudaSuccess;
  const unsigned grid = cdiv(C.nJ * 32, 256);
  const bool fast = k == 16 || k == 32 || k == 64 || k == 128 || k == 256;
  if (!fast) {
    ++g_launches;
    launch_k(scatter_add_generic, grid, 256, 0, st, C.nJ, k, C.J, C.colptr, C.row, C.val, Z, X);
    return cudaGetLastError();
  }
  Scratch ws(st);
  LongPlan lp;
  cudaError_t e0 = long_plan(st, C.nJ, C.J, C.colptr, nnz, k, k, lp, ws);
  if (e0) return e0;
  g_launches += lp.items ? 3 : 2;
#define SS(L, V)                                                                                                      \
  launch_k(scatter_add_kernel<L, V>, grid, 256, 0, st, C.nJ, C.J, C.colptr, C.row, C.val, Z, X);                      \
  launch_k(rowsum_long_kernel<L, V, true>, 296, 32 * LongCfg<L, V>::WARPS, 0, st, lp.list, lp.cnt, C.J, C.colptr, C.row, \
           C.val, Z, X, (int64_t)(2 * L * V), (int64_t)(2 * L * V), lp.items, lp.nch, lp.base, lp.base2, lp.part);       \
  break;
  switch (k) {
    case 16: SS(8, 1)
    case 32: SS(16, 1)
    case 64: SS(32, 1)
    case 128: SS(32, 2)
    default: SS(32, 4)
  }
#undef SS
  if (lp.items)
    launch_k(chunk_reduce_kernel<true>, 148, 256, 0, st, lp.list, lp.cnt, C.J, lp.nch, lp.base2, lp.part, k, X,
             (int64_t)k);
  return cudaGetLastError();
}

cudaError_t row_sqnorms(cudaStream_t st, const DevCSR& E, double* out) {
  if (E.s == 0) return cudaSuccess;
  ++g_launches;
  launch_k(row_sqnorm_kernel, cdiv(E.s * 32, 256), 256, 0, st, E.s, E.row_ptr, E.val, out);
  return cudaGetLastError();
}

}  // namespace tsvd
