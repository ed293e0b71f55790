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
__global__ void validate_kernel(int64_t s, int64_t dim, int64_t nnz, const int64_t* __restrict__ rp,
                                const int32_t* __restrict__ ci, const double* __restrict__ v, int* flag) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s) return;
  int64_t b = rp[w], e = rp[w + 1];
  int bad = 0;
  // the row_ptr endpoints are checked on the host after this kernel: stay inside [0, nnz)
  if (b < 0 || e > nnz) {
    bad |= 1;
    b = e = 0;
  }
  if (e < b) bad |= 1;
  for (int64_t p = b + lane; p < e; p += 32) {
    int c = ci[p];
    if (c < 0 || c >= dim) bad |= 1;
    if (p > b && ci[p - 1] >= c) bad |= 1;
    double x = v[p];
    if (!isfinite(x)) bad |= 2;
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (lane == 0 && bad) atomicOr(flag, bad);
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
// Warp per output row i of G = E E^T.  The products v_ij v_i'j of row i are enumerated in
// (column p of row i, entry q of CSC column j) order as one flat list, 32 at a time: a chunk of
// 32 nnz of the row loads its (j, v, column extent) in parallel, a warp scan of the column
// degrees maps flat index -> (column, entry) by binary search over the lanes, and each lane
// loads its entry (one memory latency per 32 products instead of three per nnz of the row —
// hub rows of thousands of nnz were latency bound).  Products hitting the same acc[i'] inside
// a batch are added leader by leader in lane (= flat) order, so every acc[i'] sums in the
// same (p, q) order as a sequential walk: deterministic, independent of the batching.
// acc[i'] += the flat products [F0, F1) of row i, the walk starting at nnz pstart whose first
// product has flat index fbase
__device__ __forceinline__ void gram_range(int64_t pstart, int64_t pe, int64_t fbase, int64_t F0, int64_t F1,
                                           const int32_t* __restrict__ ci, const double* __restrict__ v,
                                           const int64_t* __restrict__ colptr, const int32_t* __restrict__ crow,
                                           const double* __restrict__ cval, double* acc, int64_t hot) {
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  int64_t fb = fbase;
  for (int64_t p0 = pstart; p0 < pe && fb < F1; p0 += 32) {
    const int np = (int)(pe - p0 < 32 ? pe - p0 : 32);
    double vij = 0.0;
    int64_t cb = 0;
    int dg = 0;
    if (lane < np) {
      const int j = ci[p0 + lane];
      vij = v[p0 + lane];
      cb = colptr[j];
      dg = (int)(colptr[j + 1] - cb);
      if (dg > hot) dg = 0;   // a hot column's products come from the dense SYRK
    }
    int incl = dg;  // inclusive scan of the column degrees over the lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(FULL, incl, 31);
    const int tb = (int)max((int64_t)0, F0 - fb), te = (int)min((int64_t)total, F1 - fb);
    for (int t0 = tb; t0 < te; t0 += 32) {
      const int t = t0 + lane;
      const bool live = t < te;
      // column of flat index t: the first lane c with incl[c] > t
      int lo = 0, hi = 31;
#pragma unroll
      for (int it = 0; it < 5; ++it) {
        const int mid = (lo + hi) >> 1;
        const int im = __shfl_sync(FULL, incl, mid);
        if (im > t) hi = mid;
        else lo = mid + 1;
      }
      const int c = lo;
      const int ic = __shfl_sync(FULL, incl, c), dc = __shfl_sync(FULL, dg, c);
      const int64_t cbc = __shfl_sync(FULL, cb, c);
      const double vc = __shfl_sync(FULL, vij, c);
      int r = 0;
      double prod = 0.0;
      if (live) {
        const int64_t q = cbc + (t - (ic - dc));
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
    fb += total;
  }
  __syncwarp();
}

// Per row: the flat product count W_i = sum_{j in row i} |column j|, the exclusive prefix of
// the column degrees along the row (pref, per nnz), and nseg_i = ceil(W_i / GRAM_SEG) when a
// row needs more than one segment (else 0).  The segment slots are the exclusive scan of nseg
// (deterministic); rows whose slots would pass the capacity stay on the one-warp path.
constexpr int GRAM_SEG = 2048;
__global__ void gram_plan_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const int64_t* __restrict__ colptr, int32_t* __restrict__ pref,
                                 int64_t* __restrict__ nseg, int64_t hot) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s) return;
  int carry = 0;
  for (int64_t p0 = rp[w]; p0 < rp[w + 1]; p0 += 32) {
    const int64_t p = p0 + lane;
    int dg = 0;
    if (p < rp[w + 1]) {
      const int j = ci[p];
      dg = (int)(colptr[j + 1] - colptr[j]);
      if (dg > hot) dg = 0;
    }
    int incl = dg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (p < rp[w + 1]) pref[p] = carry + incl - dg;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) {
    const int ns = (carry + GRAM_SEG - 1) / GRAM_SEG;
    nseg[w] = ns > 1 ? ns : 0;
  }
}

__global__ void gram_slots_kernel(int64_t s, const int64_t* __restrict__ nseg, const int64_t* __restrict__ base,
                                  int maxseg, int* __restrict__ segmented, int2* __restrict__ seglist) {
  pdl_begin();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ns = nseg[i], b = base[i];
    const int ok = ns > 1 && b + ns <= maxseg;
    segmented[i] = ok;
    if (ok)
      for (int64_t k = 0; k < ns; ++k) seglist[b + k] = make_int2((int)i, (int)k);
  }
}

// K3 one warp per light row (all its products, straight into G), accumulator in shared memory.
template <bool SMEM>
__global__ void __launch_bounds__(128) sparse_gram_kernel(int64_t s, const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ ci, const double* __restrict__ v,
                                                          const int64_t* __restrict__ colptr,
                                                          const int32_t* __restrict__ crow,
                                                          const double* __restrict__ cval, double* __restrict__ G,
                                                          const int* __restrict__ segmented, int64_t hot) {
  pdl_begin();
  extern __shared__ double smem_acc[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; i < s; i += nw) {
    if (segmented[i]) continue;  // sparse_gram_seg_kernel + gram_merge_kernel
    double* acc = SMEM ? smem_acc + (int64_t)wib * s : G + i * s;
    for (int64_t c = lane; c < s; c += 32) acc[c] = 0.0;
    __syncwarp();
    gram_range(rp[i], rp[i + 1], 0, 0, INT64_MAX, ci, v, colptr, crow, cval, acc, hot);
    if (SMEM) {
      for (int64_t c = lane; c < s; c += 32) G[i * s + c] = acc[c];
      __syncwarp();
    }
  }
}

// K3 heavy rows: one warp per segment of GRAM_SEG products into its own partial row
template <bool SMEM>
__global__ void __launch_bounds__(128) sparse_gram_seg_kernel(int64_t s, const int64_t* __restrict__ rp,
                                                              const int32_t* __restrict__ ci,
                                                              const double* __restrict__ v,
                                                              const int64_t* __restrict__ colptr,
                                                              const int32_t* __restrict__ crow,
                                                              const double* __restrict__ cval,
                                                              const int32_t* __restrict__ pref,
                                                              const int2* __restrict__ seglist,
                                                              const int64_t* __restrict__ segcnt, int maxseg,
                                                              double* __restrict__ part, int64_t hot) {
  pdl_begin();
  extern __shared__ double smem_acc[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nsl = (int)min(*segcnt, (int64_t)maxseg);
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int slot = blockIdx.x * (blockDim.x >> 5) + wib; slot < nsl; slot += nw) {
    const int2 sg = seglist[slot];
    if (sg.x < 0) continue;
    const int64_t i = sg.x, b = rp[i], e = rp[i + 1];
    const int64_t F0 = (int64_t)sg.y * GRAM_SEG, F1 = F0 + GRAM_SEG;
    // the nnz holding flat index F0: the last p with pref[p] <= F0
    int64_t lo = b, hi = e - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (pref[mid] <= F0) lo = mid;
      else hi = mid - 1;
    }
    double* acc = SMEM ? smem_acc + (int64_t)wib * s : part + (int64_t)slot * s;
    for (int64_t c = lane; c < s; c += 32) acc[c] = 0.0;
    __syncwarp();
    gram_range(lo, e, pref[lo], F0, F1, ci, v, colptr, crow, cval, acc, hot);
    if (SMEM) {
      for (int64_t c = lane; c < s; c += 32) part[(int64_t)slot * s + c] = acc[c];
      __syncwarp();
    }
  }
}

// G[i, :] = sum over the segments of row i in segment order (deterministic); a row is found
// by its first slot
__global__ void gram_merge_kernel(int64_t s, const int2* __restrict__ seglist, const int64_t* __restrict__ segcnt,
                                  int maxseg, const int64_t* __restrict__ nseg, const double* __restrict__ part,
                                  double* __restrict__ G) {
  pdl_begin();
  const int nsl = (int)min(*segcnt, (int64_t)maxseg);
  for (int slot = blockIdx.y; slot < nsl; slot += gridDim.y) {
    const int2 sg = seglist[slot];
    if (sg.x < 0 || sg.y != 0) continue;
    const int64_t i = sg.x, ns = nseg[i];
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < s; c += (int64_t)gridDim.x * blockDim.x) {
      double a = 0.0;
      for (int64_t k = 0; k < ns; ++k) a += part[(int64_t)(slot + k) * s + c];
      G[i * s + c] = a;
    }
  }
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
  ++g_launches;
  launch_k(validate_kernel, cdiv(E.s * 32, 256), 256, 0, st, E.s, E.dim, E.nnz, E.row_ptr, E.col_idx, E.val, d_flag);
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
// the number of scalar products of the sparse Gram: sum over the nonzeros (i, j) of c_j (the
// count of column j) — the algorithmic flops (2 per product) of the profiling pass's accounting
__global__ void gram_products_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                     const int64_t* __restrict__ colptr, unsigned long long* __restrict__ total) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s) return;
  unsigned long long a = 0;
  for (int64_t p = rp[w] + lane; p < rp[w + 1]; p += 32) a += (unsigned long long)(colptr[ci[p] + 1] - colptr[ci[p]]);
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (lane == 0 && a) atomicAdd(total, a);
}
}  // namespace

double sparse_gram_products(cudaStream_t st, const DevCSR& E, const DevCSC& C) {
  if (E.s == 0) return 0.0;
  unsigned long long* d = nullptr;
  unsigned long long h = 0;
  if (cudaMallocAsync(&d, sizeof(unsigned long long), st) != cudaSuccess) return 0.0;
  cudaMemsetAsync(d, 0, sizeof(unsigned long long), st);
  launch_k(gram_products_kernel, cdiv(E.s * 32, 256), 256, 0, st, E.s, E.row_ptr, E.col_idx, C.colptr, d);
  cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  cudaStreamSynchronize(st);
  return (double)h;
}

namespace {
__global__ void hot_flag_kernel(int64_t nJ, const int32_t* __restrict__ J, const int64_t* __restrict__ colptr,
                                int64_t hot, int64_t* __restrict__ flag) {
  pdl_begin();
  const int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (jj < nJ) flag[jj] = (colptr[J[jj] + 1] - colptr[J[jj]] > hot) ? 1 : 0;
  if (jj == nJ) flag[nJ] = 0;
}
// D[i, hidx(j)] = v_ij for the nonzeros of the hot columns (D zeroed, s x h row-major)
__global__ void hot_dense_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const double* __restrict__ v, const int64_t* __restrict__ jpos,
                                 const int64_t* __restrict__ hpos, const int64_t* __restrict__ colptr, int64_t hot,
                                 int64_t h, double* __restrict__ D) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s) return;
  for (int64_t p = rp[w] + lane; p < rp[w + 1]; p += 32) {
    const int j = ci[p];
    if (colptr[j + 1] - colptr[j] > hot) D[w * h + hpos[jpos[j]]] = v[p];
  }
}
}  // namespace

// K3: the products of the cold columns by the flat sparse enumeration below; the hot columns
// (more than `hot` entries: Zipf-popular items, graph hubs — a few hundred columns that carry
// most of sum_j c_j^2) as a dense s x h block whose SYRK D D^T the DMMA GEMM adds to the upper
// triangle (the triangle the consumers read).  configs[2]: 2.6e8 products, 9.6 ms -> a 3.1e9-flop
// SYRK over ~250 hot items plus 1e7 cold products.
cudaError_t sparse_gram(cudaStream_t st, const DevCSR& E, const DevCSC& C, double* G, Scratch& ws) {
  const int64_t s = E.s;
  if (s == 0) return cudaSuccess;
  static const int64_t hot_env = getenv("TSVD_GRAM_HOT") ? atoll(getenv("TSVD_GRAM_HOT")) : 0;  // tuning; <0: off
  // (batches with few nonzeros per vector — graph node batches, ~5 — stay fully sparse: their
  // hub columns carry few products and the split costs a host synchronisation)
  const bool split = hot_env >= 0 && (hot_env > 0 || E.nnz >= 16 * s);
  const int64_t hot = !split ? INT64_MAX : (hot_env > 0 ? hot_env : std::max<int64_t>(64, s / 16));
  int64_t h = 0;
  int64_t* hpos = nullptr;
  if (hot != INT64_MAX && C.nJ > 0) {
    int64_t* hflag = ws.alloc<int64_t>(C.nJ + 1);
    hpos = ws.alloc<int64_t>(C.nJ + 1);
    if (ws.err) return ws.err;
    ++g_launches;
    launch_k(hot_flag_kernel, cdiv(C.nJ + 1, 256), 256, 0, st, C.nJ, C.J, C.colptr, hot, hflag);
    cudaError_t e1 = scan_exclusive(st, hflag, hpos, C.nJ + 1, ws);
    if (e1) return e1;
    static thread_local int64_t* h_cnt = nullptr;
    if (!h_cnt && cudaMallocHost(&h_cnt, sizeof(int64_t)) != cudaSuccess) return cudaErrorMemoryAllocation;
    if ((e1 = cudaMemcpyAsync(h_cnt, hpos + C.nJ, sizeof(int64_t), cudaMemcpyDeviceToHost, st))) return e1;
    if ((e1 = cudaStreamSynchronize(st))) return e1;
    h = *h_cnt;
  }
  const int64_t hot_used = h > 0 ? hot : INT64_MAX;
  cudaError_t e0 = sparse_gram_cold(st, E, C, G, ws, hot_used);
  if (e0 || h == 0) return e0;
  double* D = ws.alloc<double>((size_t)s * h);
  if (ws.err) return ws.err;
  if ((e0 = cudaMemsetAsync(D, 0, (size_t)s * h * sizeof(double), st))) return e0;
  ++g_launches;
  launch_k(hot_dense_kernel, cdiv(s * 32, 256), 256, 0, st, s, E.row_ptr, E.col_idx, E.val, C.jpos, hpos, C.colptr,
           hot, h, D);
  return dgemm(st, s, s, h, 1.0, CMat{D, h, 1}, CMat{D, 1, h}, 1.0, Mat{G, s, 1}, 1);
}

cudaError_t sparse_gram_cold(cudaStream_t st, const DevCSR& E, const DevCSC& C, double* G, Scratch& ws, int64_t hot) {
  const int64_t s = E.s;
  if (s == 0) return cudaSuccess;
  // segment capacity: up to 2048 partial rows within 128 MB
  const int maxseg = (int)std::max<int64_t>(64, std::min<int64_t>(2048, (int64_t(128) << 20) / (8 * s)));
  int32_t* pref = ws.alloc<int32_t>(std::max<int64_t>(E.nnz, 1));
  int64_t* nseg = ws.alloc<int64_t>(s + 1);
  int64_t* base = ws.alloc<int64_t>(s + 1);
  int* segmented = ws.alloc<int>(s);
  int2* seglist = ws.alloc<int2>(maxseg);
  double* part = ws.alloc<double>((size_t)maxseg * s);
  if (ws.err) return ws.err;
  cudaError_t e;
  if ((e = cudaMemsetAsync(seglist, 0xff, maxseg * sizeof(int2), st))) return e;
  if ((e = cudaMemsetAsync(nseg + s, 0, sizeof(int64_t), st))) return e;
  g_launches += 5;
  launch_k(gram_plan_kernel, cdiv(s * 32, 256), 256, 0, st, s, E.row_ptr, E.col_idx, C.colptr, pref, nseg, hot);
  if ((e = scan_exclusive(st, nseg, base, s + 1, ws))) return e;
  launch_k(gram_slots_kernel, (unsigned)std::min<int64_t>(cdiv(s, 256), 148 * 4), 256, 0, st, s, nseg, base, maxseg,
                                                                                        segmented, seglist);
  const size_t smem = 4 * (size_t)s * sizeof(double);
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(s, 4), 148 * 8);
  const unsigned sblocks = (unsigned)std::min<int64_t>(cdiv(maxseg, 4), 148 * 8);
  // the row accumulator in global memory (L2) by default: a shared-memory row of s doubles per
  // warp allows only 4 warps per SM, too few to hide the CSC walk's load latency (configs[1]:
  // 0.86 -> 0.67 ms per batch); TSVD_GRAM_SMEM=1 keeps the shared-memory accumulator
  static const bool smem_on = getenv("TSVD_GRAM_SMEM") && atoi(getenv("TSVD_GRAM_SMEM")) == 1;
  if (smem <= 200 * 1024 && smem_on) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(sparse_gram_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(sparse_gram_seg_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    launch_k(sparse_gram_seg_kernel<true>, sblocks, 128, smem, st, s, E.row_ptr, E.col_idx, E.val, C.colptr, C.row, C.val,
                                                             pref, seglist, base + s, maxseg, part, hot);
    launch_k(sparse_gram_kernel<true>, blocks, 128, smem, st, s, E.row_ptr, E.col_idx, E.val, C.colptr, C.row, C.val, G,
                                                        segmented, hot);
  } else {
    launch_k(sparse_gram_seg_kernel<false>, sblocks, 128, 0, st, s, E.row_ptr, E.col_idx, E.val, C.colptr, C.row, C.val,
                                                           pref, seglist, base + s, maxseg, part, hot);
    launch_k(sparse_gram_kernel<false>, blocks, 128, 0, st, s, E.row_ptr, E.col_idx, E.val, C.colptr, C.row, C.val, G,
                                                      segmented, hot);
  }
  dim3 mg(cdiv(s, 256), 32);
  launch_k(gram_merge_kernel, mg, 256, 0, st, s, seglist, base + s, maxseg, nseg, part, G);
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
