// api.cu — the C-ABI (include/tsvd.h, include/tsvd_kernels.h) and the host orchestration
// of one update: which kernels run, in which order, on which side.
//
// State (Eq (4)): per side x in {U, V}: base factor X' (rows x k,
// row-major, capacity-grown), multiplier X'' (k x k), and Σ (k).  U = U' U'', V = V' V''.
//
// One exact update with lift side X and (for rows/columns) append side Y
// (Alg 3, Alg 9; SURVEY §3 call stack (2)):
//   A1  K1 build_csc: E^T -> CSC over the X' rows it touches (J)
//   A2  K2 gather_spmm W = E X';  K4  C0^T = W X''                      (Lemma 1)
//   A3  K3 sparse_gram E E^T;  K4 SYRK  G = E E^T - C0^T C0            (Lemma 2)
//   A4  K5 chol_deflate G = R^T R with deflation; compaction of kept pivots  (Alg 2)
//   A5  core K = [[Σ, 0], [C0^T, R_kept^T]];  K7/K8 jacobi_svd -> F, Θ, G
//   A6  Y'' <- Y'' F[:k];  K6 Y = R^{-1} G[k:];  X'' <- X'' (G[:k] - C0 Y);  K15 inverses + cond
//   A7  append rows F[k:] Y''^{-1} to Y'   (or reset: Y' <- Y' Y'', rows F[k:], Y'' = I)
//   A8  K10 X'[J] += E^T (Y X''^{-1})      (or reset: X' <- X' X'', += E^T Y, X'' = I)
// Weight updates lift both sides and form the core diag(Σ,0) + L_D L_E^T (Alg 4).
// Everything up to the commit writes scratch only, so a failed update leaves the state
// unchanged.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <fcntl.h>
#include <unistd.h>

#include "../../include/tsvd.h"
#include "../../include/tsvd_kernels.h"
#include "ops.h"

namespace tsvd {
thread_local long long g_launches = 0;
thread_local KProfiler* g_prof = nullptr;

cudaEvent_t KProfiler::get() {
  if (used == pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
  }
  return pool[used++];
}

int KProfiler::begin(int cls, double flops, double bytes, cudaStream_t on) {
  Rec r{cls, get(), get(), flops, bytes, g_launches, g_launches, on ? on : st};
  cudaEventRecord(r.a, r.s);
  recs.push_back(r);
  return (int)recs.size() - 1;
}

void KProfiler::end(int idx) {
  cudaEventRecord(recs[idx].b, recs[idx].s);
  recs[idx].l1 = g_launches;
}

void KProfiler::resolve(float* ms, double* flops, double* bytes, int* launches) {
  for (int c = 0; c < KC_N; ++c) {
    ms[c] = 0.f;
    flops[c] = bytes[c] = 0.0;
    launches[c] = 0;
  }
  if (recs.empty()) return;
  for (const Rec& r : recs) cudaEventSynchronize(r.b);
  for (const Rec& r : recs) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) {
      cudaGetLastError();
      t = 0.f;
    }
    ms[r.cls] += t;
    flops[r.cls] += r.flops;
    bytes[r.cls] += r.bytes;
    launches[r.cls] += (int)(r.l1 - r.l0);
  }
}

KProfiler::~KProfiler() {
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
}
}  // namespace tsvd

using namespace tsvd;

struct tsvd_ctx {
  int device = 0;
  bool times_pending = false;  // the last update's phase times await its events
  int k = 0;
  int64_t rows[2] = {0, 0};  // global m (U side), n (V side)
  // Row sharding (shard.cu): global row i of U' / V' lives on shard
  // (i / block) % world.  This context holds nloc shards starting at shard0: NCCL mode
  // nloc = 1, shard0 = rank; virtual mode nloc = world, shard0 = 0; unsharded world = 1.
  int world = 1, nloc = 1, shard0 = 0, block = 1024;
  void* comm = nullptr;              // ncclComm_t (NCCL mode, world > 1)
  std::vector<double*> X[2];         // U', V' per local shard (local rows x k, row-major)
  std::vector<int64_t> cap[2];       // capacity per local shard (rows)
  double* M[2] = {nullptr, nullptr};  // U'', V'' (replicated)
  // deferred MII resets of an append-only side: global rows [r0, r1) hold U = X' P M (P k x k,
  // device) — the materialisation X' <- X' P is postponed until the side is read as a whole or
  // becomes a lift side (flush_pending); a row query applies P M directly
  struct PendBlock {
    int64_t r0, r1;
    double* P;
  };
  std::vector<PendBlock> pend[2];
  double* Sigma = nullptr;
  bool initialized = false;
  int total_resets = 0;
  // per core kind (0: column update, 1: row update, 2: weight update)
  int core_hint[3] = {0, 0, 0};  // subspace iterations the last core SVD needed
  double core_growth[3] = {0, 0, 0};  // its per-step growth (theta_1 / theta_b)^2
  double core_thb2[3] = {0, 0, 0};    // its last Ritz theta_b^2 (Chebyshev interval)
  int core_b[3] = {0, 0, 0};          // subspace width suggested for the next core (CoreInfo::b_next)
  tsvd_stats stats;
  std::string err;
  KProfiler kprof;
  int64_t* h_i64 = nullptr;  // pinned staging for small read-backs
  double* h_f64 = nullptr;
  cudaEvent_t ev[4];
  // second stream of the weight update: the U side (D) and the V side (E) of an approximate
  // (RPI / GKL) weight update are independent until the core, and run concurrently
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
};

namespace {

#define CK(call)                                                                                 \
  do {                                                                                           \
    cudaError_t _e = (call);                                                                     \
    if (_e != cudaSuccess) {                                                                     \
      ctx->err = std::string(#call) + " -> " + cudaGetErrorString(_e);                          \
      return TSVD_E_CUDA;                                                                        \
    }                                                                                            \
  } while (0)

#define CKS(stmt)                                                                                \
  do {                                                                                           \
    tsvd_status _s = (stmt);                                                                     \
    if (_s != TSVD_OK) return _s;                                                                \
  } while (0)

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Borrow device arrays directly; copy host arrays into scratch.
template <class T>
const T* stage(const T* p, size_t count, Scratch& ws, cudaStream_t st, cudaError_t* err) {
  if (count == 0 || p == nullptr) return p;
  if (is_device_ptr(p)) return p;
  T* d = ws.alloc<T>(count);
  if (!d) { *err = ws.err; return nullptr; }
  *err = cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, st);
  return d;
}

tsvd_status set_err(tsvd_ctx* ctx, tsvd_status s, const std::string& msg) {
  ctx->err = msg;
  return s;
}

// local row count of shard g at a given global row count (declared below)
int64_t lrows(const tsvd_ctx* ctx, int side, int g, int64_t global_rows);

// Materialise the deferred resets of one side (X' <- X' P on each pending row range, per
// local shard: a global range maps to a contiguous local range) and drop them.
tsvd_status flush_pending(tsvd_ctx* ctx, int side, cudaStream_t st) {
  if (ctx->pend[side].empty()) return TSVD_OK;
  const int k = ctx->k;
  for (auto& b : ctx->pend[side]) {
    for (int g = 0; g < ctx->nloc; ++g) {
      const int64_t lo = lrows(ctx, side, g, b.r0), hi = lrows(ctx, side, g, b.r1);
      if (hi > lo) CK(materialize_rows(st, ctx->X[side][g] + lo * k, hi - lo, k, b.P));
    }
    CK(cudaFreeAsync(b.P, st));
  }
  ctx->pend[side].clear();
  return TSVD_OK;
}

void drop_pending(tsvd_ctx* ctx) {  // (re-)initialisation / destroy: the factors are replaced
  for (int s = 0; s < 2; ++s) {
    for (auto& b : ctx->pend[s]) cudaFree(b.P);
    ctx->pend[s].clear();
  }
}

// The multiplier of global row i of a side: M, or P M (into tmp) inside a pending block
tsvd_status row_multiplier(tsvd_ctx* ctx, int side, int64_t i, double* tmp, const double** out, cudaStream_t st) {
  *out = ctx->M[side];
  for (auto& b : ctx->pend[side])
    if (i >= b.r0 && i < b.r1) {
      const int k = ctx->k;
      CK(dgemm_rm(st, false, false, k, k, k, 1.0, b.P, k, ctx->M[side], k, 0.0, tmp, k));
      *out = tmp;
      break;
    }
  return TSVD_OK;
}

int64_t lrows(const tsvd_ctx* ctx, int side, int g, int64_t global_rows) {
  const int64_t R = global_rows < 0 ? ctx->rows[side] : global_rows;
  return ctx->world == 1 ? R : shard_rows(R, ctx->shard0 + g, ctx->world, ctx->block);
}

int64_t lrows(const tsvd_ctx* ctx, int side, int g) { return lrows(ctx, side, g, -1); }

// grow every local shard of one side to hold `need` global rows
tsvd_status ensure_cap(tsvd_ctx* ctx, int side, int64_t need, cudaStream_t st) {
  for (int g = 0; g < ctx->nloc; ++g) {
    const int64_t nl = lrows(ctx, side, g, need), cur = lrows(ctx, side, g);
    if (nl <= ctx->cap[side][g]) continue;
    int64_t nc = std::max<int64_t>(nl, ctx->cap[side][g] + ctx->cap[side][g] / 2 + 1024);
    double* p = nullptr;
    CK(cudaMallocAsync(&p, (size_t)nc * ctx->k * sizeof(double), st));
    if (ctx->X[side][g] && cur > 0)
      CK(cudaMemcpyAsync(p, ctx->X[side][g], (size_t)cur * ctx->k * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (ctx->X[side][g]) CK(cudaFreeAsync(ctx->X[side][g], st));
    ctx->X[side][g] = p;
    ctx->cap[side][g] = nc;
  }
  return TSVD_OK;
}

// Sum count doubles over all shards: parts[g] is local shard g's partial; the total ends
// in parts[0] (on every process in NCCL mode).
tsvd_status reduce_parts(tsvd_ctx* ctx, const std::vector<double*>& parts, int64_t count, cudaStream_t st) {
  for (int g = 1; g < (int)parts.size(); ++g) CK(add_into(st, parts[0], parts[g], count));
  if (ctx->comm && count > 0) {
    const int rc = nccl_allreduce_sum_f64(ctx->comm, parts[0], count, st);
    if (rc != 0) return set_err(ctx, TSVD_E_NCCL, std::string("ncclAllReduce: ") + nccl_error(rc));
  }
  return TSVD_OK;
}

// partial buffers: parts[0] is the result buffer, parts[1..] scratch (virtual shards)
std::vector<double*> alloc_parts(tsvd_ctx* ctx, int64_t count, Scratch& ws) {
  std::vector<double*> v(ctx->nloc);
  for (int g = 0; g < ctx->nloc; ++g) v[g] = ws.alloc<double>((size_t)std::max<int64_t>(count, 1));
  return v;
}

// Validate + stage one sparse block on the device.
tsvd_status stage_sparse(tsvd_ctx* ctx, const tsvd_sparse* in, int64_t expect_dim, Scratch& ws, cudaStream_t st,
                         DevCSR& out, int* d_flag, bool validate) {
  if (!in) return set_err(ctx, TSVD_E_INVALID, "null sparse block");
  if (in->s < 0 || in->nnz < 0 || in->dim < 0) return set_err(ctx, TSVD_E_INVALID, "negative size");
  if (in->dim != expect_dim)
    return set_err(ctx, TSVD_E_SHAPE, "update dim " + std::to_string(in->dim) + " != " + std::to_string(expect_dim));
  if (in->s > 0 && in->nnz > 0 && (!in->row_ptr || !in->col_idx || !in->val))
    return set_err(ctx, TSVD_E_INVALID, "null CSR array");
  if (in->s > 0 && !in->row_ptr) return set_err(ctx, TSVD_E_INVALID, "null row_ptr");
  cudaError_t e = cudaSuccess;
  out.s = in->s;
  out.dim = in->dim;
  out.nnz = in->nnz;
  if (in->s == 0) {
    if (in->nnz != 0) return set_err(ctx, TSVD_E_INVALID, "s == 0 with nnz > 0");
    return TSVD_OK;
  }
  out.row_ptr = stage(in->row_ptr, (size_t)in->s + 1, ws, st, &e);
  if (e) return set_err(ctx, TSVD_E_CUDA, cudaGetErrorString(e));
  out.col_idx = stage(in->col_idx, (size_t)in->nnz, ws, st, &e);
  if (e) return set_err(ctx, TSVD_E_CUDA, cudaGetErrorString(e));
  out.val = stage(in->val, (size_t)in->nnz, ws, st, &e);
  if (e) return set_err(ctx, TSVD_E_CUDA, cudaGetErrorString(e));
  // row_ptr[0] == 0 and row_ptr[s] == nnz, and (validate) the per-row checks: one readback
  // (the validation kernel keeps its reads inside [0, nnz) whatever the endpoints are)
  if (validate) CK(validate_csr(st, out, d_flag));
  CK(cudaMemcpyAsync(ctx->h_i64, out.row_ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ctx->h_i64 + 1, out.row_ptr + in->s, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  if (validate) CK(cudaMemcpyAsync(ctx->h_i64 + 2, d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (ctx->h_i64[0] != 0 || ctx->h_i64[1] != in->nnz) return set_err(ctx, TSVD_E_INVALID, "row_ptr endpoints");
  if (validate) {
    // must be known before any kernel indexes with col_idx (K1 histogram)
    const int flag = *reinterpret_cast<int*>(ctx->h_i64 + 2);
    if (flag & 1) return set_err(ctx, TSVD_E_INVALID, "CSR column index out of range, unsorted or duplicate");
    if (flag & 2) return set_err(ctx, TSVD_E_NUMERIC, "non-finite value in update");
  }
  return TSVD_OK;
}

// One lift side: A1-A2 always; A3-A4 (exact, Alg 2 as Cholesky-QR) or the approximate
// augmented space (RPI Alg 8 / GKL Alg 6, App D).
struct LiftShard {
  DevCSR E;                 // the columns of E owned by this shard (local indices)
  DevCSC C;                 // its CSC over the touched local rows J
  GatherMaps gm;            // approx: index maps for the gather-SpMM form of E P and E^T B'
  double* BJ = nullptr;     // approx: B' on J (nJ x l)
};

struct Lift {
  int side = 0;
  int mode = TSVD_EXACT;
  DevCSR E;                 // the whole update block (replicated)
  std::vector<LiftShard> sh;
  double* P0 = nullptr;     // s x k : C0^T = E X
  int64_t nJ = 0;           // |J| over the local shards
  // exact
  DevCSC Cfull;             // CSC of the whole E (sparse Gram); = sh[0].C when unsharded
  double* R = nullptr;      // s x s : Gram -> R (upper)
  double* enorm2 = nullptr; // s
  int32_t* keep = nullptr;  // s
  double* Tb = nullptr;     // ceil(s/64) x 64 x 64 : R_qq^+ of the diagonal tiles (dag.cu)
  int32_t* kidx = nullptr;  // 2s : kidx | klist
  int64_t r = 0;
  // approximate (RPI / GKL): Q = B' - X C'
  int64_t l = 0;
  double* Cp = nullptr;     // k x l  : C'
  double* Pa = nullptr;     // s x l  : P (Q^T Z = P^T)
  int64_t extra() const { return mode == TSVD_EXACT ? r : l; }
};

// A1 + A2: per local shard the split of E, its CSC over J and the partial W_g = E_g X'_g;
// W = sum_g W_g (Reducer), C0^T = W X''  (Lemma 1 under the extended decomposition)
tsvd_status lift_common(tsvd_ctx* ctx, Lift& L, Scratch& ws, cudaStream_t st) {
  const int k = ctx->k;
  const int64_t s = L.E.s;
  L.sh.assign(ctx->nloc, LiftShard());
  std::vector<double*> Wp = alloc_parts(ctx, s * k, ws);
  L.P0 = ws.alloc<double>((size_t)s * k);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  L.nJ = 0;
  for (int g = 0; g < ctx->nloc; ++g) {
    LiftShard& S = L.sh[g];
    if (ctx->world == 1) {
      S.E = L.E;
    } else {
      CK(shard_split(st, L.E, ctx->shard0 + g, ctx->world, ctx->block, lrows(ctx, L.side, g), S.E, ws, ctx->h_i64));
    }
    int64_t h_nJ = 0;
    CK(build_csc(st, S.E, S.C, ws, &h_nJ));  // synchronises (|J| read-back)
    L.nJ += h_nJ;
    KScope sc(KC_GATHER, 2.0 * S.E.nnz * k, 12.0 * S.E.nnz + 8.0 * k * (h_nJ + s));
    CK(gather_spmm(st, S.E, ctx->X[L.side][g], k, Wp[g]));
  }
  CKS(reduce_parts(ctx, Wp, s * k, st));
  CK(dgemm_rm(st, false, false, s, k, k, 1.0, Wp[0], k, ctx->M[L.side], k, 0.0, L.P0, k));
  return TSVD_OK;
}

tsvd_status lift_exact(tsvd_ctx* ctx, Lift& L, double tau, Scratch& ws, cudaStream_t st) {
  const int k = ctx->k;
  const int64_t s = L.E.s;
  CKS(lift_common(ctx, L, ws, st));
  if (ctx->world == 1) {
    L.Cfull = L.sh[0].C;
  } else {  // the sparse Gram needs all columns of E (replicated work, no s x s allreduce)
    int64_t nJf = 0;
    CK(build_csc(st, L.E, L.Cfull, ws, &nJf));
  }
  L.R = ws.alloc<double>((size_t)s * s);
  L.enorm2 = ws.alloc<double>(s);
  L.keep = ws.alloc<int32_t>(s);
  L.Tb = ws.alloc<double>((size_t)((s + 63) / 64) * 64 * 64);
  L.kidx = ws.alloc<int32_t>(2 * s);
  int64_t* d_r = ws.alloc<int64_t>(1);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  {
    // algorithmic work: 2 flops per scalar product (counted on the device in the profiling pass)
    const double prods = g_prof ? sparse_gram_products(st, L.E, L.Cfull) : 0.0;
    KScope sc(KC_SGRAM, 2.0 * prods, 4.0 * s * (s + 1) + 24.0 * L.E.nnz);
    CK(sparse_gram(st, L.E, L.Cfull, L.R, ws));
  }
  CK(copy_diag(st, L.R, s, L.enorm2));
  CK(dgemm_rm(st, false, true, s, s, k, -1.0, L.P0, k, L.P0, k, 1.0, L.R, s, 1));
  CK(chol_deflate(st, L.R, s, L.enorm2, tau, L.keep, L.Tb));
  CK(compact_keep(st, L.keep, s, L.kidx, d_r, ws));
  CK(cudaMemcpyAsync(ctx->h_i64, d_r, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  L.r = ctx->h_i64[0];
  return TSVD_OK;
}

// Approximate augmented space.  sketch: this side's s x l start block (RPI) or s-vector
// (GKL), host or device, or null to draw it with K12 from (seed, side_id).
tsvd_status lift_approx(tsvd_ctx* ctx, Lift& L, const tsvd_opts& o, const double* sketch, int side_id, Scratch& ws,
                        cudaStream_t st) {
  const int k = ctx->k;
  const int64_t s = L.E.s;
  CKS(lift_common(ctx, L, ws, st));
  L.l = std::min<int64_t>(o.l, s);  // l >= s spans R^s: identical range, exact result (R15)
  const int64_t l = L.l;
  if (o.mode == TSVD_GKL && ctx->world > 1)
    return set_err(ctx, TSVD_E_UNSUPPORTED, "GKL on a sharded context is not implemented (use RPI or exact)");
  for (int g = 0; g < ctx->nloc; ++g) {
    L.sh[g].BJ = ws.alloc<double>((size_t)std::max<int64_t>(L.sh[g].C.nJ, 1) * l);
    if (o.mode == TSVD_RPI) CK(gather_maps(st, L.sh[g].E, L.sh[g].C, L.sh[g].gm, ws));
  }
  L.Cp = ws.alloc<double>((size_t)k * l);
  L.Pa = ws.alloc<double>((size_t)s * l);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  const int64_t ncols_in = (o.mode == TSVD_RPI) ? o.l : 1;
  // the library's own RPI start block with l = o.l is drawn straight into P (a 226 MB s x l
  // device copy per side on configs[3] otherwise)
  const bool direct = o.mode == TSVD_RPI && !sketch && ncols_in == l;
  double* start = direct ? L.Pa : ws.alloc<double>((size_t)s * ncols_in);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  if (sketch) {
    if (is_device_ptr(sketch))
      CK(cudaMemcpyAsync(start, sketch, (size_t)s * ncols_in * sizeof(double), cudaMemcpyDeviceToDevice, st));
    else
      CK(cudaMemcpyAsync(start, sketch, (size_t)s * ncols_in * sizeof(double), cudaMemcpyHostToDevice, st));
  } else {
    CK(counter_gaussian(st, o.seed, side_id, s, ncols_in, start));
  }
  if (o.mode == TSVD_RPI) {
    // keep the first l of the o.l start columns (l < o.l only when o.l > s: same range)
    if (!direct)
      CK(cudaMemcpy2DAsync(L.Pa, l * sizeof(double), start, ncols_in * sizeof(double), l * sizeof(double), s,
                           cudaMemcpyDeviceToDevice, st));
    std::vector<double*> Pp = alloc_parts(ctx, s * l, ws);
    std::vector<double*> Gp = alloc_parts(ctx, l * l, ws);
    double* en = ws.alloc<double>(l);
    int32_t* keep = ws.alloc<int32_t>(l);
    double* T = ws.alloc<double>((size_t)l * l);
    double* Pa2 = ws.alloc<double>((size_t)s * l);   // ping-pong partners (no copies back)
    double* Cp2 = ws.alloc<double>((size_t)k * l);
    std::vector<double*> BJ2(ctx->nloc);
    for (int g = 0; g < ctx->nloc; ++g) BJ2[g] = ws.alloc<double>((size_t)std::max<int64_t>(L.sh[g].C.nJ, 1) * l);
    if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
    // (under NCCL each rank sees only its own part of J: the choice would not be replicated, so
    // the fold is off there — every rank must launch the same products to stay bitwise equal)
    int64_t nJtot = 0;
    for (int g = 0; g < ctx->nloc; ++g) nJtot += L.sh[g].C.nJ;
    static const bool fold_env = !(getenv("TSVD_RPI_FOLD") && atoi(getenv("TSVD_RPI_FOLD")) == 0);  // tuning
    const bool fold_on = fold_env && ctx->comm == nullptr;
    const Scratch::Mark it_mark = ws.mark();
    for (int it = 0; it < o.t; ++it) {
      ws.rewind(it_mark);  // per-iteration Cholesky-QR workspaces
      // Alg 7 line 4 (P <- QR(P)): Z P depends on range(P) only, and one Cholesky-QR pass
      // returns a well-conditioned basis of exactly that range (a second pass would only
      // sharpen its orthogonality, which nothing downstream uses)
      // (the library's own K12 start block with s >= 4 l is an i.i.d. Gaussian block, condition
      // number <= (1 + sqrt(l/s)) / (1 - sqrt(l/s)) <= 3 with overwhelming probability: its range
      // needs no conditioning pass; a caller's sketch always gets one)
      if (!(it == 0 && !sketch && s >= 4 * l)) {
        CK(cholqr_dense(st, L.Pa, s, l, o.defl_tol, 1, nullptr, ws, Pa2));
        std::swap(L.Pa, Pa2);
      }
      for (int g = 0; g < ctx->nloc; ++g)
        CK(csc_spmm(st, L.sh[g].C, &L.sh[g].gm, L.sh[g].E.nnz, L.Pa, (int)l, L.sh[g].BJ));   // B' = E P
      CK(dgemm_rm(st, true, false, k, l, s, 1.0, L.P0, k, L.Pa, l, 0.0, L.Cp, l));          // C' = C0 P
      // Alg 2 on the tuples (Q = B' - X C') as Cholesky-QR: Gram sum_g B'_g^T B'_g - C'^T C'.
      // Intermediate iterations carry only the range of Q into P = Z^T Q: one pass; the last
      // Q is the basis of the core (App D.3 assumes Q^T Q = I): two passes (Cholesky-QR2)
      const bool last = it + 1 == o.t;
      const int qpasses = last ? 2 : 1;
      // an intermediate tuple is used only through P = Z^T Q = (E^T B' - C0^T C') T: when the
      // support J has more rows than the update (configs[4]: |J| = 1.26M against s = 1e5) T is
      // applied to the s x l P instead of the |J| x l B' (same product in exact arithmetic)
      const bool fold = !last && fold_on && nJtot * 2 > 3 * s;
      for (int pass = 0; pass < qpasses; ++pass) {
        for (int g = 0; g < ctx->nloc; ++g)
          CK(dgemm_rm(st, true, false, l, l, L.sh[g].C.nJ, 1.0, L.sh[g].BJ, l, L.sh[g].BJ, l, 0.0, Gp[g], l, 1));
        CKS(reduce_parts(ctx, Gp, l * l, st));
        CK(copy_diag(st, Gp[0], l, en));
        CK(dgemm_rm(st, true, false, l, l, k, -1.0, L.Cp, l, L.Cp, l, 1.0, Gp[0], l, 1));
        CK(chol_rinv(st, Gp[0], l, en, o.defl_tol, keep, T, ws, false));
        if (fold) break;
        for (int g = 0; g < ctx->nloc; ++g) {
          if (L.sh[g].C.nJ) CK(dgemm_rm_btri(st, L.sh[g].C.nJ, l, l, L.sh[g].BJ, l, T, l, BJ2[g], l));
          std::swap(L.sh[g].BJ, BJ2[g]);
        }
        CK(dgemm_rm_btri(st, k, l, l, L.Cp, l, T, l, Cp2, l));   // T = R^+ is upper triangular
        std::swap(L.Cp, Cp2);
      }
      // P = sum_g E_g^T B'_g - C0^T C'
      for (int g = 0; g < ctx->nloc; ++g)
        CK(csr_gather_compact(st, L.sh[g].E, L.sh[g].C.jpos, &L.sh[g].gm, L.sh[g].BJ, (int)l, Pp[g]));
      CKS(reduce_parts(ctx, Pp, s * l, st));
      std::swap(L.Pa, Pp[0]);   // (Pp[0] takes the old P buffer: both live until the update ends)
      CK(dgemm_rm(st, false, false, s, l, k, -1.0, L.P0, k, L.Cp, l, 1.0, L.Pa, l));
      if (fold) {
        CK(dgemm_rm_btri(st, s, l, l, L.Pa, l, T, l, Pa2, l));
        std::swap(L.Pa, Pa2);
      }
    }
  } else {
    CK(gkl_basis(st, L.sh[0].E, L.sh[0].C, L.P0, k, start, (int)l, o.defl_tol, L.sh[0].BJ, L.Cp, L.Pa, ws));
  }
  return TSVD_OK;
}

tsvd_status lift_any(tsvd_ctx* ctx, Lift& L, const tsvd_opts& o, const double* sketch, int side_id, Scratch& ws,
                     cudaStream_t st) {
  L.mode = o.mode;
  if (o.mode == TSVD_EXACT) return lift_exact(ctx, L, o.defl_tol, ws, st);
  return lift_approx(ctx, L, o, sketch, side_id, ws, st);
}

// A6 for a lift side from its block Gs ((k+extra) x k col-major, ld) of the core's
// singular vectors: T = Gs[:k] - C Gs[k:], Mnew = X'' T, Minv, cond, and the coefficient
// rows Y of the sparse row update (exact: R^{-1} Gs[k:] over s; approx: Gs[k:] over l).
struct LiftPost {
  double* Y = nullptr;     // (s or l) x k
  double* Mnew = nullptr;  // k x k
  double* Minv = nullptr;
  double* cond = nullptr;  // device scalar
};

tsvd_status lift_post(tsvd_ctx* ctx, const Lift& L, const double* Fs, int64_t ld, LiftPost& P, Scratch& ws,
                      cudaStream_t st) {
  const int k = ctx->k;
  const int64_t s = L.E.s;
  const bool exact = L.mode == TSVD_EXACT;
  const int64_t yrows = exact ? s : L.l;
  P.Y = ws.alloc<double>((size_t)std::max<int64_t>(yrows, 1) * k);
  double* T = ws.alloc<double>((size_t)k * k);
  P.Mnew = ws.alloc<double>((size_t)k * k);
  P.Minv = ws.alloc<double>((size_t)k * k);
  P.cond = ws.alloc<double>(1);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  if (exact) {
    CK(expand_rows(st, Fs, ld, k, s, L.kidx, P.Y));
    CK(trsm_upper(st, L.R, s, L.keep, P.Y, k, L.Tb));
    // T = Fs[:k] - C0 Y   (C0 = P0^T; C0 R^{-1} Gs[k:] = C Gs[k:], R5)
    CK(dgemm(st, k, k, s, -1.0, CMat{L.P0, 1, k}, CMat{P.Y, k, 1}, 0.0, Mat{T, k, 1}, 0));
  } else {
    CK(colmajor_to_rowmajor(st, Fs + k, ld, L.l, k, P.Y, k));
    // T = Fs[:k] - C' Gs[k:]   (App D.3, PAPER.md:940 / 966)
    CK(dgemm(st, k, k, L.l, -1.0, CMat{L.Cp, L.l, 1}, CMat{P.Y, k, 1}, 0.0, Mat{T, k, 1}, 0));
  }
  CK(mat_axpby(st, k, k, 1.0, CMat{Fs, 1, ld}, 1.0, Mat{T, k, 1}));
  CK(dgemm_rm(st, false, false, k, k, k, 1.0, ctx->M[L.side], k, T, k, 0.0, P.Mnew, k));
  CK(inverse_gj(st, P.Mnew, k, P.Minv, P.cond, ws));
  return TSVD_OK;
}

// MII decision (reading R18): reset a new multiplier M when its 2-norm condition number
// exceeds tau.  cond_1 (Gauss-Jordan, always computed) decides the common case — no reset while
// cond_1 <= tau; above, cond_2 = ||M||_2 ||M^-1||_2 is estimated by power iterations (one small
// launch and one synchronisation, only then): cond_1 overstates cond_2 by up to k (k = 256: C5
// reset about every third batch on cond_1, each a materialisation of the 18M x 256 U').
// in: c1[i] for the nm multipliers (M[i], Minv[i]); out: reset[i]
tsvd_status mii_decide(tsvd_ctx* ctx, int nm, const double* const* M, const double* const* Minv, const double* c1,
                       double tau, bool* reset, Scratch& ws, cudaStream_t st) {
  const double* mats[4];
  int idx[2], n = 0;
  for (int i = 0; i < nm; ++i) {
    reset[i] = false;
    if (!(c1[i] <= tau)) {
      if (!std::isfinite(c1[i])) {
        reset[i] = true;  // singular or non-finite: reset outright
        continue;
      }
      mats[2 * n] = M[i];
      mats[2 * n + 1] = Minv[i];
      idx[n++] = i;
    }
  }
  if (n == 0) return TSVD_OK;
  double* d = ws.alloc<double>(4);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  CK(norm2_estimates(st, mats, 2 * n, ctx->k, d));
  CK(cudaMemcpyAsync(ctx->h_f64 + 8, d, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int q = 0; q < n; ++q) {
    const double c2 = ctx->h_f64[8 + 2 * q] * ctx->h_f64[9 + 2 * q];
    reset[idx[q]] = !(c2 <= tau);
  }
  return TSVD_OK;
}

// A8 commit for a lift side (+ MII reset): X'[J] += (E^T R^{-1} or B') Gs[k:] M^{-1}, per shard.
tsvd_status lift_commit(tsvd_ctx* ctx, const Lift& L, const LiftPost& P, bool reset, Scratch& ws, cudaStream_t st) {
  const int k = ctx->k;
  const int side = L.side;
  const bool exact = L.mode == TSVD_EXACT;
  const int64_t yrows = exact ? L.E.s : L.l;
  const double* Z = P.Y;
  if (!reset) {
    double* Zi = ws.alloc<double>((size_t)std::max<int64_t>(yrows, 1) * k);
    if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
    CK(dgemm_rm(st, false, false, yrows, k, k, 1.0, P.Y, k, P.Minv, k, 0.0, Zi, k));
    Z = Zi;
  } else {
    for (int g = 0; g < ctx->nloc; ++g) CK(materialize_rows(st, ctx->X[side][g], lrows(ctx, side, g), k, P.Mnew));
  }
  KScope sc(KC_SCATTER, 2.0 * L.E.nnz * k, 12.0 * L.E.nnz + 16.0 * k * L.nJ + 8.0 * k * yrows);
  for (int g = 0; g < (int)L.sh.size(); ++g) {  // (no shards when every update vector was empty)
    const LiftShard& S = L.sh[g];
    if (exact) {
      CK(scatter_add(st, S.C, S.E.nnz, Z, k, ctx->X[side][g]));
    } else if (S.C.nJ > 0) {
      double* ZJ = ws.alloc<double>((size_t)S.C.nJ * k);
      if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
      CK(dgemm_rm(st, false, false, S.C.nJ, k, L.l, 1.0, S.BJ, L.l, Z, k, 0.0, ZJ, k));
      CK(index_add_rows(st, S.C.J, S.C.nJ, ZJ, k, ctx->X[side][g]));
    }
  }
  if (!reset)
    CK(cudaMemcpyAsync(ctx->M[side], P.Mnew, (size_t)k * k * sizeof(double), cudaMemcpyDeviceToDevice, st));
  else
    CK(set_identity(st, ctx->M[side], k));
  return TSVD_OK;
}

// A7: write the s new rows R (s x k, row-major, replicated) at global rows rows[side]..
tsvd_status append_rows(tsvd_ctx* ctx, int side, const double* R, int64_t s, cudaStream_t st) {
  for (int g = 0; g < ctx->nloc; ++g) {
    if (ctx->world == 1)
      CK(cudaMemcpyAsync(ctx->X[side][g] + ctx->rows[side] * ctx->k, R, (size_t)s * ctx->k * sizeof(double),
                         cudaMemcpyDeviceToDevice, st));
    else
      CK(shard_put_rows(st, R, s, ctx->k, ctx->rows[side], ctx->shard0 + g, ctx->world, ctx->block,
                        ctx->X[side][g]));
  }
  return TSVD_OK;
}

tsvd_opts default_opts() {
  tsvd_opts o;
  memset(&o, 0, sizeof(o));
  o.mode = TSVD_EXACT;
  o.l = 10;
  o.t = 3;
  o.reset_cond = 1e4;
  o.defl_tol = 1e-12;
  return o;
}

tsvd_opts resolve_opts(const tsvd_opts* in) {
  tsvd_opts o = in ? *in : default_opts();
  if (!(o.reset_cond > 0)) o.reset_cond = 1e4;
  if (!(o.defl_tol > 0)) o.defl_tol = 1e-12;
  return o;
}

void begin_stats(tsvd_ctx* ctx, cudaStream_t st, int64_t s, int64_t nnz, bool profile) {
  memset(&ctx->stats, 0, sizeof(ctx->stats));
  ctx->stats.s = s;
  ctx->stats.nnz = nnz;
  ctx->stats.rank[0] = ctx->stats.rank[1] = -1;
  ctx->stats.touched[0] = ctx->stats.touched[1] = -1;
  g_launches = 0;
  ctx->kprof.reset(st);
  g_prof = profile ? &ctx->kprof : nullptr;  // per-kernel events only when asked (flag bit 1)
  cudaEventRecord(ctx->ev[0], st);
}

// the phase times of the last update: resolved from its events when read (tsvd_last_stats) or
// right away in a profiling pass, so that an update returns without waiting for the device
void resolve_times(tsvd_ctx* ctx) {
  if (!ctx->times_pending) return;
  cudaEventSynchronize(ctx->ev[3]);
  float a = 0, b = 0, c = 0;
  cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
  cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]);
  cudaEventElapsedTime(&c, ctx->ev[2], ctx->ev[3]);
  ctx->stats.ms_pre = a;
  ctx->stats.ms_svd = b;
  ctx->stats.ms_post = c;
  ctx->stats.ms_total = a + b + c;
  ctx->times_pending = false;
}

bool pad_on() {  // TSVD_PAD=0: no even padding of the exact path's s (A/B tests)
  static const bool v = !(getenv("TSVD_PAD") && atoi(getenv("TSVD_PAD")) == 0);
  return v;
}
// TSVD_DEDUP=0: keep duplicate update vectors (only empty ones are dropped)
bool dedup_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TSVD_DEDUP");
    v = !(e && atoi(e) == 0);
  }
  return v == 1;
}

void end_stats(tsvd_ctx* ctx, cudaStream_t st) {
  cudaEventRecord(ctx->ev[3], st);
  ctx->stats.launches = (int32_t)g_launches;
  ctx->stats.total_resets = ctx->total_resets;
  ctx->times_pending = true;
  for (int c = 0; c < KC_N; ++c) {
    ctx->stats.kern_ms[c] = 0.0;
    ctx->stats.kern_flops[c] = 0.0;
    ctx->stats.kern_bytes[c] = 0.0;
    ctx->stats.kern_launches[c] = 0;
  }
  ctx->stats.top_class = 0;
  ctx->stats.top_launches = 0;
  ctx->stats.top_ms = ctx->stats.top_flops = ctx->stats.top_bytes = 0.0;
  if (!g_prof) return;  // phase times resolved when read
  resolve_times(ctx);
  ctx->kprof.resolve(ctx->stats.kern_ms, ctx->stats.kern_flops, ctx->stats.kern_bytes, ctx->stats.kern_launches);
  g_prof = nullptr;
  int top = 0;
  for (int c = 1; c < KC_N; ++c)
    if (ctx->stats.kern_ms[c] > ctx->stats.kern_ms[top]) top = c;
  ctx->stats.top_class = top;
  ctx->stats.top_launches = ctx->stats.kern_launches[top];
  ctx->stats.top_ms = ctx->stats.kern_ms[top];
  ctx->stats.top_flops = ctx->stats.kern_flops[top];
  ctx->stats.top_bytes = ctx->stats.kern_bytes[top];
}


bool opts_valid(tsvd_ctx* ctx, const tsvd_opts& o) {
  if (o.mode != TSVD_EXACT && o.mode != TSVD_RPI && o.mode != TSVD_GKL) {
    ctx->err = "unknown mode";
    return false;
  }
  if (o.mode != TSVD_EXACT && (o.l < 1 || (o.mode == TSVD_RPI && o.t < 1))) {
    ctx->err = "GKL/RPI need l >= 1 (and t >= 1 for RPI)";
    return false;
  }
  return true;
}

// Rows (lift = V side 1, append = U side 0) or columns (lift = U side 0, append = V side 1).
// Exact: Alg 9 / Alg 3.  RPI / GKL: App D.3.
tsvd_status update_append(tsvd_ctx* ctx, int lift_side, const tsvd_sparse* Ein, const tsvd_opts* opts_in,
                          cudaStream_t st) {
  if (!ctx->initialized) return set_err(ctx, TSVD_E_INVALID, "context not initialised");
  const tsvd_opts o = resolve_opts(opts_in);
  if (!opts_valid(ctx, o)) return TSVD_E_INVALID;
  const int app = 1 - lift_side, k = ctx->k;
  Scratch ws(st);
  int* d_flag = ws.alloc<int>(1);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, "scratch");
  CK(cudaMemsetAsync(d_flag, 0, sizeof(int), st));
  Lift L;
  L.side = lift_side;
  CKS(flush_pending(ctx, lift_side, st));  // the lift reads and updates X' rows
  begin_stats(ctx, st, 0, 0, (o.flags & 2) != 0);
  CKS(stage_sparse(ctx, Ein, ctx->rows[lift_side], ws, st, L.E, d_flag, !(o.flags & 1)));
  const int64_t s_in = L.E.s;
  ctx->stats.s = s_in;
  ctx->stats.nnz = L.E.nnz;
  if (s_in == 0) {  // no-op
    cudaEventRecord(ctx->ev[1], st);
    cudaEventRecord(ctx->ev[2], st);
    end_stats(ctx, st);
    return TSVD_OK;
  }
  // exact mode drops empty update vectors (their rows of U_new are zero)
  RowSel sel;
  if (o.mode == TSVD_EXACT) {
    DevCSR Ec;
    if (dedup_on()) CK(select_unique(st, L.E, Ec, sel, ws, ctx->h_i64));
    else CK(select_nonempty(st, L.E, nullptr, Ec, nullptr, sel, ws, ctx->h_i64));
    L.E = Ec;
  }
  const int64_t s_sel = L.E.s;
  ctx->stats.s_eff = s_sel;
  const bool compacted = o.mode == TSVD_EXACT && s_sel < s_in;
  // an odd s gets one empty update vector (deflated, no effect): even s x s leading dimensions
  if (o.mode == TSVD_EXACT && (s_sel & 1) && pad_on()) CK(pad_even_rows(st, L.E, ws));
  const int64_t s = L.E.s;
  if (s > 0) CKS(lift_any(ctx, L, o, o.sketch, lift_side, ws, st));
  const int64_t xr = s > 0 ? L.extra() : 0, mc = k + s, nc = k + xr;
  ctx->stats.rank[lift_side] = xr;
  ctx->stats.touched[lift_side] = L.nJ;
  // A5: core (col-major mc x nc), tall since r, l <= s:  [Σ, 0; C0^T, R_kept^T]  or  [Σ, 0; C0^T, P]
  double* K = ws.alloc<double>((size_t)mc * nc);
  double* theta = ws.alloc<double>(k + 1);
  double* F = ws.alloc<double>((size_t)mc * k);
  double* G = ws.alloc<double>((size_t)nc * k);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  if (L.mode == TSVD_EXACT)
    CK(build_core_rows(st, k, s, xr, ctx->Sigma, L.P0, L.R, L.kidx, K));
  else
    CK(build_core_approx(st, k, s, xr, ctx->Sigma, L.P0, L.Pa, K));
  cudaEventRecord(ctx->ev[1], st);
  CoreInfo ci;
  ci.hint = ctx->core_hint[lift_side];
  ci.growth = ctx->core_growth[lift_side];
  ci.thb2 = ctx->core_thb2[lift_side];
  ci.b_hint = ctx->core_b[lift_side];
  ci.defer_theta_next = true;  // read with the condition numbers below
  ci.theta_next_dst = ctx->h_f64 + 2;  // context-owned pinned word
  CoreShape shape{k, s, xr, L.mode == TSVD_EXACT ? L.kidx + s : nullptr};
  CK(core_svd(st, K, mc, mc, nc, k, theta, F, mc, G, nc, &ci, ws, nullptr, L.mode == TSVD_EXACT ? &shape : nullptr));
  if (ci.path == 2) {
    ctx->core_hint[lift_side] = ci.hint_next > 0 ? ci.hint_next : ci.iters;
    ctx->core_growth[lift_side] = ci.growth;
    ctx->core_thb2[lift_side] = ci.thb2;
    ctx->core_b[lift_side] = ci.b_next;
  }
  ctx->stats.jacobi_sweeps = ci.sweeps;
  ctx->stats.core_iters = ci.iters;
  ctx->stats.core_path = ci.path;
  ctx->stats.core_rows = (int32_t)mc;
  ctx->stats.core_cols = (int32_t)nc;
  if (!ci.converged) return set_err(ctx, TSVD_E_SVD_FAIL, "core SVD did not converge");
  ctx->stats.energy = ci.energy;
  ctx->stats.theta_next = ci.theta_next;
  cudaEventRecord(ctx->ev[2], st);
  // A6 append side: Y''_new = Y'' F[:k], its inverse and cond
  double* Mapp = ws.alloc<double>((size_t)k * k);
  double* Mapp_inv = ws.alloc<double>((size_t)k * k);
  double* cond_app = ws.alloc<double>(1);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  CK(dgemm(st, k, k, k, 1.0, CMat{ctx->M[app], k, 1}, CMat{F, 1, mc}, 0.0, Mat{Mapp, k, 1}, 0));
  CK(inverse_gj(st, Mapp, k, Mapp_inv, cond_app, ws));
  // A6 lift side (G is the lift side's singular-vector block)
  LiftPost P;
  CKS(lift_post(ctx, L, G, nc, P, ws, st));
  CK(cudaMemcpyAsync(ctx->h_f64, cond_app, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ctx->h_f64 + 1, P.cond, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double capp = ctx->h_f64[0], clift = ctx->h_f64[1];
  if (ci.theta_next_host) ctx->stats.theta_next = *ci.theta_next_host;
  ctx->stats.cond[app] = capp;
  ctx->stats.cond[lift_side] = clift;
  bool rs[2];
  {
    const double* Ms[2] = {Mapp, P.Mnew};
    const double* Mi[2] = {Mapp_inv, P.Minv};
    const double c1[2] = {capp, clift};
    CKS(mii_decide(ctx, 2, Ms, Mi, c1, o.reset_cond, rs, ws, st));
  }
  const bool reset_app = rs[0], reset_lift = rs[1];
  // ---- commit
  CKS(ensure_cap(ctx, app, ctx->rows[app] + s_in, st));
  double* newrows = ws.alloc<double>((size_t)std::max<int64_t>(s, 1) * k);
  double* newfull = compacted ? ws.alloc<double>((size_t)s_in * k) : newrows;
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  if (!reset_app) {
    CK(dgemm(st, s, k, k, 1.0, CMat{F + k, 1, mc}, CMat{Mapp_inv, k, 1}, 0.0, Mat{newrows, k, 1}, 0));
    CK(cudaMemcpyAsync(ctx->M[app], Mapp, (size_t)k * k * sizeof(double), cudaMemcpyDeviceToDevice, st));
  } else {
    // MII reset of the append side, deferred (an append side is only ever written, until it
    // is read as a whole or lifted): the existing rows keep X' and record P = Mapp (earlier
    // pending blocks: P <- P Mapp) instead of the m x k x k materialisation (C5: 18M x 256,
    // ~100 ms); at most 16 pending blocks
    if (ctx->pend[app].size() >= 16) CKS(flush_pending(ctx, app, st));
    for (auto& b : ctx->pend[app]) {
      double* np = nullptr;
      CK(cudaMallocAsync(&np, (size_t)k * k * sizeof(double), st));
      CK(dgemm_rm(st, false, false, k, k, k, 1.0, b.P, k, Mapp, k, 0.0, np, k));
      CK(cudaFreeAsync(b.P, st));
      b.P = np;
    }
    const int64_t r0 = ctx->pend[app].empty() ? 0 : ctx->pend[app].back().r1, r1 = ctx->rows[app];
    if (r1 > r0) {
      double* np = nullptr;
      CK(cudaMallocAsync(&np, (size_t)k * k * sizeof(double), st));
      CK(cudaMemcpyAsync(np, Mapp, (size_t)k * k * sizeof(double), cudaMemcpyDeviceToDevice, st));
      ctx->pend[app].push_back({r0, r1, np});
    }
    CK(colmajor_to_rowmajor(st, F + k, mc, s, k, newrows, k));
    CK(set_identity(st, ctx->M[app], k));
  }
  if (compacted) CK(expand_selected(st, sel, newrows, k, newfull));
  CKS(append_rows(ctx, app, newfull, s_in, st));
  CKS(lift_commit(ctx, L, P, reset_lift, ws, st));
  CK(cudaMemcpyAsync(ctx->Sigma, theta, k * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (nc < k) CK(cudaMemsetAsync(ctx->Sigma + nc, 0, (k - nc) * sizeof(double), st));
  ctx->rows[app] += s_in;
  ctx->stats.reset[app] = reset_app;
  ctx->stats.reset[lift_side] = reset_lift;
  ctx->total_resets += (int)reset_app + (int)reset_lift;
  end_stats(ctx, st);
  return TSVD_OK;
}

// Alg 4 (R2 fix) exact; App D.3 'update weights' for RPI / GKL.
tsvd_status update_weights_impl(tsvd_ctx* ctx, const tsvd_sparse* DT, const tsvd_sparse* EmT, const tsvd_opts* opts_in,
                                cudaStream_t st) {
  if (!ctx->initialized) return set_err(ctx, TSVD_E_INVALID, "context not initialised");
  const tsvd_opts o = resolve_opts(opts_in);
  if (!opts_valid(ctx, o)) return TSVD_E_INVALID;
  if (!DT || !EmT) return set_err(ctx, TSVD_E_INVALID, "null sparse block");
  if (DT->s != EmT->s) return set_err(ctx, TSVD_E_SHAPE, "D and E_m have different s");
  const int k = ctx->k;
  Scratch ws(st);
  int* d_flag = ws.alloc<int>(1);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, "scratch");
  CK(cudaMemsetAsync(d_flag, 0, sizeof(int), st));
  Lift LD, LE;
  LD.side = 0;
  LE.side = 1;
  CKS(flush_pending(ctx, 0, st));
  CKS(flush_pending(ctx, 1, st));
  begin_stats(ctx, st, 0, 0, (o.flags & 2) != 0);
  CKS(stage_sparse(ctx, DT, ctx->rows[0], ws, st, LD.E, d_flag, !(o.flags & 1)));
  CKS(stage_sparse(ctx, EmT, ctx->rows[1], ws, st, LE.E, d_flag, !(o.flags & 1)));
  ctx->stats.s = LD.E.s;
  ctx->stats.nnz = LD.E.nnz + LE.E.nnz;
  if (LD.E.s == 0) {
    cudaEventRecord(ctx->ev[1], st);
    cudaEventRecord(ctx->ev[2], st);
    end_stats(ctx, st);
    return TSVD_OK;
  }
  if (o.mode == TSVD_EXACT) {  // d_i e_i^T = 0 when either is empty: drop the pair
    RowSel sel;
    DevCSR Dc, Ec;
    CK(select_nonempty(st, LD.E, &LE.E, Dc, &Ec, sel, ws, ctx->h_i64));
    LD.E = Dc;
    LE.E = Ec;
  }
  const int64_t s = LD.E.s;
  ctx->stats.s_eff = s;
  const int64_t blk = (o.mode == TSVD_RPI) ? s * (int64_t)o.l : s;  // per-side start block
  const double* skD = o.sketch;
  const double* skE = o.sketch ? o.sketch + blk : nullptr;
  // The two sides' approximate augmented spaces are independent: the E side runs on the
  // context's second stream (its own stream-ordered scratch), joined before the core.  Not in
  // the profiling pass (per-class events are recorded on the update's stream), not with NCCL
  // (both sides' all-reduces must be issued in the same order on every rank), not in exact
  // mode (its lifts synchronise with the host for the kept rank).
  const bool overlap = o.mode != TSVD_EXACT && ctx->world == 1 && !(o.flags & 2) && s > 0;
  cudaStream_t st2 = st;
  if (overlap) {
    if (!ctx->side) {
      CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
    }
    st2 = ctx->side;
    CK(cudaEventRecord(ctx->fork_ev, st));
    CK(cudaStreamWaitEvent(st2, ctx->fork_ev, 0));
  }
  Scratch ws2(st2);
  // (declared after ws2, so destroyed before it: st2 frees the E side's buffers only after
  // everything enqueued on st — the core, the updates — that reads them)
  struct Rejoin {
    cudaStream_t a, b;
    cudaEvent_t ev;
    ~Rejoin() {
      if (a != b) {
        cudaEventRecord(ev, a);
        cudaStreamWaitEvent(b, ev, 0);
      }
    }
  } rejoin{st, st2, ctx->join_ev};
  if (s > 0) {
    CKS(lift_any(ctx, LD, o, skD, 0, ws, st));
    CKS(lift_any(ctx, LE, o, skE, 1, overlap ? ws2 : ws, st2));
    if (overlap) {
      CK(cudaEventRecord(ctx->join_ev, st2));
      CK(cudaStreamWaitEvent(st, ctx->join_ev, 0));
    }
  }
  ctx->stats.rank[0] = LD.extra();
  ctx->stats.rank[1] = LE.extra();
  ctx->stats.touched[0] = LD.nJ;
  ctx->stats.touched[1] = LE.nJ;
  const int64_t nD = k + LD.extra(), nE = k + LE.extra();
  // core, tall orientation: rows = the larger of nD, nE
  const bool tr = nE > nD;
  const int64_t mc = tr ? nE : nD, nc = tr ? nD : nE;
  double* K = ws.alloc<double>((size_t)mc * nc);
  double* theta = ws.alloc<double>(k + 1);
  double* F = ws.alloc<double>((size_t)mc * k);
  double* G = ws.alloc<double>((size_t)nc * k);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  if (LD.mode == TSVD_EXACT) {
    double* BD = ws.alloc<double>((size_t)nD * s);
    double* BE = ws.alloc<double>((size_t)nE * s);
    if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
    CK(build_lift_block(st, k, s, LD.r, LD.P0, LD.R, LD.kidx, BD));
    CK(build_lift_block(st, k, s, LE.r, LE.P0, LE.R, LE.kidx, BE));
    const double* BL = tr ? BE : BD;  // left factor rows
    const double* BR = tr ? BD : BE;
    // K(i, j) = sum_c BL(i, c) BR(j, c), column-major
    CK(dgemm(st, mc, nc, s, 1.0, CMat{BL, s, 1}, CMat{BR, 1, s}, 0.0, Mat{K, 1, mc}, 0));
  } else {
    // K = [C0_L; P_L^T] [C0_R; P_R^T]^T (App D.3) by its 2 x 2 blocks, the operands read in place
    // from the s x k / s x l row-major P0 and P (no (k + l) x s transposed copies: 2 x 220 us of
    // strided copy kernels per configs[3] update)
    const Lift& LL = tr ? LE : LD;
    const Lift& LR = tr ? LD : LE;
    const int64_t rl[2] = {k, LL.l}, rr[2] = {k, LR.l};
    const CMat Ab[2] = {CMat{LL.P0, 1, k}, CMat{LL.Pa, 1, LL.l}};
    const CMat Bb[2] = {CMat{LR.P0, k, 1}, CMat{LR.Pa, LR.l, 1}};
    for (int bi = 0; bi < 2; ++bi)
      for (int bj = 0; bj < 2; ++bj) {
        const int64_t i0 = bi ? k : 0, j0 = bj ? k : 0;
        if (rl[bi] > 0 && rr[bj] > 0)
          CK(dgemm(st, rl[bi], rr[bj], s, 1.0, Ab[bi], Bb[bj], 0.0, Mat{K + i0 + j0 * mc, 1, mc}, 0));
      }
  }
  CK(add_diag_sigma(st, K, mc, k, ctx->Sigma, true));
  cudaEventRecord(ctx->ev[1], st);
  CoreInfo ci;
  ci.hint = ctx->core_hint[2];
  ci.growth = ctx->core_growth[2];
  ci.thb2 = ctx->core_thb2[2];
  ci.b_hint = ctx->core_b[2];
  CK(core_svd(st, K, mc, mc, nc, k, theta, F, mc, G, nc, &ci, ws));
  if (ci.path == 2) {
    ctx->core_hint[2] = ci.hint_next > 0 ? ci.hint_next : ci.iters;
    ctx->core_growth[2] = ci.growth;
    ctx->core_thb2[2] = ci.thb2;
    ctx->core_b[2] = ci.b_next;
  }
  ctx->stats.jacobi_sweeps = ci.sweeps;
  ctx->stats.core_iters = ci.iters;
  ctx->stats.core_path = ci.path;
  ctx->stats.core_rows = (int32_t)mc;
  ctx->stats.core_cols = (int32_t)nc;
  if (!ci.converged) return set_err(ctx, TSVD_E_SVD_FAIL, "core SVD did not converge");
  ctx->stats.energy = ci.energy;
  ctx->stats.theta_next = ci.theta_next;
  cudaEventRecord(ctx->ev[2], st);
  const double* FU = tr ? G : F;
  const int64_t ldU = tr ? nc : mc;
  const double* GV = tr ? F : G;
  const int64_t ldV = tr ? mc : nc;
  LiftPost PD, PE;
  // the two sides' multipliers and their inverses (small GEMMs + one single-CTA Gauss-Jordan
  // each) are independent: the E side again on the second stream
  if (overlap) {
    CK(cudaEventRecord(ctx->fork_ev, st));
    CK(cudaStreamWaitEvent(st2, ctx->fork_ev, 0));
  }
  CKS(lift_post(ctx, LD, FU, ldU, PD, ws, st));
  CKS(lift_post(ctx, LE, GV, ldV, PE, overlap ? ws2 : ws, st2));
  if (overlap) {
    CK(cudaEventRecord(ctx->join_ev, st2));
    CK(cudaStreamWaitEvent(st, ctx->join_ev, 0));
  }
  CK(cudaMemcpyAsync(ctx->h_f64, PD.cond, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ctx->h_f64 + 1, PE.cond, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double cu = ctx->h_f64[0], cv = ctx->h_f64[1];
  ctx->stats.cond[0] = cu;
  ctx->stats.cond[1] = cv;
  bool rs[2];
  {
    const double* Ms[2] = {PD.Mnew, PE.Mnew};
    const double* Mi[2] = {PD.Minv, PE.Minv};
    const double c1[2] = {cu, cv};
    CKS(mii_decide(ctx, 2, Ms, Mi, c1, o.reset_cond, rs, ws, st));
  }
  const bool ru = rs[0], rv = rs[1];
  if (overlap) {  // the commits (X'[J] += B' Z, the multiplier or its reset) per side as well
    CK(cudaEventRecord(ctx->fork_ev, st));
    CK(cudaStreamWaitEvent(st2, ctx->fork_ev, 0));
  }
  CKS(lift_commit(ctx, LD, PD, ru, ws, st));
  CKS(lift_commit(ctx, LE, PE, rv, overlap ? ws2 : ws, st2));
  if (overlap) {
    CK(cudaEventRecord(ctx->join_ev, st2));
    CK(cudaStreamWaitEvent(st, ctx->join_ev, 0));
  }
  CK(cudaMemcpyAsync(ctx->Sigma, theta, k * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (nc < k) CK(cudaMemsetAsync(ctx->Sigma + nc, 0, (k - nc) * sizeof(double), st));
  ctx->stats.reset[0] = ru;
  ctx->stats.reset[1] = rv;
  ctx->total_resets += (int)ru + (int)rv;
  end_stats(ctx, st);
  return TSVD_OK;
}

tsvd_status get_factor(tsvd_ctx* ctx, int side, double* out, cudaStream_t st) {
  if (!ctx->initialized) return set_err(ctx, TSVD_E_INVALID, "context not initialised");
  if (!out) return set_err(ctx, TSVD_E_INVALID, "null output");
  CKS(flush_pending(ctx, side, st));
  const int k = ctx->k;
  const int64_t rows = ctx->rows[side];
  if (rows == 0) return TSVD_OK;
  Scratch ws(st);
  const bool dev = is_device_ptr(out);
  double* dst = dev ? out : ws.alloc<double>((size_t)rows * k);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  if (ctx->world == 1) {
    CK(dgemm_rm(st, false, false, rows, k, k, 1.0, ctx->X[side][0], k, ctx->M[side], k, 0.0, dst, k));
  } else if (ctx->comm) {
    // NCCL mode: every process materialises its own rows into a block of maxl rows; one
    // all-gather (m k doubles received per process — an all-reduce of the zero-padded factor
    // would move twice that) and a row permutation place them at their global positions
    const int64_t maxl = shard_rows(rows, 0, ctx->world, ctx->block);  // shard 0 holds the most rows
    double* mine = ws.alloc<double>((size_t)std::max<int64_t>(maxl, 1) * k);
    double* all = ws.alloc<double>((size_t)std::max<int64_t>(maxl, 1) * k * ctx->world);
    if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
    const int64_t lr = lrows(ctx, side, 0);
    if (lr) CK(dgemm_rm(st, false, false, lr, k, k, 1.0, ctx->X[side][0], k, ctx->M[side], k, 0.0, mine, k));
    const int rc = nccl_allgather_f64(ctx->comm, mine, all, maxl * k, st);
    if (rc != 0) return set_err(ctx, TSVD_E_NCCL, std::string("ncclAllGather: ") + nccl_error(rc));
    CK(shard_unshuffle(st, all, rows, maxl, k, ctx->world, ctx->block, dst));
  } else {
    // virtual shards: each materialises its rows into their global positions
    CK(cudaMemsetAsync(dst, 0, (size_t)rows * k * sizeof(double), st));
    for (int g = 0; g < ctx->nloc; ++g) {
      const int64_t lr = lrows(ctx, side, g);
      double* tmp = ws.alloc<double>((size_t)std::max<int64_t>(lr, 1) * k);
      if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
      if (lr) CK(dgemm_rm(st, false, false, lr, k, k, 1.0, ctx->X[side][g], k, ctx->M[side], k, 0.0, tmp, k));
      CK(shard_scatter_owned(st, tmp, rows, k, ctx->shard0 + g, ctx->world, ctx->block, dst));
    }
  }
  if (!dev) {
    CK(cudaMemcpyAsync(out, dst, (size_t)rows * k * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return TSVD_OK;
}

std::string g_create_err;  // why the last tsvd_create* failed (tsvd_last_error(NULL))

tsvd_status create_impl(tsvd_ctx** out, int32_t device, int world, int rank, int nvirt, int block, const void* id,
                        int64_t m_capacity, int64_t n_capacity, int32_t k) {
  if (!out || k <= 0 || k > 1024 || m_capacity < 0 || n_capacity < 0 || world < 1) return TSVD_E_INVALID;
  if (world > 1 && !(nvirt == world || (nvirt == 1 && rank >= 0 && rank < world && id))) return TSVD_E_INVALID;
  if (world == 1 && nvirt != 1) return TSVD_E_INVALID;
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return TSVD_E_CUDA;
  tsvd_ctx* ctx = new tsvd_ctx();
  ctx->device = device;
  ctx->k = k;
  ctx->world = world;
  ctx->nloc = world == 1 ? 1 : nvirt;
  ctx->shard0 = (world > 1 && nvirt == 1) ? rank : 0;
  ctx->block = block > 0 ? block : 1024;
  // keep freed scratch in the stream-ordered pool between updates
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  bool ok = cudaMallocHost(&ctx->h_i64, 64 * sizeof(int64_t)) == cudaSuccess &&
            cudaMallocHost(&ctx->h_f64, 64 * sizeof(double)) == cudaSuccess;
  for (int i = 0; i < 4 && ok; ++i) ok = cudaEventCreate(&ctx->ev[i]) == cudaSuccess;
  for (int s = 0; s < 2 && ok; ++s) ok = cudaMalloc(&ctx->M[s], (size_t)k * k * sizeof(double)) == cudaSuccess;
  ok = ok && cudaMalloc(&ctx->Sigma, (size_t)k * sizeof(double)) == cudaSuccess;
  const int64_t caps[2] = {std::max<int64_t>(m_capacity, 1), std::max<int64_t>(n_capacity, 1)};
  for (int s = 0; s < 2; ++s) {
    ctx->X[s].assign(ctx->nloc, nullptr);
    ctx->cap[s].assign(ctx->nloc, 0);
    for (int g = 0; g < ctx->nloc && ok; ++g) {
      const int64_t c = std::max<int64_t>(lrows(ctx, s, g, caps[s]), 1);
      ok = cudaMalloc(&ctx->X[s][g], (size_t)c * k * sizeof(double)) == cudaSuccess;
      ctx->cap[s][g] = c;
    }
  }
  tsvd_status rc = ok ? TSVD_OK : TSVD_E_OOM;
  // NCCL mode (a 1-rank communicator when world == 1: the same code path, an identity sum)
  if (ok && id && nvirt == 1) {
    const int e = nccl_comm_init(&ctx->comm, world, id, rank);
    if (e != 0) {
      ctx->comm = nullptr;
      rc = TSVD_E_NCCL;
      g_create_err = std::string("ncclCommInitRank: ") + nccl_error(e) + " (rc " + std::to_string(e) + ")";
    }
  }
  if (rc != TSVD_OK) {
    tsvd_destroy(ctx);
    cudaGetLastError();
    return rc;
  }
  *out = ctx;
  return TSVD_OK;
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

const char* tsvd_version(void) { return "tsvd-b200 0.1 (sm_100a, fp64)"; }

tsvd_status tsvd_create(tsvd_ctx** out, int32_t device, int64_t m_capacity, int64_t n_capacity, int32_t k) {
  return create_impl(out, device, 1, 0, 1, 0, nullptr, m_capacity, n_capacity, k);
}

tsvd_status tsvd_create_sharded(tsvd_ctx** out, int32_t device, const tsvd_shard_opts* so, int64_t m_capacity,
                                int64_t n_capacity, int32_t k) {
  if (!so) return TSVD_E_INVALID;
  return create_impl(out, device, so->world, so->rank, so->virtual_shards, so->block, so->nccl_id, m_capacity,
                     n_capacity, k);
}

tsvd_status tsvd_shard_owner(int64_t i, int32_t world, int32_t block, int32_t* shard, int64_t* local) {
  if (i < 0 || world < 1 || block < 1) return TSVD_E_INVALID;
  if (shard) *shard = (int32_t)((i / block) % world);
  if (local) *local = (i / ((int64_t)block * world)) * block + i % block;
  return TSVD_OK;
}

tsvd_status tsvd_shard_split_host(const tsvd_sparse* E, int32_t world, int32_t block, int32_t shard, int64_t* row_ptr,
                                  int32_t* col_idx, double* val, int64_t* nnz) {
  if (!E || world < 1 || block < 1 || shard < 0 || shard >= world || !nnz) return TSVD_E_INVALID;
  if (E->s > 0 && !E->row_ptr) return TSVD_E_INVALID;
  int64_t q = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (int64_t r = 0; r < E->s; ++r) {
    for (int64_t p = E->row_ptr[r]; p < E->row_ptr[r + 1]; ++p) {
      const int64_t c = E->col_idx[p];
      if ((c / block) % world != shard) continue;
      if (col_idx) col_idx[q] = (int32_t)((c / ((int64_t)block * world)) * block + c % block);
      if (val) val[q] = E->val[p];
      ++q;
    }
    if (row_ptr) row_ptr[r + 1] = q;
  }
  *nnz = q;
  return TSVD_OK;
}

tsvd_status tsvd_nccl_unique_id(void* out128) {
  if (!out128) return TSVD_E_INVALID;
  return nccl_unique_id(out128) == 0 ? TSVD_OK : TSVD_E_NCCL;
}

void tsvd_destroy(tsvd_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  drop_pending(ctx);
  for (int s = 0; s < 2; ++s) {
    for (double* p : ctx->X[s])
      if (p) cudaFree(p);
    if (ctx->M[s]) cudaFree(ctx->M[s]);
  }
  if (ctx->Sigma) cudaFree(ctx->Sigma);
  if (ctx->h_i64) cudaFreeHost(ctx->h_i64);
  if (ctx->h_f64) cudaFreeHost(ctx->h_f64);
  for (int i = 0; i < 4; ++i)
    if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
  if (ctx->comm) nccl_comm_destroy(ctx->comm);
  delete ctx;
}

const char* tsvd_last_error(const tsvd_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

tsvd_status tsvd_init(tsvd_ctx* ctx, int64_t m, int64_t n, const double* U, const double* S, const double* V,
                      void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int k = ctx->k;
  if (m < k || n < k) return set_err(ctx, TSVD_E_SHAPE, "need m >= k and n >= k");
  if (!U || !S || !V) return set_err(ctx, TSVD_E_INVALID, "null factor");
  cudaStreamSynchronize(st);
  drop_pending(ctx);
  CKS(ensure_cap(ctx, 0, m, st));
  CKS(ensure_cap(ctx, 1, n, st));
  Scratch ws(st);
  cudaError_t e = cudaSuccess;
  const double* dU = stage(U, (size_t)m * k, ws, st, &e);
  if (e) return set_err(ctx, TSVD_E_CUDA, cudaGetErrorString(e));
  const double* dV = stage(V, (size_t)n * k, ws, st, &e);
  if (e) return set_err(ctx, TSVD_E_CUDA, cudaGetErrorString(e));
  std::vector<double> hs(k);
  if (is_device_ptr(S)) {
    CK(cudaMemcpyAsync(hs.data(), S, k * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  } else {
    memcpy(hs.data(), S, k * sizeof(double));
  }
  for (int i = 0; i < k; ++i) {
    if (!std::isfinite(hs[i])) return set_err(ctx, TSVD_E_NUMERIC, "non-finite sigma");
    if (hs[i] < 0 || (i > 0 && hs[i] > hs[i - 1])) return set_err(ctx, TSVD_E_BAD_SIGMA, "sigma not descending / >= 0");
  }
  double* dev = ws.alloc<double>(2);
  int* flag = ws.alloc<int>(1);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, "scratch");
  CK(cudaMemsetAsync(flag, 0, sizeof(int), st));
  CK(find_nonfinite(st, dU, m * k, flag));
  CK(find_nonfinite(st, dV, n * k, flag));
  CK(check_init(st, dU, m, k, dev, ws));
  CK(check_init(st, dV, n, k, dev + 1, ws));
  CK(cudaMemcpyAsync(ctx->h_f64, dev, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ctx->h_i64, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (*reinterpret_cast<int*>(ctx->h_i64)) return set_err(ctx, TSVD_E_NUMERIC, "non-finite factor entry");
  if (!(ctx->h_f64[0] <= 1e-10) || !(ctx->h_f64[1] <= 1e-10))
    return set_err(ctx, TSVD_E_NOT_ORTHONORMAL, "||X^T X - I||_max > 1e-10");
  ctx->rows[0] = 0;
  ctx->rows[1] = 0;
  for (int g = 0; g < ctx->nloc; ++g) {
    if (dU != ctx->X[0][g]) CK(shard_gather_owned(st, dU, m, k, ctx->shard0 + g, ctx->world, ctx->block, ctx->X[0][g]));
    if (dV != ctx->X[1][g]) CK(shard_gather_owned(st, dV, n, k, ctx->shard0 + g, ctx->world, ctx->block, ctx->X[1][g]));
  }
  CK(cudaMemcpyAsync(ctx->Sigma, hs.data(), k * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(set_identity(st, ctx->M[0], k));
  CK(set_identity(st, ctx->M[1], k));
  CK(cudaStreamSynchronize(st));
  ctx->rows[0] = m;
  ctx->rows[1] = n;
  ctx->initialized = true;
  ctx->total_resets = 0;
  return TSVD_OK;
}

tsvd_status tsvd_init_sparse(tsvd_ctx* ctx, const tsvd_sparse* A, int32_t oversample, int32_t power_iters,
                             uint64_t seed, void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int k = ctx->k;
  if (!A) return set_err(ctx, TSVD_E_INVALID, "null sparse matrix");
  if (power_iters < 0 || power_iters > 64) return set_err(ctx, TSVD_E_INVALID, "power_iters out of [0, 64]");
  cudaStreamSynchronize(st);
  drop_pending(ctx);
  const int64_t m = A->s, n = A->dim;
  int p = ((k + std::max(oversample, 0) + 15) / 16) * 16;
  p = std::min<int>(p, 512);
  if (m < p || n < p || p < k) return set_err(ctx, TSVD_E_SHAPE, "need m, n >= k + oversample (rounded to 16) <= 512");
  Scratch ws(st);
  int* d_flag = ws.alloc<int>(1);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, "scratch");
  CK(cudaMemsetAsync(d_flag, 0, sizeof(int), st));
  DevCSR dA;
  CKS(stage_sparse(ctx, A, n, ws, st, dA, d_flag, true));
  // unsharded: the factors are written straight into the context's U', V' (at configs[4] size a
  // scratch U would be another 37 GB next to the 39 GB range basis); the state is marked
  // uninitialised until the validation of tsvd_init's rules has passed
  const bool direct = ctx->world == 1;
  if (direct) {
    ctx->initialized = false;
    CKS(ensure_cap(ctx, 0, m, st));
    CKS(ensure_cap(ctx, 1, n, st));
  }
  double* U = direct ? ctx->X[0][0] : ws.alloc<double>((size_t)m * k);
  double* S = ws.alloc<double>(k);
  double* V = direct ? ctx->X[1][0] : ws.alloc<double>((size_t)n * k);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  int sw = 0;
  bool conv = false;
  const cudaError_t e = randomized_svd(st, dA, k, p, power_iters, seed, U, S, V, ws, &sw, &conv);
  if (e == cudaErrorInvalidValue) return set_err(ctx, TSVD_E_SHAPE, "A touches fewer than k + oversample columns");
  CK(e);
  if (!conv) return set_err(ctx, TSVD_E_SVD_FAIL, "Jacobi of the projected matrix did not converge");
  return tsvd_init(ctx, m, n, U, S, V, stream);
}

tsvd_status tsvd_update_rows(tsvd_ctx* ctx, const tsvd_sparse* Er, const tsvd_opts* opts, void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  cudaSetDevice(ctx->device);
  return update_append(ctx, 1, Er, opts, (cudaStream_t)stream);
}

tsvd_status tsvd_update_cols(tsvd_ctx* ctx, const tsvd_sparse* EcT, const tsvd_opts* opts, void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  cudaSetDevice(ctx->device);
  return update_append(ctx, 0, EcT, opts, (cudaStream_t)stream);
}

tsvd_status tsvd_update_weights(tsvd_ctx* ctx, const tsvd_sparse* DT, const tsvd_sparse* EmT, const tsvd_opts* opts,
                                void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  cudaSetDevice(ctx->device);
  return update_weights_impl(ctx, DT, EmT, opts, (cudaStream_t)stream);
}

tsvd_status tsvd_get_U(tsvd_ctx* ctx, double* out, void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  cudaSetDevice(ctx->device);
  return get_factor(ctx, 0, out, (cudaStream_t)stream);
}

tsvd_status tsvd_get_V(tsvd_ctx* ctx, double* out, void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  cudaSetDevice(ctx->device);
  return get_factor(ctx, 1, out, (cudaStream_t)stream);
}

tsvd_status tsvd_get_S(tsvd_ctx* ctx, double* out, void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  if (!ctx->initialized) return set_err(ctx, TSVD_E_INVALID, "context not initialised");
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(out, ctx->Sigma, ctx->k * sizeof(double), cudaMemcpyDefault, st));
  CK(cudaStreamSynchronize(st));
  return TSVD_OK;
}

tsvd_status tsvd_query_row(tsvd_ctx* ctx, int32_t side, int64_t i, double* out, void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  if (!ctx->initialized) return set_err(ctx, TSVD_E_INVALID, "context not initialised");
  if (side != 0 && side != 1) return set_err(ctx, TSVD_E_INVALID, "side must be 0 (U) or 1 (V)");
  if (i < 0 || i >= ctx->rows[side]) return set_err(ctx, TSVD_E_OOB, "row index out of range");
  if (!out) return set_err(ctx, TSVD_E_INVALID, "null output");
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int k = ctx->k;
  Scratch ws(st);
  const bool dev = is_device_ptr(out);
  double* dst = dev ? out : ws.alloc<double>(k);
  double* tmp = ws.alloc<double>((size_t)k * k);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, "scratch");
  const double* Mi = nullptr;
  CKS(row_multiplier(ctx, side, i, tmp, &Mi, st));
  if (ctx->world == 1) {
    CK(dgemm_rm(st, false, false, 1, k, k, 1.0, ctx->X[side][0] + i * k, k, Mi, k, 0.0, dst, k));
  } else {
    // the owner computes the row (O(k^2)); in NCCL mode it broadcasts it to the others
    const int owner = (int)((i / ctx->block) % ctx->world);
    const int64_t li = (i / ((int64_t)ctx->block * ctx->world)) * ctx->block + i % ctx->block;
    for (int g = 0; g < ctx->nloc; ++g)
      if (ctx->shard0 + g == owner)
        CK(dgemm_rm(st, false, false, 1, k, k, 1.0, ctx->X[side][g] + li * k, k, Mi, k, 0.0, dst, k));
    if (ctx->comm) {
      const int rc = nccl_broadcast_f64(ctx->comm, dst, dst, k, owner, st);
      if (rc != 0) return set_err(ctx, TSVD_E_NCCL, std::string("ncclBroadcast: ") + nccl_error(rc));
    }
  }
  if (!dev) CK(cudaMemcpyAsync(out, dst, k * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return TSVD_OK;
}

tsvd_status tsvd_query_row_local(tsvd_ctx* ctx, int32_t side, int64_t i, double* out, void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  if (!ctx->initialized) return set_err(ctx, TSVD_E_INVALID, "context not initialised");
  if (side != 0 && side != 1) return set_err(ctx, TSVD_E_INVALID, "side must be 0 (U) or 1 (V)");
  if (i < 0 || i >= ctx->rows[side]) return set_err(ctx, TSVD_E_OOB, "row index out of range");
  if (!out) return set_err(ctx, TSVD_E_INVALID, "null output");
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int k = ctx->k;
  const int owner = ctx->world == 1 ? 0 : (int)((i / ctx->block) % ctx->world);
  const int g = owner - ctx->shard0;
  if (g < 0 || g >= ctx->nloc) return set_err(ctx, TSVD_E_NOT_LOCAL, "row owned by shard " + std::to_string(owner));
  const int64_t li = ctx->world == 1 ? i : (i / ((int64_t)ctx->block * ctx->world)) * ctx->block + i % ctx->block;
  Scratch ws(st);
  const bool dev = is_device_ptr(out);
  double* dst = dev ? out : ws.alloc<double>(k);
  double* tmp = ws.alloc<double>((size_t)k * k);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, "scratch");
  const double* Mi = nullptr;
  CKS(row_multiplier(ctx, side, i, tmp, &Mi, st));
  CK(dgemm_rm(st, false, false, 1, k, k, 1.0, ctx->X[side][g] + li * k, k, Mi, k, 0.0, dst, k));
  if (!dev) CK(cudaMemcpyAsync(out, dst, k * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return TSVD_OK;
}

static tsvd_status tsvd_get_shard(tsvd_ctx* ctx, int32_t side, int32_t local_shard, double* out, int64_t* global_rows,
                           int64_t* nrows, void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  if (!ctx->initialized) return set_err(ctx, TSVD_E_INVALID, "context not initialised");
  if (side != 0 && side != 1) return set_err(ctx, TSVD_E_INVALID, "side must be 0 (U) or 1 (V)");
  if (local_shard < 0 || local_shard >= ctx->nloc) return set_err(ctx, TSVD_E_INVALID, "no such local shard");
  if (!nrows) return set_err(ctx, TSVD_E_INVALID, "null nrows");
  cudaSetDevice(ctx->device);
  if (out) CKS(flush_pending(ctx, side, (cudaStream_t)stream));
  const int64_t lr = lrows(ctx, side, local_shard);
  *nrows = lr;
  const int g = ctx->shard0 + local_shard;
  if (global_rows)
    for (int64_t j = 0; j < lr; ++j)
      global_rows[j] = ctx->world == 1 ? j : shard_global_row(j, g, ctx->world, ctx->block);
  if (!out || lr == 0) return TSVD_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int k = ctx->k;
  Scratch ws(st);
  const bool dev = is_device_ptr(out);
  double* dst = dev ? out : ws.alloc<double>((size_t)lr * k);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  CK(dgemm_rm(st, false, false, lr, k, k, 1.0, ctx->X[side][local_shard], k, ctx->M[side], k, 0.0, dst, k));
  if (!dev) {
    CK(cudaMemcpyAsync(out, dst, (size_t)lr * k * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return TSVD_OK;
}

tsvd_status tsvd_get_U_shard(tsvd_ctx* ctx, int32_t local_shard, double* out, int64_t* global_rows, int64_t* nrows,
                             void* stream) {
  return tsvd_get_shard(ctx, 0, local_shard, out, global_rows, nrows, stream);
}

tsvd_status tsvd_get_V_shard(tsvd_ctx* ctx, int32_t local_shard, double* out, int64_t* global_rows, int64_t* nrows,
                             void* stream) {
  return tsvd_get_shard(ctx, 1, local_shard, out, global_rows, nrows, stream);
}

tsvd_status tsvd_score_pairs(tsvd_ctx* ctx, int64_t n, const int64_t* rows, const int64_t* cols, double* out,
                             void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  if (!ctx->initialized) return set_err(ctx, TSVD_E_INVALID, "context not initialised");
  if (ctx->world > 1) return set_err(ctx, TSVD_E_UNSUPPORTED, "score_pairs on a sharded context");
  if (n < 0 || (n > 0 && (!rows || !cols || !out))) return set_err(ctx, TSVD_E_INVALID, "null pair arrays");
  if (n == 0) return TSVD_OK;
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  Scratch ws(st);
  cudaError_t e = cudaSuccess;
  const int64_t* dr = stage(rows, (size_t)n, ws, st, &e);
  if (e) return set_err(ctx, TSVD_E_CUDA, cudaGetErrorString(e));
  const int64_t* dc = stage(cols, (size_t)n, ws, st, &e);
  if (e) return set_err(ctx, TSVD_E_CUDA, cudaGetErrorString(e));
  int* flag = ws.alloc<int>(1);
  const bool dev = is_device_ptr(out);
  double* dst = dev ? out : ws.alloc<double>((size_t)n);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, cudaGetErrorString(ws.err));
  bool ok = false;
  CK(pairs_in_range(st, n, dr, dc, ctx->rows[0], ctx->rows[1], flag, &ok));
  if (!ok) return set_err(ctx, TSVD_E_OOB, "pair index out of range");
  CKS(flush_pending(ctx, 0, st));
  CKS(flush_pending(ctx, 1, st));
  CK(score_pairs(st, ctx->X[0][0], ctx->M[0], ctx->X[1][0], ctx->M[1], ctx->Sigma, ctx->k, n, dr, dc, dst, ws));
  if (!dev) CK(cudaMemcpyAsync(out, dst, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return TSVD_OK;
}

tsvd_status tsvd_residual_fro(tsvd_ctx* ctx, const tsvd_sparse* A, double* out3, void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  if (!ctx->initialized) return set_err(ctx, TSVD_E_INVALID, "context not initialised");
  if (ctx->world > 1) return set_err(ctx, TSVD_E_UNSUPPORTED, "residual_fro on a sharded context");
  if (!A || !out3) return set_err(ctx, TSVD_E_INVALID, "null argument");
  if (A->s != ctx->rows[0]) return set_err(ctx, TSVD_E_SHAPE, "A must have m rows");
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  Scratch ws(st);
  int* d_flag = ws.alloc<int>(1);
  if (ws.err) return set_err(ctx, TSVD_E_OOM, "scratch");
  CK(cudaMemsetAsync(d_flag, 0, sizeof(int), st));
  DevCSR dA;
  CKS(stage_sparse(ctx, A, ctx->rows[1], ws, st, dA, d_flag, true));
  double io[2] = {0.0, 0.0};
  CKS(flush_pending(ctx, 0, st));
  CKS(flush_pending(ctx, 1, st));
  CK(sparse_inner(st, ctx->X[0][0], ctx->M[0], ctx->X[1][0], ctx->M[1], ctx->Sigma, ctx->k, dA, io, ws));
  std::vector<double> hs(ctx->k);
  CK(cudaMemcpyAsync(hs.data(), ctx->Sigma, ctx->k * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double s2 = 0.0;
  for (double x : hs) s2 += x * x;
  const double r2 = io[1] - 2.0 * io[0] + s2;  // ||A||^2 - 2 <A, Ã> + ||Ã||^2 (U, V orthonormal)
  out3[0] = std::sqrt(std::max(r2, 0.0));
  out3[1] = io[0];
  out3[2] = io[1];
  return TSVD_OK;
}

tsvd_status tsvd_materialize(tsvd_ctx* ctx, void* stream) {
  if (!ctx) return TSVD_E_INVALID;
  if (!ctx->initialized) return set_err(ctx, TSVD_E_INVALID, "context not initialised");
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  for (int s = 0; s < 2; ++s) {
    CKS(flush_pending(ctx, s, st));
    for (int g = 0; g < ctx->nloc; ++g) CK(materialize_rows(st, ctx->X[s][g], lrows(ctx, s, g), ctx->k, ctx->M[s]));
    CK(set_identity(st, ctx->M[s], ctx->k));
  }
  CK(cudaStreamSynchronize(st));
  return TSVD_OK;
}

// ------------------------------------------------------------------ F4: state persistence
// (tsvd.h "State persistence").  Host-side file I/O around device copies.
namespace {
constexpr char kStateMagic[8] = {'T', 'S', 'V', 'D', 'S', 'T', 'A', 'T'};
constexpr uint32_t kStateVersion = 1;
constexpr size_t kStateHeader = 64;

uint64_t fnv1a(const void* p, size_t n, uint64_t h = 1469598103934665603ull) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}

struct StateHeader {
  uint32_t version = 0;
  int32_t k = 0;
  int64_t m = 0, n = 0, resets = 0;
  uint64_t payload_sum = 0;
};

void put_header(unsigned char* h, const StateHeader& H) {  // little-endian host (x86-64 / aarch64)
  memset(h, 0, kStateHeader);
  memcpy(h, kStateMagic, 8);
  memcpy(h + 8, &H.version, 4);
  memcpy(h + 12, &H.k, 4);
  memcpy(h + 16, &H.m, 8);
  memcpy(h + 24, &H.n, 8);
  memcpy(h + 32, &H.resets, 8);
  memcpy(h + 40, &H.payload_sum, 8);
  const uint64_t hs = fnv1a(h, 48);
  memcpy(h + 48, &hs, 8);
}

// 0 ok, else a message
const char* get_header(const unsigned char* h, StateHeader& H, tsvd_status* st) {
  *st = TSVD_E_IO;
  if (memcmp(h, kStateMagic, 8) != 0) return "not a tsvd state file (bad magic)";
  uint64_t hs;
  memcpy(&hs, h + 48, 8);
  if (hs != fnv1a(h, 48)) return "state file header checksum mismatch";
  memcpy(&H.version, h + 8, 4);
  memcpy(&H.k, h + 12, 4);
  memcpy(&H.m, h + 16, 8);
  memcpy(&H.n, h + 24, 8);
  memcpy(&H.resets, h + 32, 8);
  memcpy(&H.payload_sum, h + 40, 8);
  if (H.version != kStateVersion) {
    *st = TSVD_E_STATE_VERSION;
    return "state_version: unsupported state file version";
  }
  if (H.k <= 0 || H.m < H.k || H.n < H.k) return "state file header: bad dimensions";
  *st = TSVD_OK;
  return nullptr;
}

bool write_all(int fd, const void* p, size_t n) {
  const char* b = static_cast<const char*>(p);
  while (n) {
    const ssize_t w = ::write(fd, b, n);
    if (w <= 0) return false;
    b += w;
    n -= (size_t)w;
  }
  return true;
}

bool read_all(FILE* f, void* p, size_t n) { return fread(p, 1, n, f) == n; }
}  // namespace

tsvd_status tsvd_save(tsvd_ctx* ctx, const char* path, void* stream) {
  if (!ctx || !path) return TSVD_E_INVALID;
  if (!ctx->initialized) return set_err(ctx, TSVD_E_INVALID, "context not initialised");
  if (ctx->world != 1) return set_err(ctx, TSVD_E_UNSUPPORTED, "tsvd_save: sharded context");
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int k = ctx->k;
  const int64_t m = ctx->rows[0], n = ctx->rows[1];
  for (int s = 0; s < 2; ++s) CKS(flush_pending(ctx, s, st));
  // payload in file order: U', U'', Sigma, V', V''
  const size_t cnt[5] = {(size_t)m * k, (size_t)k * k, (size_t)k, (size_t)n * k, (size_t)k * k};
  const double* src[5] = {ctx->X[0][0], ctx->M[0], ctx->Sigma, ctx->X[1][0], ctx->M[1]};
  size_t total = 0;
  for (size_t c : cnt) total += c;
  double* h = nullptr;
  CK(cudaMallocHost(&h, total * sizeof(double)));
  struct Free { double* p; ~Free() { cudaFreeHost(p); } } fr{h};
  size_t off = 0;
  for (int i = 0; i < 5; ++i) {
    CK(cudaMemcpyAsync(h + off, src[i], cnt[i] * sizeof(double), cudaMemcpyDeviceToHost, st));
    off += cnt[i];
  }
  CK(cudaStreamSynchronize(st));
  StateHeader H;
  H.version = kStateVersion;
  H.k = k;
  H.m = m;
  H.n = n;
  H.resets = ctx->total_resets;
  H.payload_sum = fnv1a(h, total * sizeof(double));
  unsigned char hdr[kStateHeader];
  put_header(hdr, H);
  const std::string tmp = std::string(path) + ".tmp";
  const int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) return set_err(ctx, TSVD_E_IO, "tsvd_save: cannot open " + tmp);
  const bool ok = write_all(fd, hdr, kStateHeader) && write_all(fd, h, total * sizeof(double)) && ::fsync(fd) == 0;
  ::close(fd);
  if (!ok) {
    ::unlink(tmp.c_str());
    return set_err(ctx, TSVD_E_IO, "tsvd_save: write failed: " + tmp);
  }
  if (::rename(tmp.c_str(), path) != 0) {
    ::unlink(tmp.c_str());
    return set_err(ctx, TSVD_E_IO, std::string("tsvd_save: rename failed: ") + path);
  }
  return TSVD_OK;
}

tsvd_status tsvd_state_info(const char* path, int32_t* k, int64_t* m, int64_t* n) {
  if (!path) return TSVD_E_INVALID;
  FILE* f = fopen(path, "rb");
  if (!f) return TSVD_E_IO;
  unsigned char hdr[kStateHeader];
  const bool ok = read_all(f, hdr, kStateHeader);
  fclose(f);
  if (!ok) return TSVD_E_IO;
  StateHeader H;
  tsvd_status s;
  if (get_header(hdr, H, &s)) return s;
  if (k) *k = H.k;
  if (m) *m = H.m;
  if (n) *n = H.n;
  return TSVD_OK;
}

tsvd_status tsvd_load(tsvd_ctx* ctx, const char* path, void* stream) {
  if (!ctx || !path) return TSVD_E_INVALID;
  if (ctx->world != 1) return set_err(ctx, TSVD_E_UNSUPPORTED, "tsvd_load: sharded context");
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  FILE* f = fopen(path, "rb");
  if (!f) return set_err(ctx, TSVD_E_IO, std::string("tsvd_load: cannot open ") + path);
  struct Close { FILE* f; ~Close() { fclose(f); } } cl{f};
  unsigned char hdr[kStateHeader];
  if (!read_all(f, hdr, kStateHeader)) return set_err(ctx, TSVD_E_IO, "tsvd_load: truncated header");
  StateHeader H;
  tsvd_status hs;
  if (const char* msg = get_header(hdr, H, &hs)) return set_err(ctx, hs, msg);
  const int k = ctx->k;
  if (H.k != k) return set_err(ctx, TSVD_E_SHAPE, "tsvd_load: the file's k differs from the context's");
  const int64_t m = H.m, n = H.n;
  const size_t cnt[5] = {(size_t)m * k, (size_t)k * k, (size_t)k, (size_t)n * k, (size_t)k * k};
  size_t total = 0;
  for (size_t c : cnt) total += c;
  double* h = nullptr;
  CK(cudaMallocHost(&h, total * sizeof(double)));
  struct Free { double* p; ~Free() { cudaFreeHost(p); } } fr{h};
  if (!read_all(f, h, total * sizeof(double))) return set_err(ctx, TSVD_E_IO, "tsvd_load: truncated payload");
  if (fgetc(f) != EOF) return set_err(ctx, TSVD_E_IO, "tsvd_load: trailing bytes after the payload");
  if (fnv1a(h, total * sizeof(double)) != H.payload_sum) return set_err(ctx, TSVD_E_IO, "tsvd_load: payload checksum mismatch");
  // validate before touching the context (a failed load leaves it unchanged)
  for (size_t i = 0; i < total; ++i)
    if (!std::isfinite(h[i])) return set_err(ctx, TSVD_E_NUMERIC, "tsvd_load: non-finite value");
  const double* sig = h + cnt[0] + cnt[1];
  for (int i = 0; i < k; ++i)
    if (sig[i] < 0 || (i > 0 && sig[i] > sig[i - 1])) return set_err(ctx, TSVD_E_BAD_SIGMA, "tsvd_load: sigma not descending / >= 0");
  CK(cudaStreamSynchronize(st));
  drop_pending(ctx);
  CKS(ensure_cap(ctx, 0, m, st));
  CKS(ensure_cap(ctx, 1, n, st));
  double* dst[5] = {ctx->X[0][0], ctx->M[0], ctx->Sigma, ctx->X[1][0], ctx->M[1]};
  size_t off = 0;
  for (int i = 0; i < 5; ++i) {
    CK(cudaMemcpyAsync(dst[i], h + off, cnt[i] * sizeof(double), cudaMemcpyHostToDevice, st));
    off += cnt[i];
  }
  CK(cudaStreamSynchronize(st));
  ctx->rows[0] = m;
  ctx->rows[1] = n;
  ctx->initialized = true;
  ctx->total_resets = (int)H.resets;
  for (int q = 0; q < 3; ++q) {
    ctx->core_hint[q] = 0;
    ctx->core_growth[q] = 0;
    ctx->core_thb2[q] = 0;
    ctx->core_b[q] = 0;
  }
  return TSVD_OK;
}

tsvd_status tsvd_dims(const tsvd_ctx* ctx, int64_t* m, int64_t* n, int32_t* k) {
  if (!ctx) return TSVD_E_INVALID;
  if (m) *m = ctx->rows[0];
  if (n) *n = ctx->rows[1];
  if (k) *k = ctx->k;
  return TSVD_OK;
}

tsvd_status tsvd_reserve(tsvd_ctx* ctx, int64_t bytes, void* stream) {
  if (!ctx || bytes < 0) return TSVD_E_INVALID;
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  void* p = nullptr;
  CK(cudaMallocAsync(&p, (size_t)bytes, st));
  CK(cudaFreeAsync(p, st));
  CK(cudaStreamSynchronize(st));
  return TSVD_OK;
}

tsvd_status tsvd_last_stats_nowait(const tsvd_ctx* ctx, tsvd_stats* out) {
  if (!ctx || !out) return TSVD_E_INVALID;
  *out = ctx->stats;
  return TSVD_OK;
}

tsvd_status tsvd_last_stats(const tsvd_ctx* ctx, tsvd_stats* out) {
  if (!ctx || !out) return TSVD_E_INVALID;
  resolve_times(const_cast<tsvd_ctx*>(ctx));
  *out = ctx->stats;
  return TSVD_OK;
}

// ---------------------------------------------------------------- step-level entry points
#define KCK(call)                                   \
  do {                                              \
    cudaError_t _e = (call);                        \
    if (_e != cudaSuccess) return TSVD_E_CUDA;      \
  } while (0)

static DevCSR dev_csr(const tsvd_sparse* E) {
  DevCSR d;
  d.s = E->s;
  d.dim = E->dim;
  d.nnz = E->nnz;
  d.row_ptr = E->row_ptr;
  d.col_idx = E->col_idx;
  d.val = E->val;
  return d;
}

tsvd_status tsvd_k_dgemm(int32_t transA, int32_t transB, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int32_t uplo,
                         void* stream) {
  if (M < 0 || N < 0 || K < 0) return TSVD_E_INVALID;
  KCK(dgemm_rm((cudaStream_t)stream, transA != 0, transB != 0, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, uplo));
  return TSVD_OK;
}

tsvd_status tsvd_k_gather_spmm(const tsvd_sparse* E, const double* X, int32_t k, double* W, void* stream) {
  if (!E || k <= 0) return TSVD_E_INVALID;
  KCK(gather_spmm((cudaStream_t)stream, dev_csr(E), X, k, W));
  return TSVD_OK;
}

tsvd_status tsvd_k_sparse_gram(const tsvd_sparse* E, double* G, void* stream) {
  if (!E) return TSVD_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch ws(st);
  DevCSC C;
  int64_t nJ = 0;
  KCK(build_csc(st, dev_csr(E), C, ws, &nJ));
  KCK(sparse_gram(st, dev_csr(E), C, G, ws));
  KCK(cudaStreamSynchronize(st));
  return TSVD_OK;
}

tsvd_status tsvd_k_chol_deflate(double* G, int64_t s, const double* enorm2, double tau, int32_t* keep, int64_t* rank,
                                void* stream) {
  if (s < 0) return TSVD_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch ws(st);
  int32_t* kidx = ws.alloc<int32_t>(2 * s + 1);
  int64_t* d_r = ws.alloc<int64_t>(1);
  if (ws.err) return TSVD_E_OOM;
  KCK(chol_deflate(st, G, s, enorm2, tau, keep));
  KCK(compact_keep(st, keep, s, kidx, d_r, ws));
  int64_t r = 0;
  KCK(cudaMemcpyAsync(&r, d_r, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  KCK(cudaStreamSynchronize(st));
  if (rank) *rank = r;
  return TSVD_OK;
}

tsvd_status tsvd_k_trsm_upper(const double* R, int64_t s, const int32_t* keep, double* X, int32_t k, void* stream) {
  if (s < 0 || k <= 0) return TSVD_E_INVALID;
  KCK(trsm_upper((cudaStream_t)stream, R, s, keep, X, k));
  return TSVD_OK;
}

tsvd_status tsvd_k_jacobi_svd(const double* K, int64_t m, int64_t n, int32_t kk, double* theta, double* F, double* G,
                              int32_t* sweeps, void* stream) {
  if (m < n || kk > n || kk < 0) return TSVD_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch ws(st);
  int sw = 0;
  bool conv = false;
  KCK(jacobi_svd(st, K, m, m, n, kk, theta, F, m, G, n, &sw, &conv, ws));
  KCK(cudaStreamSynchronize(st));
  if (sweeps) *sweeps = sw;
  return conv ? TSVD_OK : TSVD_E_SVD_FAIL;
}

tsvd_status tsvd_k_core_svd(const double* K, int64_t m, int64_t n, int32_t kk, double* theta, double* F, double* G,
                            double* info, void* stream) {
  if (m < n || kk > n || kk < 0) return TSVD_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch ws(st);
  CoreInfo ci;
  KCK(core_svd(st, K, m, m, n, kk, theta, F, m, G, n, &ci, ws));
  KCK(cudaStreamSynchronize(st));
  if (info) {
    info[0] = ci.path;
    info[1] = ci.iters;
    info[2] = ci.sweeps;
    info[3] = ci.energy;
  }
  return ci.converged ? TSVD_OK : TSVD_E_SVD_FAIL;
}

tsvd_status tsvd_k_cholqr(double* X, int64_t rows, int64_t l, int32_t passes, double tau, double* R, void* stream) {
  if (!X || rows < 0 || l <= 0 || passes < 1 || passes > 2) return TSVD_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch ws(st);
  KCK(cholqr_dense(st, X, rows, l, tau > 0 ? tau : 1e-14, passes, R, ws));
  return TSVD_OK;
}

tsvd_status tsvd_k_chol_rinv(double* G, int64_t l, const double* en, double tau, int32_t* keep, double* T,
                             void* stream) {
  if (!G || !keep || !T || l <= 0 || !(tau >= 0)) return TSVD_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch ws(st);
  KCK(chol_rinv(st, G, l, en, tau, keep, T, ws, true));
  return TSVD_OK;
}

tsvd_status tsvd_k_norm2_est(const double* M, int32_t k, double* out, void* stream) {
  if (k <= 0) return TSVD_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const double* mats[1] = {M};
  KCK(norm2_estimates(st, mats, 1, k, out));
  KCK(cudaStreamSynchronize(st));
  return TSVD_OK;
}

tsvd_status tsvd_k_inverse(const double* M, int32_t k, double* Minv, double* cond, void* stream) {
  if (k <= 0) return TSVD_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch ws(st);
  KCK(inverse_gj(st, M, k, Minv, cond, ws));
  KCK(cudaStreamSynchronize(st));
  return TSVD_OK;
}

tsvd_status tsvd_k_scatter_add(const tsvd_sparse* E, const double* Z, int32_t k, double* X, void* stream) {
  if (!E || k <= 0) return TSVD_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  Scratch ws(st);
  DevCSC C;
  int64_t nJ = 0;
  KCK(build_csc(st, dev_csr(E), C, ws, &nJ));
  KCK(scatter_add(st, C, E->nnz, Z, k, X));
  KCK(cudaStreamSynchronize(st));
  return TSVD_OK;
}

tsvd_status tsvd_k_materialize(double* X, int64_t rows, int32_t k, const double* M, void* stream) {
  if (rows < 0 || k <= 0) return TSVD_E_INVALID;
  KCK(materialize_rows((cudaStream_t)stream, X, rows, k, M));
  return TSVD_OK;
}

tsvd_status tsvd_k_gaussian(uint64_t seed, int32_t side, int64_t s, int64_t l, double* out, void* stream) {
  if (s < 0 || l < 0) return TSVD_E_INVALID;
  KCK(counter_gaussian((cudaStream_t)stream, seed, side, s, l, out));
  return TSVD_OK;
}

tsvd_status tsvd_k_approx_basis(const tsvd_sparse* E, const double* X, int32_t k, const tsvd_opts* opts,
                                int32_t side, double* BJfull, double* Cp, double* P, void* stream) {
  if (!E || !X || !opts || k <= 0 || (opts->mode != TSVD_RPI && opts->mode != TSVD_GKL)) return TSVD_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  // a throw-away context around the caller's X (M_X = I)
  tsvd_ctx tmp;
  tmp.k = k;
  tmp.rows[side & 1] = E->dim;
  tmp.X[0].assign(1, nullptr);
  tmp.X[1].assign(1, nullptr);
  tmp.X[side & 1][0] = const_cast<double*>(X);
  if (cudaMallocHost(&tmp.h_i64, 64 * sizeof(int64_t)) != cudaSuccess) return TSVD_E_OOM;
  Scratch ws(st);
  double* I = ws.alloc<double>((size_t)k * k);
  if (ws.err) { cudaFreeHost(tmp.h_i64); return TSVD_E_OOM; }
  tmp.M[side & 1] = I;
  tsvd_status rc = TSVD_OK;
  if (set_identity(st, I, k) != cudaSuccess) rc = TSVD_E_CUDA;
  Lift L;
  L.side = side & 1;
  L.mode = opts->mode;
  L.E = dev_csr(E);
  tsvd_opts o = resolve_opts(opts);
  if (rc == TSVD_OK) rc = lift_approx(&tmp, L, o, o.sketch, side, ws, st);
  if (rc == TSVD_OK && cudaMemsetAsync(BJfull, 0, (size_t)E->dim * L.l * sizeof(double), st)) rc = TSVD_E_CUDA;
  if (rc == TSVD_OK && L.nJ > 0) {
    // scatter the compact rows back to their positions: BJfull[J[jj]] = BJ[jj]
    if (index_add_rows(st, L.sh[0].C.J, L.nJ, L.sh[0].BJ, (int)L.l, BJfull) != cudaSuccess) rc = TSVD_E_CUDA;
  }
  if (rc == TSVD_OK) {
    cudaMemcpyAsync(Cp, L.Cp, (size_t)k * L.l * sizeof(double), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(P, L.Pa, (size_t)E->s * L.l * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) rc = TSVD_E_CUDA;
  }
  tmp.X[0][0] = tmp.X[1][0] = tmp.M[0] = tmp.M[1] = nullptr;
  cudaFreeHost(tmp.h_i64);
  tmp.h_i64 = nullptr;
  return rc;
}

}  // extern "C"
