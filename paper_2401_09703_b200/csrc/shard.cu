// shard.cu — row sharding of the base factors U', V' over GPUs.
//
// Rows are dealt block-cyclically: global row i lives on shard (i / B) % W at local row
// (i / (B W)) B + i % B, so appended rows spread over the shards as the factor grows.  A
// sparse update block E (replicated on every shard) is split by the owner of its column
// (= the lift-side row it touches); the partial products over the local rows (W = E X',
// B'^T B', E^T B') are then summed over the shards by the Reducer: ncclAllReduce in NCCL
// mode (one process per GPU), an on-device sum in virtual mode (all shards held by one
// context on one GPU — used to test the partitioning on a single B200).
//
// NCCL is loaded with dlopen only when a NCCL-sharded context is created, so the library
// reuses the libnccl.so.2 torch.distributed already loaded in the process.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>

#include "ops.h"

namespace tsvd {

namespace {
__device__ __forceinline__ int shard_of(int64_t i, int world, int block) { return (int)((i / block) % world); }
__device__ __forceinline__ int64_t local_of(int64_t i, int world, int block) {
  return (i / ((int64_t)block * world)) * block + i % block;
}

// rows of E: count of nonzeros whose column belongs to shard g (warp per row)
__global__ void shard_count_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int g,
                                   int world, int block, int64_t* __restrict__ cnt) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w > s) return;
  if (w == s) {  // the scan's tail slot
    if (lane == 0) cnt[s] = 0;
    return;
  }
  int64_t c = 0;
  for (int64_t p = rp[w] + lane; p < rp[w + 1]; p += 32) c += (shard_of(ci[p], world, block) == g);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[w] = c;
}

// order-preserving compaction of the owned nonzeros with local column indices
__global__ void shard_fill_kernel(int64_t s, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  const double* __restrict__ v, int g, int world, int block,
                                  const int64_t* __restrict__ rpg, int32_t* __restrict__ cig, double* __restrict__ vg) {
  pdl_begin();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= s) return;
  int64_t out = rpg[w];
  for (int64_t p0 = rp[w]; p0 < rp[w + 1]; p0 += 32) {
    const int64_t p = p0 + lane;
    const bool in = p < rp[w + 1];
    const int c = in ? ci[p] : 0;
    const bool own = in && shard_of(c, world, block) == g;
    const unsigned mask = __ballot_sync(0xffffffffu, own);
    if (own) {
      const int64_t q = out + __popc(mask & ((1u << lane) - 1));
      cig[q] = (int32_t)local_of(c, world, block);
      vg[q] = v[p];
    }
    out += __popc(mask);
  }
}

// Xg[local(i)] = Full[i] for the rows i < rows owned by g
__global__ void gather_owned_kernel(const double* __restrict__ full, int64_t rows, int k, int g, int world, int block,
                                    double* __restrict__ Xg) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / k;
    if (shard_of(i, world, block) != g) continue;
    Xg[local_of(i, world, block) * k + e % k] = full[e];
  }
}

// Xg[local(row0 + i)] = R[i] for the new rows row0 + i owned by g
__global__ void put_rows_kernel(const double* __restrict__ R, int64_t s, int k, int64_t row0, int g, int world,
                                int block, double* __restrict__ Xg) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < s * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = row0 + e / k;
    if (shard_of(i, world, block) != g) continue;
    Xg[local_of(i, world, block) * k + e % k] = R[e];
  }
}

// Out[i] = Xl[local(i)] for the global rows i owned by g (Xl: local rows x k)
__global__ void scatter_owned_kernel(const double* __restrict__ Xl, int64_t rows, int k, int g, int world, int block,
                                     double* __restrict__ out) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / k;
    if (shard_of(i, world, block) != g) continue;
    out[e] = Xl[local_of(i, world, block) * k + e % k];
  }
}

// out[i] = G[r * maxl + local(i)] with r = shard(i): the rows of an all-gather of per-shard
// blocks (each maxl rows, shard r's local rows first) placed at their global positions
__global__ void unshuffle_kernel(const double* __restrict__ G, int64_t rows, int64_t maxl, int k, int world, int block,
                                 double* __restrict__ out) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / k;
    out[e] = G[((int64_t)shard_of(i, world, block) * maxl + local_of(i, world, block)) * k + e % k];
  }
}

// global row ids of shard g's local rows 0 .. nl-1
__global__ void global_ids_kernel(int64_t nl, int g, int world, int block, int64_t* __restrict__ ids) {
  pdl_begin();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < nl) ids[j] = ((j / block) * world + g) * (int64_t)block + j % block;
}

__global__ void add_into_kernel(double* __restrict__ acc, const double* __restrict__ x, int64_t n) {
  pdl_begin();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    acc[e] += x[e];
}

inline unsigned gsz(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16)); }
}  // namespace

int64_t shard_rows(int64_t rows, int g, int world, int block) {
  const int64_t cyc = (int64_t)block * world;
  const int64_t full = rows / cyc, rem = rows % cyc;
  return full * block + std::min<int64_t>(std::max<int64_t>(rem - (int64_t)g * block, 0), block);
}

cudaError_t shard_split(cudaStream_t st, const DevCSR& E, int g, int world, int block, int64_t dim_local, DevCSR& out,
                        Scratch& ws, int64_t* h_scratch) {
  out.s = E.s;
  out.dim = dim_local;
  int64_t* cnt = ws.alloc<int64_t>(E.s + 1);
  int64_t* rpg = ws.alloc<int64_t>(E.s + 1);
  if (ws.err) return ws.err;
  g_launches += 1;
  launch_k(shard_count_kernel, cdiv((E.s + 1) * 32, 256), 256, 0, st, E.s, E.row_ptr, E.col_idx, g, world, block, cnt);
  cudaError_t e = scan_exclusive_i64(st, cnt, rpg, E.s + 1, ws);
  if (e) return e;
  if ((e = cudaMemcpyAsync(h_scratch, rpg + E.s, sizeof(int64_t), cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;
  out.nnz = *h_scratch;
  int32_t* cig = ws.alloc<int32_t>(std::max<int64_t>(out.nnz, 1));
  double* vg = ws.alloc<double>(std::max<int64_t>(out.nnz, 1));
  if (ws.err) return ws.err;
  if (E.s > 0) {
    g_launches += 1;
    launch_k(shard_fill_kernel, cdiv(E.s * 32, 256), 256, 0, st, E.s, E.row_ptr, E.col_idx, E.val, g, world, block, rpg,
                                                            cig, vg);
  }
  out.row_ptr = rpg;
  out.col_idx = cig;
  out.val = vg;
  return cudaGetLastError();
}

cudaError_t shard_gather_owned(cudaStream_t st, const double* full, int64_t rows, int k, int g, int world, int block,
                               double* Xg) {
  if (rows * k == 0) return cudaSuccess;
  ++g_launches;
  launch_k(gather_owned_kernel, gsz(rows * k), 256, 0, st, full, rows, k, g, world, block, Xg);
  return cudaGetLastError();
}

cudaError_t shard_put_rows(cudaStream_t st, const double* R, int64_t s, int k, int64_t row0, int g, int world,
                           int block, double* Xg) {
  if (s * k == 0) return cudaSuccess;
  ++g_launches;
  launch_k(put_rows_kernel, gsz(s * k), 256, 0, st, R, s, k, row0, g, world, block, Xg);
  return cudaGetLastError();
}

cudaError_t shard_scatter_owned(cudaStream_t st, const double* Xl, int64_t rows, int k, int g, int world, int block,
                                double* out) {
  if (rows * k == 0) return cudaSuccess;
  ++g_launches;
  launch_k(scatter_owned_kernel, gsz(rows * k), 256, 0, st, Xl, rows, k, g, world, block, out);
  return cudaGetLastError();
}

cudaError_t shard_unshuffle(cudaStream_t st, const double* G, int64_t rows, int64_t maxl, int k, int world, int block,
                            double* out) {
  if (rows * k == 0) return cudaSuccess;
  ++g_launches;
  launch_k(unshuffle_kernel, gsz(rows * k), 256, 0, st, G, rows, maxl, k, world, block, out);
  return cudaGetLastError();
}

int64_t shard_global_row(int64_t j, int g, int world, int block) {
  return ((j / block) * world + g) * (int64_t)block + j % block;
}

cudaError_t add_into(cudaStream_t st, double* acc, const double* x, int64_t n) {
  if (n == 0) return cudaSuccess;
  ++g_launches;
  launch_k(add_into_kernel, gsz(n), 256, 0, st, acc, x, n);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
  bool loaded = false;
  void* h = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  int (*commInitRank)(void**, int, NcclUniqueIdBytes, int) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*allGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*broadcast)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  const char* (*errorString)(int) = nullptr;
};
NcclApi g_nccl;

bool nccl_load() {
  if (g_nccl.loaded) return g_nccl.h != nullptr;
  g_nccl.loaded = true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    g_nccl.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.h) break;
  }
  if (!g_nccl.h) return false;
  g_nccl.getUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(g_nccl.h, "ncclGetUniqueId"));
  g_nccl.commInitRank =
      reinterpret_cast<int (*)(void**, int, NcclUniqueIdBytes, int)>(dlsym(g_nccl.h, "ncclCommInitRank"));
  g_nccl.allReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
      dlsym(g_nccl.h, "ncclAllReduce"));
  g_nccl.allGather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(
      dlsym(g_nccl.h, "ncclAllGather"));
  g_nccl.broadcast = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
      dlsym(g_nccl.h, "ncclBroadcast"));
  g_nccl.commDestroy = reinterpret_cast<int (*)(void*)>(dlsym(g_nccl.h, "ncclCommDestroy"));
  g_nccl.errorString = reinterpret_cast<const char* (*)(int)>(dlsym(g_nccl.h, "ncclGetErrorString"));
  if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.allReduce || !g_nccl.allGather || !g_nccl.broadcast ||
      !g_nccl.commDestroy) {
    g_nccl.h = nullptr;
    return false;
  }
  return true;
}
}  // namespace

int nccl_unique_id(void* out128) {
  if (!nccl_load()) return -1;
  return g_nccl.getUniqueId(out128);
}

int nccl_comm_init(void** comm, int world, const void* id128, int rank) {
  if (!nccl_load()) return -1;
  NcclUniqueIdBytes id;
  memcpy(id.b, id128, sizeof(id.b));
  return g_nccl.commInitRank(comm, world, id, rank);
}

int nccl_allreduce_sum_f64(void* comm, double* buf, int64_t count, cudaStream_t st) {
  // ncclFloat64 = 8, ncclSum = 0 (nccl.h enums)
  return g_nccl.allReduce(buf, buf, (size_t)count, 8, 0, comm, st);
}

int nccl_allgather_f64(void* comm, const double* send, double* recv, int64_t count, cudaStream_t st) {
  return g_nccl.allGather(send, recv, (size_t)count, 8, comm, st);
}

int nccl_broadcast_f64(void* comm, const double* send, double* recv, int64_t count, int root, cudaStream_t st) {
  return g_nccl.broadcast(send, recv, (size_t)count, 8, root, comm, st);
}

void nccl_comm_destroy(void* comm) {
  if (comm && g_nccl.commDestroy) g_nccl.commDestroy(comm);
}

const char* nccl_error(int rc) {
  if (rc < 0 || !g_nccl.h) return dlerror() ? dlerror() : "libnccl.so.2 not loadable";
  return g_nccl.errorString ? g_nccl.errorString(rc) : "nccl error";
}

}  // namespace tsvd
