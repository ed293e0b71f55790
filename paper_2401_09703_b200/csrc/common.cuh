// common.cuh — shared device helpers of libtsvd (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libtsvd is written for sm_100a (B200) only"
#endif

namespace tsvd {

constexpr int kWarp = 32;

// ---- programmatic dependent launch.  Every kernel of the library is launched with
// programmatic stream serialisation and begins with pdl_begin(): it lets the next kernel on
// the stream launch as soon as all of this grid's CTAs have started, then waits for the
// previous grid to complete and flush its memory.  The launch of kernel n+1 (its CTAs
// rasterised, resident and waiting) thus overlaps the tail of kernel n, instead of starting
// after it drains (~2 us per kernel boundary; a configs[1] step has ~500).  Correctness is
// the plain stream order: no kernel touches memory before its griddepcontrol.wait, which
// returns only when the preceding grid has completed (and that grid waited on its own
// predecessor in turn).  TSVD_PDL=0 launches without the attribute (the wait is then a no-op).
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

inline bool pdl_on() {
  static const int v = (getenv("TSVD_PDL") && atoi(getenv("TSVD_PDL")) == 0) ? 0 : 1;
  return v != 0;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Strided fp64 matrix view: element (i, j) at p[i * rs + j * cs].
struct CMat {
  const double* p;
  int64_t rs, cs;
};
struct Mat {
  double* p;
  int64_t rs, cs;
};

// FP64 tensor-core MMA (DMMA): D(8x8) += A(8x4, row) * B(4x8, col).
// Fragment layout (PTX ISA, mma.m8n8k4 .f64): lane = 4*g + t;
//   a = A[g][t], b = B[t][g], {c0, c1} = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// (e / n, e % n) with a 32-bit division when both fit (64-bit integer division is a long
// software sequence on the GPU)
__device__ __forceinline__ void divmod_idx(int64_t e, int64_t n, int64_t& q, int64_t& r) {
  if (e <= 0x7fffffff && n <= 0x7fffffff) {
    const unsigned qq = (unsigned)e / (unsigned)n;
    q = qq;
    r = e - (int64_t)qq * n;
  } else {
    q = e / n;
    r = e - q * n;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// streaming (read-once) loads that do not allocate in L1
__device__ __forceinline__ int ld_stream_i32(const int32_t* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

}  // namespace tsvd
