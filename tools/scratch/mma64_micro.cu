// Micro: the tile-DAG's 64x64x64 DMMA product (mma64 of dag.cu: 8 warps, warp tile 16 x 32,
// operands [k][m] in smem, pitch 72) — cycles per call vs the DMMA-pipe bound (4096).
#include <cstdio>
#include "../../paper_2401_09703_b200/csrc/common.cuh"
using namespace tsvd;
constexpr int TB = 64, TP = TB + 8;
// B shares the A buffer offset by 64 rows of a 2-tile array (static smem limit 48 KB)
template <bool NEG, int UNR>
__device__ __forceinline__ void mma64(double (&acc)[2][4][2], const double* As, const double* Bs, int rb, int cb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll UNR
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
template <int UNR>
__global__ void __launch_bounds__(256, 1) k(double* out, long long* cyc, int reps) {
  extern __shared__ double sm[];
  double *As = sm, *Bs = sm + TB * TP;
  for (int e = threadIdx.x; e < TB * TP; e += 256) { As[e] = e * 1e-6; Bs[e] = 1.0 - e * 1e-7; }
  __syncthreads();
  const int warp = threadIdx.x >> 5, rb = (warp >> 1) * 16, cb = (warp & 1) * 32;
  double acc[2][4][2] = {};
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) mma64<true, UNR>(acc, As, Bs, rb, cb);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int x = 0; x < 2; ++x) for (int y = 0; y < 4; ++y) s += acc[x][y][0] + acc[x][y][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}
int main() {
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TB * TP * 8);
  cudaFuncSetAttribute(k<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TB * TP * 8);
  double* o; long long* c; cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
  long long h;
  k<4><<<1, 256, 2 * TB * TP * 8>>>(o, c, 200); k<4><<<1, 256, 2 * TB * TP * 8>>>(o, c, 200); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("mma64 unroll 4: %lld cycles per call (DMMA bound 4096)\n", h);
  k<16><<<1, 256, 2 * TB * TP * 8>>>(o, c, 200); k<16><<<1, 256, 2 * TB * TP * 8>>>(o, c, 200); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("mma64 unroll 16: %lld cycles per call (%s)\n", h, cudaGetErrorString(cudaGetLastError()));
}
