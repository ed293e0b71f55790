// Micro: dependent-chain latencies on sm_100a (DFMA, DMUL, rsqrt(double), SHFL 64-bit, DMMA m8n8k4,
// LDS.64, __syncthreads with 256 threads).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 lat_micro.cu
#include <cstdio>
#include "../../paper_2401_09703_b200/csrc/common.cuh"
using namespace tsvd;
__global__ void k(double* out, long long* cyc, double seed, int n) {
  __shared__ double sm[256];
  sm[threadIdx.x] = seed + threadIdx.x;
  __syncthreads();
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
  // rsqrt chain
  double z = x + 2.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) z = rsqrt(z) + 1.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / n;
  // shfl 64-bit chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / n;
  // DMMA chain (accumulate dependency)
  double a0 = x, a1 = z;
  t0 = clock64();
  for (int i = 0; i < n; ++i) dmma8x8x4(a0, a1, y, 1e-3);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
  // LDS chain (pointer chasing through an index)
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) idx = ((int)sm[idx] + 1) & 255;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / n;
  // syncthreads
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) / n;
  // double division chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) z = 1.0 / z + 0.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = (t1 - t0) / n;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) z = sqrt(z) + 0.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[8] = (t1 - t0) / n;
  // rsqrtf on float + 1 fp64 Newton
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double r = (double)rsqrtf((float)z);
    r = r * fma(-0.5 * z * r, r, 1.5);
    z = r + 1.5;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[9] = (t1 - t0) / n;
  out[threadIdx.x] = x + a0 + a1 + z + idx;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 256 * 8);
  cudaMalloc(&c, 16 * 8);
  for (int nthr : {32, 256}) {
    k<<<1, nthr>>>(o, c, 1.0, 1000);
    k<<<1, nthr>>>(o, c, 1.0, 1000);
    long long h[10];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %d: DFMA %lld  DMUL %lld  rsqrt %lld  SHFL64 %lld  DMMA %lld  LDS %lld  bar %lld  div %lld  sqrt %lld  rsqrtf+NR %lld cycles (%s)\n",
           nthr, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9], cudaGetErrorString(cudaGetLastError()));
  }
}
