// micro-benchmarks (not part of the library): barrier cost and a flat 128x128 Cholesky
#include <cstdio>
#include <cuda_runtime.h>
__global__ void bar_loop(int n, double* out) {
  double a = threadIdx.x;
  for (int i = 0; i < n; ++i) { a = a * 1.0000001 + 1e-9; __syncthreads(); }
  if (a == 12345.0) out[0] = a;
}
__global__ void __launch_bounds__(1024) chol_flat(double* G, int l) {
  extern __shared__ double A[];
  const int LD = 129, tid = threadIdx.x, c = tid & 127, r0 = tid >> 7;
  __shared__ double rinv;
  for (int e = tid; e < 128 * 128; e += 1024) { int r = e >> 7, cc = e & 127; A[r * LD + cc] = G[e]; }
  __syncthreads();
  for (int i = 0; i < l; ++i) {
    if (tid == 0) { double d = A[i * LD + i]; double r = sqrt(d); A[i * LD + i] = r; rinv = 1.0 / r; }
    __syncthreads();
    if (tid > i && tid < l) A[i * LD + tid] *= rinv;
    __syncthreads();
    if (c > i && c < l) {
      const double ric = A[i * LD + c];
#pragma unroll
      for (int q = 0; q < 16; ++q) { const int r = r0 + 8 * q; if (r > i && r <= c) A[r * LD + c] -= A[i * LD + r] * ric; }
    }
    __syncthreads();
  }
  for (int e = tid; e < 128 * 128; e += 1024) { int r = e >> 7, cc = e & 127; G[e] = A[r * LD + cc]; }
}
// 2-D mapping with explicit ILP: all loads first, then FMAs, then stores
__global__ void __launch_bounds__(1024) chol_ilp(double* G, int l) {
  extern __shared__ double A[];
  const int LD = 129, tid = threadIdx.x, c = tid & 127, r0 = tid >> 7;
  __shared__ double rinv;
  for (int e = tid; e < 128 * 128; e += 1024) { int r = e >> 7, cc = e & 127; A[r * LD + cc] = G[e]; }
  __syncthreads();
  for (int i = 0; i < l; ++i) {
    if (tid == 0) { double d = A[i * LD + i]; double r = sqrt(d); A[i * LD + i] = r; rinv = 1.0 / r; }
    __syncthreads();
    if (tid > i && tid < l) A[i * LD + tid] *= rinv;
    __syncthreads();
    if (c > i && c < l) {
      const double ric = A[i * LD + c];
      double ar[16], rc[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) { const int r = r0 + 8 * q; ar[q] = A[i * LD + r]; rc[q] = A[r * LD + c]; }
#pragma unroll
      for (int q = 0; q < 16; ++q) { const int r = r0 + 8 * q; if (r > i && r <= c) A[r * LD + c] = rc[q] - ar[q] * ric; }
    }
    __syncthreads();
  }
  for (int e = tid; e < 128 * 128; e += 1024) { int r = e >> 7, cc = e & 127; G[e] = A[r * LD + cc]; }
}
// only pivots + scale (no update) to isolate the serial part
__global__ void __launch_bounds__(1024) chol_noupd(double* G, int l) {
  extern __shared__ double A[];
  const int LD = 129, tid = threadIdx.x;
  __shared__ double rinv;
  for (int e = tid; e < 128 * 128; e += 1024) { int r = e >> 7, cc = e & 127; A[r * LD + cc] = G[e]; }
  __syncthreads();
  for (int i = 0; i < l; ++i) {
    if (tid == 0) { double d = A[i * LD + i]; double r = sqrt(d); A[i * LD + i] = r; rinv = 1.0 / r; }
    __syncthreads();
    if (tid > i && tid < l) A[i * LD + tid] *= rinv;
    __syncthreads();
    __syncthreads();
  }
  for (int e = tid; e < 128 * 128; e += 1024) { int r = e >> 7, cc = e & 127; G[e] = A[r * LD + cc]; }
}
int main() {
  double* d; cudaMalloc(&d, 128 * 128 * 8);
  double h[128 * 128];
  for (int i = 0; i < 128; ++i) for (int j = 0; j < 128; ++j) h[i * 128 + j] = (i == j) ? 200.0 : 1.0 / (1 + i + j);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int th : {128, 256, 1024}) {
    bar_loop<<<1, th>>>(10, d); cudaDeviceSynchronize();
    cudaEventRecord(e0); bar_loop<<<1, th>>>(10000, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("barrier threads %d: %.1f ns per iteration\n", th, ms * 1e6 / 10000);
  }
  cudaFuncSetAttribute(chol_flat, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaEventRecord(e0); chol_flat<<<1, 1024, 128 * 129 * 8>>>(d, 128); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("chol_flat 128: %.1f us (%s)\n", ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(chol_ilp, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  cudaFuncSetAttribute(chol_noupd, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaEventRecord(e0); chol_ilp<<<1, 1024, 128 * 129 * 8>>>(d, 128); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("chol_ilp 128: %.1f us\n", ms * 1e3);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaEventRecord(e0); chol_noupd<<<1, 1024, 128 * 129 * 8>>>(d, 128); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("chol_noupd 128: %.1f us\n", ms * 1e3);
  }
  return 0;
}
