// Latency probe (dependent chains, one warp / one CTA): fp64 ops, shuffles, barriers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_latency tools/probe_latency.cu  (profiles/r2_probe_fp64_latency.txt)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double x0) {
  __shared__ double sm[1024];
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0, t1;
  int tid = threadIdx.x;
  sm[tid] = x;
  __syncthreads();
#define MEAS(idx, body) t0 = clock64(); for (int i = 0; i < n; ++i) { body; } t1 = clock64(); if (tid == 0) cyc[idx] = (t1 - t0) / n;
  MEAS(0, x = fma(x, y, 1e-300));
  MEAS(1, x = x + y);
  MEAS(2, x = x * y);
  MEAS(3, x = sqrt(x + 1.0));
  MEAS(4, x = 1.0 / (x + 1.0));
  MEAS(5, x = __shfl_sync(0xffffffffu, x, (tid + 1) & 31));
  MEAS(6, x = sm[(tid + (int)(x > 1e300)) & 1023] + x * 1e-300);
  MEAS(7, __syncthreads(); x = x + sm[tid & 1023] * 1e-300);
  MEAS(8, x = rsqrt(x + 1.0));
  MEAS(9, x = log(x + 2.0));
  MEAS(10, { float f = (float)x; f = f * 1.0001f + 1e-30f; x = (double)f; });
  MEAS(11, x = fmax(x, y) * 0.5 + (x > y ? 1e-300 : 0.0));
  out[tid] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 16);
  const char* names[] = {"dfma", "dadd", "dmul", "dsqrt", "ddiv(rcp)", "shfl64", "lds64", "syncthreads+lds", "drsqrt", "dlog", "f32 fma+cvt", "dmax/cmp"};
  for (int nt : {32, 1024}) {
    k<<<1, nt>>>(o, c, 1000, 1.5);
    k<<<1, nt>>>(o, c, 1000, 1.5);
    cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h, c, 8 * 12, cudaMemcpyDeviceToHost);
    printf("threads %d\n", nt);
    for (int i = 0; i < 12; ++i) printf("  %-18s %lld cycles/op\n", names[i], h[i]);
  }
  return 0;
}
