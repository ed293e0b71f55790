// Micro: FP64 FMA (non-tensor) and fp64 division issue throughput on one SM.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int n, int mode) {
  double c[8];
  for (int j = 0; j < 8; ++j) c[j] = threadIdx.x * 1e-3 + j;
  const double a = 1.0000001, b = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0) {
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = fma(c[j], a, b);
  } else {
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = 1.0 / (c[j] + 1.5);
  }
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8);
  for (int mode = 0; mode < 2; ++mode)
    for (int w : {1, 4, 8, 32}) {
      k<<<1, 32 * w>>>(o, c, 200, mode); k<<<1, 32 * w>>>(o, c, 200, mode);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("%s warps %2d: %.2f cycles per warp-op; SM rate %.2f lane-ops/clk\n", mode ? "div " : "dfma", w, h / 1600.0, 1600.0 * 32 * w / h);
    }
}
