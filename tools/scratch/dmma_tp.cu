// Micro: DMMA.8x8x4 issue throughput per SM sub-partition (8 independent chains per warp).
#include <cstdio>
__device__ __forceinline__ void dm(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k(double* out, long long* cyc, int n) {
  double c[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1e-3;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) dm(c[j][0], c[j][1], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8);
  for (int w : {1, 2, 4, 8, 16}) {
    k<<<1, 32 * w>>>(o, c, 1000);
    k<<<1, 32 * w>>>(o, c, 1000);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warps %2d: %.2f cycles per DMMA per warp; SM rate %.1f FMA/clk\n", w, h / 8000.0, 8000.0 * w * 256 / h);
  }
}
