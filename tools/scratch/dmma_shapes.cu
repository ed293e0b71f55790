// Micro: f64 MMA shape throughput on one SM (independent accumulator chains) and full-GPU rate.
#include <cstdio>
__device__ __forceinline__ void m884(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a[0]), "d"(b[0]));
}
__device__ __forceinline__ void m1684(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
__device__ __forceinline__ void m1688(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void m16816(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
template <int S>
__global__ void k(double* out, long long* cyc, int n) {
  double c[8][4] = {};
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = (threadIdx.x + i) * 1e-3;
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (i + 1);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (S == 0) m884(c[j], a, b);
      else if (S == 1) m1684(c[j], a, b);
      else if (S == 2) m1688(c[j], a, b);
      else m16816(c[j], a, b);
    }
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 64 << 20); cudaMalloc(&c, 8);
  const char* names[] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const double fl[] = {8*8*4*2, 16*8*4*2, 16*8*8*2, 16*8*16*2};
  for (int sh = 0; sh < 4; ++sh) {
    for (int w : {4, 8, 16}) {
      auto f = sh == 0 ? k<0> : sh == 1 ? k<1> : sh == 2 ? k<2> : k<3>;
      f<<<1, 32 * w>>>(o, c, 2000); f<<<1, 32 * w>>>(o, c, 2000);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("%-9s warps %2d: SM rate %.1f flop/clk\n", names[sh], w, 8.0 * 2000 * w * fl[sh] / h);
    }
    auto f = sh == 0 ? k<0> : sh == 1 ? k<1> : sh == 2 ? k<2> : k<3>;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    f<<<148 * 4, 256>>>(o, c, 2000);
    cudaEventRecord(e0); f<<<148 * 4, 256>>>(o, c, 2000); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-9s full GPU: %.1f TFLOP/s\n", names[sh], 148.0 * 4 * 8 * 8 * 2000 * fl[sh] / (ms * 1e-3) / 1e12);
  }
}
