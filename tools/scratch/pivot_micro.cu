// Micro: latency of the 16-pivot register Cholesky step (one warp) and rsqrt refinement
// accuracy.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pivot_micro pivot_micro.cu
#include <cstdio>
#include <cmath>
#include <vector>

template <int NR>
__device__ __forceinline__ double rsq(double d) {
  double y;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(d));
#pragma unroll
  for (int it = 0; it < NR; ++it) {
    const double e = fma(-d * y, y, 1.0);
    y = fma(0.5 * y, e, y);
  }
  return y;
}
__device__ __forceinline__ double rsq_ftz(double d) {  // approx via float rsqrt + 2 NR
  double y = (double)rsqrtf((float)d);
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const double e = fma(-d * y, y, 1.0);
    y = fma(0.5 * y, e, y);
  }
  return y;
}

template <int V>
__device__ __forceinline__ double rs(double d) {
  if (V == 0) return rsq<2>(d);
  if (V == 1) return rsq<1>(d);
  if (V == 2) return rsq_ftz(d);
  return rsqrt(d);
}

// SM: 16x16 block, lane: column c = lane & 15, rows 2m + p
template <int V, bool SMEMROW>
__global__ void piv_kernel(const double* __restrict__ B, int reps, long long* cyc, double* out) {
  __shared__ double row_s[16];
  const int lane = threadIdx.x, c = lane & 15, p = lane >> 4;
  double acc = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    double a[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) a[m] = B[(2 * m + p) * 16 + c];
    double d = __shfl_sync(0xffffffffu, a[0], 0);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int src = (i & 1) * 16;
      double a01 = 0.0, a11 = 0.0;
      if (i + 1 < 16) {
        a01 = __shfl_sync(0xffffffffu, a[i >> 1], src + i + 1);
        a11 = __shfl_sync(0xffffffffu, a[(i + 1) >> 1], ((i + 1) & 1) * 16 + i + 1);
      }
      const bool kp = d > 1e-300;
      const double y = kp ? rs<V>(d) : 0.0;
      const double r = kp ? d * y : 0.0;
      double ur[8], uc;
      if (SMEMROW) {
        const double aic = a[i >> 1];
        if (p == (i & 1)) row_s[c] = aic * y;
        __syncwarp();
#pragma unroll
        for (int m = 0; m < 8; ++m) ur[m] = row_s[2 * m + p];
        uc = (c > i) ? row_s[c] : (c == i ? r : 0.0);
        __syncwarp();
      } else {
        const double aic = __shfl_sync(0xffffffffu, a[i >> 1], src + c);
#pragma unroll
        for (int m = 0; m < 8; ++m) ur[m] = __shfl_sync(0xffffffffu, a[i >> 1], src + 2 * m + p) * y;
        uc = (c > i) ? aic * y : (c == i ? r : aic);
      }
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int rr = 2 * m + p;
        if (rr > i && c >= rr) a[m] = fma(-ur[m], uc, a[m]);
      }
      if (p == (i & 1)) a[i >> 1] = uc;
      if (i + 1 < 16) {
        const double u = a01 * y;
        d = fma(-u, u, a11);
      }
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) acc += a[m];
  }
  long long t1 = clock64();
  if (lane == 0) *cyc = (t1 - t0) / reps;
  out[lane] = acc;
}

template <int V>
__global__ void acc_kernel(const double* d, int n, double* maxerr) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double y = rs<V>(d[i]);
  double ref = 1.0 / sqrt(d[i]);
  double e = fabs(y - ref) / ref;
  unsigned long long* me = (unsigned long long*)maxerr;
  atomicMax(me, __double_as_longlong(e));
}

int main() {
  std::vector<double> G(256), X(16 * 32);
  for (int i = 0; i < 16 * 32; ++i) X[i] = std::sin(1.0 + i * 0.37 + 0.001 * i * i);
  for (int i = 0; i < 16; ++i) for (int j = 0; j < 16; ++j) { double s = 0; for (int k = 0; k < 32; ++k) s += X[i * 32 + k] * X[j * 32 + k]; G[i * 16 + j] = s; }
  double *dB, *dout; long long* dc;
  cudaMalloc(&dB, 256 * 8); cudaMalloc(&dout, 32 * 8); cudaMalloc(&dc, 8);
  cudaMemcpy(dB, G.data(), 256 * 8, cudaMemcpyHostToDevice);
  long long cyc;
#define RUN(V, S) piv_kernel<V, S><<<1, 32>>>(dB, 200, dc, dout); cudaDeviceSynchronize(); piv_kernel<V, S><<<1, 32>>>(dB, 1000, dc, dout); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost); printf("variant rsqrt=%d smemrow=%d: %lld cycles per 16 pivots (%.1f / pivot)\n", V, S, cyc, cyc / 16.0);
  RUN(0, false) RUN(1, false) RUN(2, false) RUN(3, false) RUN(0, true) RUN(1, true)
  const int n = 1 << 20;
  std::vector<double> h(n);
  for (int i = 0; i < n; ++i) h[i] = std::exp(-300.0 + 600.0 * (i + 0.5) / n) * (1.0 + 0.37 * std::sin(i * 1.7));
  double* dd; double* de; cudaMalloc(&dd, n * 8); cudaMalloc(&de, 8);
  cudaMemcpy(dd, h.data(), n * 8, cudaMemcpyHostToDevice);
#define ACC(V) cudaMemset(de, 0, 8); acc_kernel<V><<<n / 256, 256>>>(dd, n, de); { double e; cudaMemcpy(&e, de, 8, cudaMemcpyDeviceToHost); printf("rsqrt variant %d: max rel err %.3e\n", V, e); }
  ACC(0) ACC(1) ACC(2) ACC(3)
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
