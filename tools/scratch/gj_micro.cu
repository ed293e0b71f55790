#include <cstdio>
#include <cmath>
#include "../../paper_2401_09703_b200/csrc/common.cuh"
using namespace tsvd;
constexpr int GJ_SMEM_K = 96;
__global__ void __launch_bounds__(1024) gj_smem_kernel(const double* __restrict__ M, int k, double* __restrict__ Minv,
                                                       double* __restrict__ cond) {
  pdl_begin();
  extern __shared__ double aug_s[];  // k x (2k + 1)
  __shared__ double fac[GJ_SMEM_K];
  __shared__ double red_v[32];
  __shared__ int piv;
  __shared__ double pval;
  __shared__ int singular;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5;
  const int k2 = 2 * k, ld = k2 + 1;
  for (int e = tid; e < k * k2; e += nt) {
    const int i = e / k2, j = e - i * k2;
    aug_s[i * ld + j] = (j < k) ? M[i * k + j] : (j - k == i ? 1.0 : 0.0);
  }
  if (tid == 0) singular = 0;
  double cmax = 0.0;
  for (int j = tid; j < k; j += nt) {
    double a = 0.0;
    for (int i = 0; i < k; ++i) a += fabs(M[i * k + j]);
    cmax = fmax(cmax, a);
  }
  cmax = warp_max(cmax);
  if (lane == 0) red_v[w] = cmax;
  __syncthreads();
  double norm1 = 0.0;
  for (int i = 0; i < (nt + 31) / 32; ++i) norm1 = fmax(norm1, red_v[i]);
  // fixed map: column j = tid % k2, rows tid / k2 + q * rstep
  const int jj = tid % k2, r0 = tid / k2, rstep = nt / k2;
  const bool active = r0 < rstep;
  long long T[5] = {0,0,0,0,0}, t0 = clock64();
#define MK(i) if (tid == 0) { long long t1 = clock64(); T[i] += t1 - t0; t0 = t1; }
  for (int c = 0; c < k; ++c) {
    if (w == 0) {  // pivot search (first maximum, as gj_kernel)
      double best = -1.0;
      int bi = c;
      for (int r = c + lane; r < k; r += 32) {
        const double a = fabs(aug_s[r * ld + c]);
        if (a > best) { best = a; bi = r; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) {
        piv = bi;
        pval = 1.0 / aug_s[bi * ld + c];  // the reciprocal once, not in all 1024 threads
        if (!(best > 0.0)) singular = 1;
      }
    }
    __syncthreads();
    MK(0)
    if (singular) break;
    const int pr = piv;
    const double inv = pval;
    for (int j = tid; j < k2; j += nt) {
      const double a = aug_s[c * ld + j], b = aug_s[pr * ld + j];
      if (pr != c) aug_s[pr * ld + j] = a;
      aug_s[c * ld + j] = b * inv;
    }
    __syncthreads();
    MK(1)
    for (int r = tid; r < k; r += nt) fac[r] = (r == c) ? 0.0 : aug_s[r * ld + c];
    __syncthreads();
    MK(2)
    if (active) {
      // eight rows at a time: all loads, then the fmas and stores — a row at a time the
      // compiler cannot move the next row's load above this row's store (same shared array),
      // and every update paid the full load -> fma -> store latency (~140 cycles)
      const double pc = aug_s[c * ld + jj];
      for (int r1 = r0; r1 < k; r1 += 8 * rstep) {
        double f[8], x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int r = r1 + u * rstep;
          f[u] = r < k ? fac[r] : 0.0;
          x[u] = r < k ? aug_s[r * ld + jj] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int r = r1 + u * rstep;
          if (r < k && f[u] != 0.0) aug_s[r * ld + jj] = x[u] - f[u] * pc;
        }
      }
    }
    __syncthreads();
    MK(3)
  }
  if (tid == 0) printf("per pivot: search+bar %lld  swap+bar %lld  fac+bar %lld  update+bar %lld cycles\n", T[0]/k, T[1]/k, T[2]/k, T[3]/k);
  if (singular) {
    if (tid == 0) *cond = INFINITY;
    return;
  }
  for (int e = tid; e < k * k; e += nt) {
    const int i = e / k, j = e - i * k;
    Minv[e] = aug_s[i * ld + k + j];
  }
  double imax = 0.0;
  for (int j = tid; j < k; j += nt) {
    double a = 0.0;
    for (int i = 0; i < k; ++i) a += fabs(aug_s[i * ld + k + j]);
    imax = fmax(imax, a);
  }
  imax = warp_max(imax);
  __syncthreads();
  if (lane == 0) red_v[w] = imax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < (nt + 31) / 32; ++i) m = fmax(m, red_v[i]);
    *cond = norm1 * m;
  }
}

int main() {
  const int k = 64;
  static double h[k * k];
  for (int i = 0; i < k * k; ++i) h[i] = ((i * 7919) % 1000) / 1000.0 - 0.5 + ((i % (k + 1)) == 0 ? 2.0 : 0.0);
  double *M, *Mi, *c;
  cudaMalloc(&M, sizeof(h)); cudaMalloc(&Mi, sizeof(h)); cudaMalloc(&c, 8);
  cudaMemcpy(M, h, sizeof(h), cudaMemcpyHostToDevice);
  const int smem = k * (2 * k + 1) * 8;
  cudaFuncSetAttribute(gj_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  gj_smem_kernel<<<1, 1024, smem>>>(M, k, Mi, c);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  gj_smem_kernel<<<1, 1024, smem>>>(M, k, Mi, c);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("kernel %.1f us (%s)\n", ms * 1e3, cudaGetErrorString(cudaGetLastError()));
}
