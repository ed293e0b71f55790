// Micro: phases of potrf_core_t<64, 256> (the tile-DAG chain's diagonal factorisation) on one CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 potrf_phase.cu -o potrf_phase
#include <cstdio>
#include <cmath>
#include <vector>
__device__ long long g_ph[4];
__shared__ long long s_ph[8], s_last;
#ifndef NOMARK
#define POTRF_MARK(i)                          \
  if (threadIdx.x == 0) {                      \
    long long _t = clock64();                  \
    s_ph[i] += _t - s_last;                    \
    s_last = _t;                               \
  }
#endif
#include "../../paper_2401_09703_b200/csrc/potrf.cuh"
using namespace tsvd;
#ifndef PN
#define PN 64
#endif
#ifndef PT
#define PT 256
#endif
constexpr int N = PN, NT = PT, ALDN = 2 * N + 4;

__global__ void __launch_bounds__(NT, 1) k(const double* G, double* R, double* Y, int reps, long long* out, int* flag) {
  extern __shared__ double A[];
  __shared__ int keep[N];
  const double* en = G + N * N;  // diag
  long long tcore = 0, tstore = 0;
  if (threadIdx.x < 8) s_ph[threadIdx.x] = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < N * N; e += NT) {
      const int i = e / N, j = e % N;
      A[i * ALDN + j] = G[e];
      A[i * ALDN + N + j] = i == j ? 1.0 : 0.0;
    }
    __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x == 0) s_last = t0;
    potrf_core_t<N, NT>(A, N, en, 1e-12, keep);
    __syncthreads();
    long long t1 = clock64();
    for (int e = threadIdx.x; e < N * N; e += NT) {
      const int i = e / N, j = e % N;
      __stcg(R + e, j >= i ? A[i * ALDN + j] : 0.0);
      __stcg(Y + e, A[i * ALDN + N + j]);
    }
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(r) : "memory");
    __syncthreads();
    long long t2 = clock64();
    tcore += t1 - t0;
    tstore += t2 - t1;
  }
  if (threadIdx.x == 0) {
    out[0] = tcore / reps;
    out[1] = tstore / reps;
    for (int i = 0; i < 7; ++i) out[2 + i] = s_ph[i] / reps;
  }
}

int main() {
  std::vector<double> h(N * N + N);
  unsigned s = 12345;
  std::vector<double> X(N * 2 * N);
  for (auto& x : X) { s = s * 1664525u + 1013904223u; x = (s >> 8) / 16777216.0 - 0.5; }
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      double a = 0;
      for (int l = 0; l < 2 * N; ++l) a += X[i * 2 * N + l] * X[j * 2 * N + l];
      h[i * N + j] = a;
    }
  for (int i = 0; i < N; ++i) h[N * N + i] = h[i * N + i];
  double *dG, *dR, *dY;
  long long* dout;
  int* flag;
  cudaMalloc(&dG, h.size() * 8);
  cudaMalloc(&dR, N * N * 8);
  cudaMalloc(&dY, N * N * 8);
  cudaMalloc(&dout, 128);
  cudaMalloc(&flag, 4);
  cudaMemcpy(dG, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const int smem = N * ALDN * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int pass = 0; pass < 2; ++pass) {
    long long zero[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_ph, zero, sizeof(zero));
    k<<<1, NT, smem>>>(dG, dR, dY, 50, dout, flag);
    long long o[9];
    cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
    printf("core %lld cycles (%.2f us at 1.965 GHz)  store+release %lld  | %lld %lld %lld %lld %lld %lld %lld (%s)\n",
           o[0], o[0] / 1965.0, o[1], o[2], o[5], o[6], o[7], o[3], o[8], o[4], cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<double> R(N * N), Y(N * N);
  cudaMemcpy(R.data(), dR, N * N * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(Y.data(), dY, N * N * 8, cudaMemcpyDeviceToHost);
  double e = 0, e2 = 0;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      double a = 0, b = 0;
      for (int l = 0; l < N; ++l) { a += R[l * N + i] * R[l * N + j]; b += R[l * N + i] * Y[l * N + j]; }
      e = fmax(e, fabs(a - h[i * N + j]));
      e2 = fmax(e2, fabs(b - (i == j)));
    }
  printf("max |R^T R - G| = %.3e  max |R^T Y - I| = %.3e\n", e, e2);
}
