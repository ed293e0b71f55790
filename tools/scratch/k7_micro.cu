#include <cstdio>
#include <vector>
#include <cmath>
#include "../../paper_2401_09703_b200/csrc/common.cuh"
namespace X { using namespace tsvd;
__device__ __forceinline__ double warp_sum2(double v) { for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o); return v; }
constexpr int K7_MAX = 128;
constexpr int K7_SWEEPS = 40;
constexpr int K7_THREADS = 1024;
constexpr int K7_GL = 16;                 // lanes per column pair
constexpr int K7_GPW = 32 / K7_GL;        // pairs per warp

__device__ __forceinline__ int k7_pos(int slot, int step, int N) {  // tournament: slot -> player
  return slot == 0 ? 0 : 1 + (slot - 1 + step) % (N - 1);
}

__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = K7_GL / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(K7_THREADS) jacobi_cta_kernel(const double* __restrict__ A, int64_t lda, int m, int n,
                                                                int kk, double tol, double* __restrict__ theta,
                                                                double* __restrict__ F, int64_t ldf,
                                                                int* __restrict__ info, double* __restrict__ tiny_out, long long* __restrict__ ph) {
  long long tA = 0, tB = 0, tC = 0, tt = 0;
  extern __shared__ double Wsm[];                  // column-major, ld = mp
  __shared__ int rot_count;
  __shared__ double2 rot_s[K7_MAX / 2];
  __shared__ double pc_s[K7_MAX / 2], nrm2_s[K7_MAX];
  __shared__ double nrm_s[K7_MAX + 1];
  __shared__ int rank_s[K7_MAX + 1];
  const int mp = m | 1;                            // odd pitch: conflict-free column walks
  const int N = (n + 1) & ~1;                      // even player count (a zero column if n odd)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane / K7_GL, li = lane % K7_GL;
  for (int e = tid; e < mp * N; e += blockDim.x) {
    const int j = e / mp, i = e % mp;
    Wsm[e] = (i < m && j < n) ? A[(int64_t)j * lda + i] : 0.0;
  }
  __syncthreads();
  int sweep = 0;
  for (; sweep < K7_SWEEPS; ++sweep) {
    if (tid == 0) rot_count = 0;
    for (int j = warp; j < N; j += K7_THREADS / 32) {  // exact squared column norms
      double a = 0.0;
      for (int i = lane; i < m; i += 32) a = fma(Wsm[j * mp + i], Wsm[j * mp + i], a);
      a = warp_sum2(a);
      if (lane == 0) nrm2_s[j] = a;
    }
    __syncthreads();
    int local = 0;
    if (tid == 0) tt = clock64();
    for (int step = 0; step < N - 1; ++step) {
      // (A) every 16-lane group dots its pair (held in registers until (C)); (B) one lane per
      // pair turns (a, b, c) into the rotation, so the divide / square-root chain is issued by
      // two warps instead of all 32; (C) the groups rotate.  N / 2 <= 64 pairs = one per group.
      const int pr = warp * K7_GPW + grp;
      const bool live = pr < N / 2;
      const int p0 = live ? k7_pos(pr, step, N) : 0, q0 = live ? k7_pos(N - 1 - pr, step, N) : 0;
      const int p = min(p0, q0), q = max(p0, q0);
      double* xp = Wsm + p * mp;
      double* xq = Wsm + q * mp;
      constexpr int NU = K7_MAX / K7_GL;
      double u[NU], v[NU];
      double c0 = 0.0, c1 = 0.0;  // two chains
#pragma unroll
      for (int x = 0; x < NU; ++x) {
        const int i = li + K7_GL * x;
        const bool in = live && i < m;
        u[x] = in ? xp[i] : 0.0;
        v[x] = in ? xq[i] : 0.0;
        if (x & 1) c1 = fma(u[x], v[x], c1);
        else c0 = fma(u[x], v[x], c0);
      }
      const double c = group_sum(c0 + c1);
      if (live && li == 0) pc_s[pr] = c;
      __syncthreads();
      if (tid == 0) { long long t1 = clock64(); tA += t1 - tt; tt = t1; }
      // the squared norms are carried through the rotation (a' = a - t c, b' = b + t c) and
      // recomputed exactly at every sweep start, so a round only dots the pair once
      if (tid < N / 2) {
        const int pp = k7_pos(tid, step, N), qq = k7_pos(N - 1 - tid, step, N);
        const int p1 = min(pp, qq), q1 = max(pp, qq);
        const double a = nrm2_s[p1], b = nrm2_s[q1], cc = pc_s[tid];
        double cs = 1.0, sn = 0.0;
        if (a > 0.0 && b > 0.0 && fabs(cc) > tol * sqrt(a * b)) {
          const double zeta = (b - a) / (2.0 * cc);
          const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          cs = rsqrt(1.0 + t * t);
          sn = cs * t;
          nrm2_s[p1] = fma(-t, cc, a);
          nrm2_s[q1] = fma(t, cc, b);
          ++local;
        }
        rot_s[tid] = make_double2(cs, sn);
      }
      __syncthreads();
      if (tid == 0) { long long t1 = clock64(); tB += t1 - tt; tt = t1; }
      if (live) {
        const double2 r = rot_s[pr];
        if (r.y != 0.0) {
#pragma unroll
          for (int x = 0; x < NU; ++x) {
            const int i = li + K7_GL * x;
            if (i < m) {
              xp[i] = r.x * u[x] - r.y * v[x];
              xq[i] = r.y * u[x] + r.x * v[x];
            }
          }
        }
      }
      __syncthreads();
      if (tid == 0) { long long t1 = clock64(); tC += t1 - tt; tt = t1; }
    }
    if (local) atomicAdd(&rot_count, local);
    __syncthreads();
    if (rot_count == 0) break;
    __syncthreads();
  }
  // column norms, descending rank (index tie-break)
  const int nwarps = blockDim.x >> 5;
  for (int j = warp; j < n; j += nwarps) {
    double a = 0.0;
    for (int i = lane; i < m; i += 32) a = fma(Wsm[j * mp + i], Wsm[j * mp + i], a);
    a = warp_sum2(a);
    if (lane == 0) nrm_s[j] = sqrt(a);
  }
  __syncthreads();
  for (int j = tid; j < n; j += blockDim.x) {
    const double v = nrm_s[j];
    int r = 0;
    for (int l = 0; l < n; ++l) r += (nrm_s[l] > v) || (nrm_s[l] == v && l < j);
    rank_s[j] = r;
    theta[r] = v;
  }
  __syncthreads();
  double fro = 0.0;
  for (int j = 0; j < n; ++j) fro = fma(nrm_s[j], nrm_s[j], fro);
  const double tiny = 1e-14 * sqrt(fro) + 1e-300;
  for (int j = warp; j < n; j += nwarps) {
    const int r = rank_s[j];
    if (r >= kk) continue;
    const double inv = nrm_s[j] > tiny ? 1.0 / nrm_s[j] : 0.0;
    for (int i = lane; i < m; i += 32) F[(int64_t)r * ldf + i] = Wsm[j * mp + i] * inv;
  }
  if (tid == 0) { ph[0] = tA; ph[1] = tB; ph[2] = tC; }
  if (tid == 0 && info) {
    info[0] = sweep + 1;
    info[1] = sweep < K7_SWEEPS;
    *tiny_out = tiny;
  }
}
}
int main() {
  const int n = 128;
  std::vector<double> A(n * n);
  for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) A[j * n + i] = (i >= j) ? std::sin(1.0 + (i * n + j) * 0.37 + 0.001 * i * j) * std::pow(0.97, j) : 0.0;
  double *dA, *th, *F, *tiny; int* info; long long* ph;
  cudaMalloc(&dA, n * n * 8); cudaMalloc(&th, n * 8); cudaMalloc(&F, n * n * 8); cudaMalloc(&tiny, 8); cudaMalloc(&info, 16); cudaMalloc(&ph, 64);
  cudaMemcpy(dA, A.data(), n * n * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(X::jacobi_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const size_t smem = (size_t)(n | 1) * n * 8;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    X::jacobi_cta_kernel<<<1, X::K7_THREADS, smem>>>(dA, n, n, n, 64, 1e-14, th, F, n, info, tiny, ph);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int hi[4]; long long hp[3]; cudaMemcpy(hi, info, 16, cudaMemcpyDeviceToHost); cudaMemcpy(hp, ph, 24, cudaMemcpyDeviceToHost);
  printf("%s: %.3f ms, sweeps %d conv %d; cycles A %lld B %lld C %lld; per round A %.0f B %.0f C %.0f\n", cudaGetErrorString(cudaGetLastError()), ms, hi[0], hi[1], hp[0], hp[1], hp[2], hp[0] / (127.0 * hi[0]), hp[1] / (127.0 * hi[0]), hp[2] / (127.0 * hi[0]));
}
