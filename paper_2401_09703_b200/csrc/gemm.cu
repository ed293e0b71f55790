// gemm.cu — K4: small-dense FP64 GEMM / SYRK on the DMMA tensor path (mma.sync m8n8k4 f64).
//
// Used for every dense step of the update: the lift epilogue C0^T = W M_X (Eq (5)
// P:325, App E note P:1083), the SV-LCOV Gram  E E^T - C0^T C0 (Lemma 2), the
// Cholesky trailing update, the weight-update core L_D L_E^T (Alg 4 line 3 P:381-390),
// the multiplier products M F[:k] / M (G[:k] - C G[k:]) (Alg 9 lines 3, 6 P:1196/1199)
// and the new-row block F[k:] M^{-1} (Alg 9 line 4 P:1197).
//
// B200 has no tcgen05 f64 kind; FP64 tensor work is the legacy DMMA path.
// Tile 64x64x16, 4 warps in 2x2, each warp 32x32 = 4x4 DMMA tiles, operands staged in
// shared memory with a 68-double row pitch (conflict-free 64-bit fragment loads),
// register double-buffering of the next K tile.
#include <algorithm>

#include "ops.h"

namespace tsvd {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, LDS = BM + 4;

// blockIdx.z = split-K slice: this CTA sums k in [z kchunk, (z+1) kchunk); with split-K
// the caller passes a partial buffer as C (alpha = 1, beta = 0, C.p offset by z).
template <bool UPPER>
__global__ void __launch_bounds__(128) dgemm_kernel(int64_t M, int64_t N, int64_t Ktot, int64_t kchunk, double alpha,
                                                    CMat A, CMat B, double beta, Mat C, int64_t zstride) {
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t K = min(Ktot - kbeg, kchunk);
  A.p += kbeg * A.cs;
  B.p += kbeg * B.rs;
  C.p += (int64_t)blockIdx.z * zstride;
  if (UPPER && m0 > n0 + BN - 1) return;  // tile strictly below the diagonal
  __shared__ __align__(16) double As[BK][LDS];  // [k][m]
  __shared__ __align__(16) double Bs[BK][LDS];  // [k][n]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // per-thread load coordinates (8 elements of A and of B per K tile)
  const bool a_mfast = (A.rs == 1);  // m contiguous in memory
  const bool b_nfast = (B.cs == 1);  // n contiguous in memory
  double ra[8], rb[8];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int idx = tid + e * 128;
      int mm, kk;
      if (a_mfast) { mm = idx & 63; kk = idx >> 6; } else { kk = idx & 15; mm = idx >> 4; }
      int64_t gm = m0 + mm, gk = k0 + kk;
      ra[e] = (gm < M && gk < K) ? A.p[gm * A.rs + gk * A.cs] : 0.0;
      int nn, kb;
      if (b_nfast) { nn = idx & 63; kb = idx >> 6; } else { kb = idx & 15; nn = idx >> 4; }
      int64_t gn = n0 + nn, gkb = k0 + kb;
      rb[e] = (gn < N && gkb < K) ? B.p[gkb * B.rs + gn * B.cs] : 0.0;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int idx = tid + e * 128;
      int mm, kk;
      if (a_mfast) { mm = idx & 63; kk = idx >> 6; } else { kk = idx & 15; mm = idx >> 4; }
      As[kk][mm] = ra[e];
      int nn, kb;
      if (b_nfast) { nn = idx & 63; kb = idx >> 6; } else { kb = idx & 15; nn = idx >> 4; }
      Bs[kb][nn] = rb[e];
    }
  };

  load(0);
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
    store();
    __syncthreads();
    if (k0 + BK < K) load(k0 + BK);  // overlaps the global latency with the MMAs below
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk + t][wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk + t][wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + wm + i * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t col = n0 + wn + j * 8 + 2 * t + h;
        if (col >= N || (UPPER && row > col)) continue;
        double* c = C.p + row * C.rs + col * C.cs;
        double v = alpha * acc[i][j][h];
        if (beta != 0.0) v += beta * (*c);
        *c = v;
      }
    }
  }
}
// C = alpha sum_z part[z] + beta C  (part: nz slices of M x N row-major)
template <bool UPPER>
__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int nz, const double* __restrict__ part, double alpha,
                                     double beta, Mat C) {
  const int64_t mn = M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < mn; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / N, j = e % N;
    if (UPPER && i > j) continue;
    double acc = 0.0;
    for (int z = 0; z < nz; ++z) acc += part[(int64_t)z * mn + e];
    double* c = C.p + i * C.rs + j * C.cs;
    double v = alpha * acc;
    if (beta != 0.0) v += beta * (*c);
    *c = v;
  }
}
}  // namespace

cudaError_t dgemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, CMat A, CMat B, double beta,
                  Mat C, int uplo) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  dim3 grid(cdiv(M, BM), cdiv(N, BN));
  if (grid.y > 65535) return cudaErrorInvalidValue;
  const int64_t tiles = (int64_t)grid.x * grid.y;
  // split-K for tall-skinny products (few output tiles, long K): deterministic two-pass
  int nz = 1;
  if (tiles < 148 && K >= 2048) nz = (int)std::min<int64_t>(std::min<int64_t>(cdiv(296, tiles), K / 1024), 64);
  if (nz > 1) {
    const int64_t kchunk = ((K + nz - 1) / nz + BK - 1) / BK * BK;
    nz = (int)cdiv(K, kchunk);
    double* part = nullptr;
    cudaError_t e = cudaMallocAsync(&part, (size_t)nz * M * N * sizeof(double), st);
    if (e) return e;
    grid.z = nz;
    g_launches += 2;
    if (uplo)
      dgemm_kernel<true><<<grid, 128, 0, st>>>(M, N, K, kchunk, 1.0, A, B, 0.0, Mat{part, N, 1}, M * N);
    else
      dgemm_kernel<false><<<grid, 128, 0, st>>>(M, N, K, kchunk, 1.0, A, B, 0.0, Mat{part, N, 1}, M * N);
    const unsigned rb = (unsigned)std::min<int64_t>(cdiv(M * N, 256), 148 * 8);
    if (uplo)
      splitk_reduce_kernel<true><<<rb, 256, 0, st>>>(M, N, nz, part, alpha, beta, C);
    else
      splitk_reduce_kernel<false><<<rb, 256, 0, st>>>(M, N, nz, part, alpha, beta, C);
    cudaFreeAsync(part, st);
    return cudaGetLastError();
  }
  ++g_launches;
  if (uplo)
    dgemm_kernel<true><<<grid, 128, 0, st>>>(M, N, K, K, alpha, A, B, beta, C, 0);
  else
    dgemm_kernel<false><<<grid, 128, 0, st>>>(M, N, K, K, alpha, A, B, beta, C, 0);
  return cudaGetLastError();
}

cudaError_t dgemm_rm(cudaStream_t st, bool tA, bool tB, int64_t M, int64_t N, int64_t K, double alpha,
                     const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                     int64_t ldc, int uplo) {
  CMat a = tA ? CMat{A, 1, lda} : CMat{A, lda, 1};
  CMat b = tB ? CMat{B, 1, ldb} : CMat{B, ldb, 1};
  return dgemm(st, M, N, K, alpha, a, b, beta, Mat{C, ldc, 1}, uplo);
}

}  // namespace tsvd
