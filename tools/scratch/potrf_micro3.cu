#include <cstdio>
#include <vector>
#include <cmath>
#include "../../paper_2401_09703_b200/csrc/common.cuh"
namespace X { using namespace tsvd;

constexpr int TB = 64;         // tile
constexpr int TP = TB + 8;     // smem pitch of [k][m] operands (== 8 mod 16: conflict-free fragments)
constexpr int SUB = 16;        // sub-panel of the diagonal factorisation
constexpr int DAG_THREADS = 256;
// [A | I] factor tile (TB x (2 TB + 4)) + one operand tile; the bulk uses two operand tiles
constexpr size_t DAG_SMEM = ((size_t)TB * (2 * TB + 4) + (size_t)TB * TP) * sizeof(double);

constexpr int ALD = 2 * TB + 4;  // pitch of [A | I] (== 4 mod 16)

// [A | I] <- the diagonal tile at D (upper part; identity padding for pivots >= nb)
__device__ __forceinline__ void potrf_load(double* A, const double* D, int64_t ld, int nb) {
  const int tid = threadIdx.x;
  {
    const int c = tid & (TB - 1), r0 = tid >> 6;
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int r = r0 + 4 * u;
      v[u] = (r < nb && c < nb && c >= r) ? __ldcg(D + (int64_t)r * ld + c) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int r = r0 + 4 * u;
      A[r * ALD + c] = (r < nb && c < nb) ? v[u] : (r == c ? 1.0 : 0.0);
      A[r * ALD + TB + c] = (r == c) ? 1.0 : 0.0;
    }
  }
}

// [A | I] <- a warp-fragment accumulator holding the (updated) diagonal tile
__device__ __forceinline__ void potrf_from_acc(double* A, const double (&acc)[2][4][2], int nb, int rb, int cb) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int r = rb + 8 * x + g, c = cb + 8 * y + 2 * t + z;
        A[r * ALD + c] = (r < nb && c < nb) ? (c >= r ? acc[x][y][z] : 0.0) : (r == c ? 1.0 : 0.0);
      }
  for (int e = threadIdx.x; e < TB * TB; e += DAG_THREADS) {
    const int r = e >> 6, c = e & (TB - 1);
    A[r * ALD + TB + c] = (r == c) ? 1.0 : 0.0;
  }
}

template <int V> __device__ void potrf_core(int mask, double* A, int nb, const double* __restrict__ en, double tau, int32_t* __restrict__ keep) {
  __shared__ double rinv[TB], en_s[TB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  if (tid < TB) en_s[tid] = tid < nb ? en[tid] : 1.0;
  __syncthreads();
  for (int j0 = 0; j0 < TB; j0 += SUB) {
    const int j1 = j0 + SUB;
    if ((mask & 1) && warp == 0) {
      const int c = lane & 15, p = lane >> 4;
      double a[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = A[(j0 + 2 * m + p) * ALD + j0 + c];
      // the next pivot's Schur diagonal is formed redundantly in every lane from values read
      // before this pivot's update (same fma as the owning lane's update), so the sequential
      // chain per pivot is rsqrt + two flops rather than a shuffle round trip through the update
      double d = __shfl_sync(0xffffffffu, a[0], 0);
      double myy = 0.0;
      int mykp = 0;
#pragma unroll
      for (int i = 0; i < SUB; ++i) {
        const int src = (i & 1) * 16;
        double a01 = 0.0, a11 = 0.0;
        if (i + 1 < SUB) {
          a01 = __shfl_sync(0xffffffffu, a[i >> 1], src + i + 1);
          a11 = __shfl_sync(0xffffffffu, a[(i + 1) >> 1], ((i + 1) & 1) * 16 + i + 1);
        }
        const int gi = j0 + i;
        const bool real = gi < nb;
        const double e = en_s[gi];
        const bool kp = real && !(e == 0.0 || d <= tau * e);
        // rsqrt of a safe argument, unconditionally, then a select: a conditional call makes the
        // compiler branch around the (warp-uniform) pivot chain, ~100 cycles per pivot
        const double y0 = rsqrt(kp ? d : 1.0);
        const double y = kp ? y0 : (real ? 0.0 : 1.0);
        const double r = kp ? d * y : (real ? 0.0 : 1.0);
        const double aic = __shfl_sync(0xffffffffu, a[i >> 1], src + c);
        double ur[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) ur[m] = __shfl_sync(0xffffffffu, a[i >> 1], src + 2 * m + p) * y;
        const double uc = (c > i) ? aic * y : (c == i ? r : aic);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const int rr = 2 * m + p;
          if (rr > i && c >= rr) a[m] = fma(-ur[m], uc, a[m]);
        }
        if (p == (i & 1)) a[i >> 1] = uc;
        if (i + 1 < SUB) {
          const double u = a01 * y;
          d = fma(-u, u, a11);
        }
        // no divergent stores inside the pivot chain: lane i keeps pivot i's results
        if (lane == i) {
          myy = y;
          mykp = kp;
        }
      }
      if (lane < SUB) {
        rinv[j0 + lane] = myy;
        if (j0 + lane < nb) keep[j0 + lane] = mykp;
      }
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int rr = 2 * m + p;
        if (c >= rr) A[(j0 + rr) * ALD + j0 + c] = a[m];
      }
    }
    __syncthreads();
    // row block: rows j0..j1 of the columns j1..63 of A and 64..64+j1 of [I] (64 columns)
    if ((mask & 2) && tid < TB) {
      const int col = tid < TB - j1 ? j1 + tid : TB + (tid - (TB - j1));
      // right-looking within the 16 rows: the chain per row is one multiply + one fma (the
      // same fmas in the same order as the dot-product form)
      double v[SUB];
#pragma unroll
      for (int q = 0; q < SUB; ++q) v[q] = A[(j0 + q) * ALD + col];
#pragma unroll
      for (int q = 0; q < SUB; ++q) {
        const double x = v[q] * rinv[j0 + q];
        A[(j0 + q) * ALD + col] = x;
#pragma unroll
        for (int q2 = q + 1; q2 < SUB; ++q2) v[q2] = fma(-A[(j0 + q) * ALD + j0 + q2], x, v[q2]);
      }
    }
    __syncthreads();
    if ((mask & 4) && j1 < TB) {
      // trailing: A[j1:, j1:] (upper tiles) and the right block rows j1.., columns < j1
      const int ntl = (TB - j1) / 8, nup = ntl * ntl, nright = ntl * (j1 / 8);
      for (int tile = warp; tile < nup + nright; tile += DAG_THREADS / 32) {
        int r0, c0;
        if (tile < nup) {
          const int tr = tile / ntl, tc = tile % ntl;
          if (tr > tc) continue;
          r0 = j1 + tr * 8;
          c0 = j1 + tc * 8;
        } else {
          const int x = tile - nup, nc = j1 / 8;
          r0 = j1 + (x / nc) * 8;
          c0 = TB + (x % nc) * 8;
        }
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < SUB; kk += 4)
          dmma8x8x4(a0, a1, A[(j0 + kk + t) * ALD + r0 + g], A[(j0 + kk + t) * ALD + c0 + g]);
        const int r = r0 + g, c = c0 + 2 * t;
        if (c0 >= TB || r <= c) A[r * ALD + c] -= a0;
        if (c0 >= TB || r <= c + 1) A[r * ALD + c + 1] -= a1;
      }
      __syncthreads();
    }
  }
}

// R (upper, zero below) -> D; Y = R^{-T} (zero-padded) -> Yq
__device__ __forceinline__ void potrf_store(const double* A, double* D, int64_t ld, int nb, double* __restrict__ Yq) {
  const int tid = threadIdx.x;
  {
    const int c = tid & (TB - 1), r0 = tid >> 6;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int r = r0 + 4 * u;
      if (r < nb && c < nb) __stcg(D + (int64_t)r * ld + c, c >= r ? A[r * ALD + c] : 0.0);
      __stcg(Yq + r * TB + c, (r < nb && c < nb) ? A[r * ALD + TB + c] : 0.0);
    }
  }
}


template <int V> __global__ void kern(int mask, double* D, const double* en, int32_t* keep, double* T, long long* stamps) {
  extern __shared__ double sm[];
  potrf_load(sm, D, 64, 64);
  __syncthreads();
  long long t0 = clock64();
  potrf_core<V>(mask, sm, 64, en, 1e-12, keep);
  __syncthreads();
  long long t1 = clock64();
  potrf_store(sm, D, 64, 64, T);
  if (threadIdx.x == 0) { stamps[6] = t0; stamps[7] = t1; }
}
}
int main() {
  const int n = 64;
  std::vector<double> B(n * 2 * n), G(n * n, 0.0), en(n);
  for (size_t i = 0; i < B.size(); ++i) B[i] = std::sin(1.0 + i * 0.37 + 0.001 * i * i);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double s = 0; for (int k = 0; k < 2 * n; ++k) s += B[i * 2 * n + k] * B[j * 2 * n + k]; G[i * n + j] = s; }
  for (int i = 0; i < n; ++i) en[i] = G[i * n + i];
  double *dD, *dE, *dT; int32_t* dk; long long* ds;
  cudaMalloc(&dD, n * n * 8); cudaMalloc(&dE, n * 8); cudaMalloc(&dT, n * n * 8); cudaMalloc(&dk, n * 4); cudaMalloc(&ds, 64 * 8);
  cudaMemcpy(dE, en.data(), n * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(X::kern<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110000);
  cudaFuncSetAttribute(X::kern<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110000);
  cudaFuncSetAttribute(X::kern<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110000);
  long long st[64];
  for (int variant = 0; variant < 3; ++variant)
  for (int mask : {7, 1, 0}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemcpy(dD, G.data(), n * n * 8, cudaMemcpyHostToDevice);
      if (variant == 0) X::kern<0><<<1, 256, 110000>>>(mask, dD, dE, dk, dT, ds);
      else if (variant == 1) X::kern<1><<<1, 256, 110000>>>(mask, dD, dE, dk, dT, ds);
      else X::kern<2><<<1, 256, 110000>>>(mask, dD, dE, dk, dT, ds);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(st, ds, 64 * 8, cudaMemcpyDeviceToHost);
    printf("variant %d mask %d (1 pivots, 2 rowblk, 4 trailing): core %lld cycles\n", variant, mask, st[7] - st[6]);
    if (mask == 7) {
      std::vector<double> R(n*n), Y(n*n); cudaMemcpy(R.data(), dD, n*n*8, cudaMemcpyDeviceToHost); cudaMemcpy(Y.data(), dT, n*n*8, cudaMemcpyDeviceToHost);
      double e = 0; for (int i = 0; i < n; ++i) for (int j = i; j < n; ++j) { double s = 0; for (int k = 0; k <= i; ++k) s += R[k*n+i]*R[k*n+j]; e = std::fmax(e, std::fabs(s - G[i*n+j])); }
      double e2 = 0; for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double s = 0; for (int k = 0; k < n; ++k) s += R[k*n+i]*Y[k*n+j]; e2 = std::fmax(e2, std::fabs(s - (i==j))); }
      printf("  max |R^T R - G| = %.3e   max |R^T Y - I| = %.3e  (%s)\n", e, e2, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
