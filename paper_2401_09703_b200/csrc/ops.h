// ops.h — host-side launchers of the libtsvd kernels (internal; C++ linkage).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace tsvd {

// Number of kernels this library launched on the calling thread (reported in
// tsvd_stats.launches and by bench.py as gpu_launches).
extern thread_local long long g_launches;

// Device-resident CSR of s update vectors of length dim.
struct DevCSR {
  int64_t s = 0, dim = 0, nnz = 0;
  const int64_t* row_ptr = nullptr;
  const int32_t* col_idx = nullptr;
  const double* val = nullptr;
};

// Device CSC (the transpose) restricted to the touched columns J.
struct DevCSC {
  int64_t nJ = 0;           // |J| (host copy)
  int64_t* colptr = nullptr;  // dim+1 (over all columns)
  int32_t* J = nullptr;       // touched columns, ascending, nJ entries (device)
  int32_t* row = nullptr;     // nnz: row (update-vector) index
  double* val = nullptr;      // nnz
};

// Simple stream-ordered scratch arena: every allocation made between mark() and
// release() is freed by release().
struct Scratch {
  cudaStream_t st;
  void* ptrs[128];
  int n = 0;
  cudaError_t err = cudaSuccess;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMallocAsync(&p, count * sizeof(T), st);
    if (e != cudaSuccess) { err = e; return nullptr; }
    if (n < 128) ptrs[n++] = p;
    return static_cast<T*>(p);
  }
  void release() {
    for (int i = 0; i < n; ++i) cudaFreeAsync(ptrs[i], st);
    n = 0;
  }
  ~Scratch() { release(); }
};

// ---- gemm.cu
cudaError_t dgemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, double alpha, CMat A, CMat B,
                  double beta, Mat C, int uplo);
// row-major convenience: C(MxN, ldc) = alpha op(A) op(B) + beta C
cudaError_t dgemm_rm(cudaStream_t st, bool tA, bool tB, int64_t M, int64_t N, int64_t K, double alpha,
                     const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                     int64_t ldc, int uplo = 0);

// ---- sparse.cu
cudaError_t validate_csr(cudaStream_t st, const DevCSR& E, int* d_flag);
cudaError_t build_csc(cudaStream_t st, const DevCSR& E, DevCSC& out, Scratch& ws, int64_t* h_nJ);
cudaError_t gather_spmm(cudaStream_t st, const DevCSR& E, const double* X, int k, double* W);
cudaError_t sparse_gram(cudaStream_t st, const DevCSR& E, const DevCSC& C, double* G, Scratch& ws);
cudaError_t scatter_add(cudaStream_t st, const DevCSC& C, int64_t nnz, const double* Z, int k, double* X);
cudaError_t row_sqnorms(cudaStream_t st, const DevCSR& E, double* out);

// ---- dense.cu
cudaError_t chol_deflate(cudaStream_t st, double* G, int64_t s, const double* enorm2, double tau,
                         int32_t* keep);
cudaError_t trsm_upper(cudaStream_t st, const double* R, int64_t s, const int32_t* keep, double* X, int k);
cudaError_t inverse_gj(cudaStream_t st, const double* M, int k, double* Minv, double* cond, Scratch& ws);
cudaError_t materialize_rows(cudaStream_t st, double* X, int64_t rows, int k, const double* M);
cudaError_t set_identity(cudaStream_t st, double* M, int k);
cudaError_t compact_keep(cudaStream_t st, const int32_t* keep, int64_t s, int32_t* kidx, int64_t* d_r,
                         Scratch& ws);
cudaError_t copy_diag(cudaStream_t st, const double* G, int64_t s, double* d);
cudaError_t build_core_rows(cudaStream_t st, int k, int64_t s, int64_t r, const double* Sigma,
                            const double* P0, const double* R, const int32_t* kidx, double* K);
cudaError_t build_lift_block(cudaStream_t st, int k, int64_t s, int64_t r, const double* P0,
                             const double* R, const int32_t* kidx, double* L);
cudaError_t add_diag_sigma(cudaStream_t st, double* K, int64_t ldk, int k, const double* Sigma,
                           bool colmajor);
cudaError_t expand_rows(cudaStream_t st, const double* Gc, int64_t ldg, int k, int64_t s, const int32_t* kidx,
                        double* Gfull);
cudaError_t colmajor_to_rowmajor(cudaStream_t st, const double* A, int64_t lda, int64_t rows, int64_t cols,
                                 double* out, int64_t ldo);
cudaError_t check_init(cudaStream_t st, const double* X, int64_t rows, int k, double* d_maxdev, Scratch& ws);
cudaError_t find_nonfinite(cudaStream_t st, const double* v, int64_t n, int* d_flag);
// C(i,j) = beta C(i,j) + alpha A(i,j) over rows x cols (strided views)
cudaError_t mat_axpby(cudaStream_t st, int64_t rows, int64_t cols, double alpha, CMat A, double beta, Mat C);

// Device-time account of one kernel class (bench.py roofline, tsvd_stats.top_*).
struct KProf {
  float ms = 0.f;
  int launches = 0;
  double flops = 0.0, bytes = 0.0;
};

// ---- jacobi.cu
// One-sided block Jacobi SVD of A (m x n col-major, lda), top kk triplets.
// theta(n) all values descending; F (m x kk, ldf) and G (n x kk, ldg) col-major.
cudaError_t jacobi_svd(cudaStream_t st, const double* A, int64_t lda, int64_t m, int64_t n, int kk,
                       double* theta, double* F, int64_t ldf, double* G, int64_t ldg, int* sweeps,
                       bool* converged, Scratch& ws, KProf* prof = nullptr);

}  // namespace tsvd
