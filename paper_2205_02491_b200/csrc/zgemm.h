// Host interface of the fused complex-double GEMM (see zgemm.cuh for the kernel).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace chase {

struct ZgemmDesc {
  int M = 0, N = 0, K = 0;
  bool conjA = false;            // op(A) = A^H with A stored K x M
  const void* A = nullptr; int64_t lda = 0;
  const void* B = nullptr; int64_t ldb = 0;
  void* C = nullptr; int64_t ldc = 0;
  double alpha = 1.0, beta = 0.0, gamma = 0.0;
  const void* S = nullptr; int64_t lds = 0;   // shift source (may be null)
  int shift_lo = 0, shift_hi = 0; int64_t shift_off = 0;
  bool use3m = false;            // 3M (Gauss) complex product: 3 real DMMAs per complex MAC
  bool upper_only = false;       // only tiles on/above the diagonal are computed (Hermitian C)
  bool b_upper = false;          // B upper triangular (zeros below the diagonal are skipped)
};

// C = alpha*op(A)*B - alpha*gamma*S[shift rows] + beta*C   (all complex double, column-major)
void zgemm(const ZgemmDesc& d, cudaStream_t st);
// The same contract for real double (op(A) = A^T when conjA; use3m ignored).  Real-symmetric f2.
void dgemm(const ZgemmDesc& d, cudaStream_t st);

}  // namespace chase

namespace chase {
// Skinny product C[M x L] = alpha * A[M x K] * B[K x L] for L <= 8 (HBM-bound: streams A once;
// used by the Lanczos step).  `work` must hold skinny_work_bytes(M, K, L).
size_t skinny_work_bytes(int M, int K, int L);
// a_c64: A is complex single (c64 shard), read and accumulated in FP64
void zgemm_skinny(int M, int L, int K, double alpha, const void* A, int64_t lda, const void* B,
                  int64_t ldb, void* C, int64_t ldc, void* work, cudaStream_t st, bool a_c64 = false);
// real variant (f2); `work` as for the complex one (it needs half of it)
void dgemm_skinny(int M, int L, int K, double alpha, const void* A, int64_t lda, const void* B,
                  int64_t ldb, void* C, int64_t ldc, void* work, cudaStream_t st);
}  // namespace chase
