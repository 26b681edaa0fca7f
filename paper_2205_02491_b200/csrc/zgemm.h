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
};

// C = alpha*op(A)*B - alpha*gamma*S[shift rows] + beta*C   (all complex double, column-major)
void zgemm(const ZgemmDesc& d, cudaStream_t st);

}  // namespace chase
