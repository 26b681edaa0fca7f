// Vector / small dense kernels used by the non-filter rows of Alg. 1 (Lanczos, CholQR2,
// Rayleigh-Ritz, residuals, locking).  All column-major complex double unless stated; all
// reductions use a fixed order (no atomics) so results are bitwise reproducible and identical on
// every rank that computes them redundantly (ledger #20).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace chase {

// Z[:, a] = 0 for a block; generic complex 2-D copy dst(rows x cols) <- src
void zcopy2d(void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows, int cols, cudaStream_t st);
void zzero2d(void* dst, int64_t ldd, int64_t rows, int cols, cudaStream_t st);

// out[a] = sum_k conj(X[k, a]) * Y[k, a], a < ncols  (complex; written as 2 doubles per column)
// and out_norm2[a] = sum_k |X[k,a] - theta[a] Y[k,a]|^2 variants.  `part` is device scratch of
// at least colreduce_scratch(ncols) doubles.
size_t colreduce_scratch(int ncols);
void col_dots(const void* X, int64_t ldx, const void* Y, int64_t ldy, int64_t rows, int ncols,
              double* out /* 2*ncols */, double* part, cudaStream_t st);
// out[a] = sum_k |HV[k,a] - theta[a] V[k,a]|^2   (theta on device, ncols doubles)
void resid_norms2(const void* HV, int64_t ldh, const void* V, int64_t ldv, const double* theta,
                  int64_t rows, int ncols, double* out, double* part, cudaStream_t st);

// G <- (G + G^H)/2 in place (n x n, ld)
void hermitize(void* G, int64_t ld, int n, cudaStream_t st);
// dst[:, a] = src[:, perm[a]] for a < ncols (perm on device)
void permute_cols(void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows,
                  const int* perm, int ncols, cudaStream_t st);
// G[i,i] += s for i < n
void add_diag(void* G, int64_t ld, int n, double s, cudaStream_t st);
// Lanczos helpers (full-length vectors, L runs side by side; see lanczos.cu)
void scale_cols_inv(void* X, int64_t ld, int64_t rows, int ncols, const double* nrm2, cudaStream_t st);

}  // namespace chase
