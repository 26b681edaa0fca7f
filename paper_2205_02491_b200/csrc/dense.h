// Vector / small dense kernels used by the non-filter rows of Alg. 1 (Lanczos, CholQR2,
// Rayleigh-Ritz, residuals, locking).  Column-major; T = double2 (complex double) or double (real
// symmetric variant).  All reductions use a fixed order (no atomics) so results are bitwise
// reproducible and identical on every rank that computes them redundantly (ledger #20).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace chase {

template <class T>
void copy2d(void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows, int cols, cudaStream_t st);
template <class T>
void zero2d(void* dst, int64_t ldd, int64_t rows, int cols, cudaStream_t st);

// out[2a], out[2a+1] = re, im of sum_k conj(X[k, a]) * Y[k, a]; `part` is device scratch of at least
// colreduce_scratch(ncols) doubles.
size_t colreduce_scratch(int ncols);
template <class T>
void col_dots(const void* X, int64_t ldx, const void* Y, int64_t ldy, int64_t rows, int ncols, double* out,
              double* part, cudaStream_t st);
// out[a] = sum_k |HV[k,a] - theta[a] V[k,a]|^2   (theta on device, ncols doubles)
template <class T>
void resid_norms2(const void* HV, int64_t ldh, const void* V, int64_t ldv, const double* theta, int64_t rows,
                  int ncols, double* out, double* part, cudaStream_t st);
// G <- (G + G^H)/2 in place (n x n, ld)
template <class T>
void hermitize(void* G, int64_t ld, int n, cudaStream_t st);
// dst[:, a] = src[:, perm[a]] for a < ncols (perm on device)
template <class T>
void permute_cols(void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows, const int* perm, int ncols,
                  cudaStream_t st);
// G[i,i] += s for i < n
template <class T>
void add_diag(void* G, int64_t ld, int n, double s, cudaStream_t st);
// real <-> complex copies of an n x n matrix (the real path reuses the complex small-matrix solvers)
void real_to_complex(double2* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols, cudaStream_t st);
void complex_to_real(double* dst, int64_t ldd, const double2* src, int64_t lds, int rows, int cols, cudaStream_t st);

// legacy complex names
inline void zcopy2d(void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows, int cols, cudaStream_t st) {
  copy2d<double2>(dst, ldd, src, lds, rows, cols, st);
}
inline void zzero2d(void* dst, int64_t ldd, int64_t rows, int cols, cudaStream_t st) {
  zero2d<double2>(dst, ldd, rows, cols, st);
}

}  // namespace chase
