// Small dense linear algebra on the device for the non-filter rows of Alg. 1.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace chase {

// Upper Cholesky in place: G (n x n, ld; upper triangle read) = R^H R, R written to the upper
// triangle.  Returns false if a pivot was not positive (matrix not numerically HPD).
// Synchronizes `st` (reads the device info flag).
bool cholesky_upper(void* G, int64_t ld, int n, int* d_info, cudaStream_t st);

// X = R^{-1} for upper-triangular R (n x n); X (ldx) gets zeros below the diagonal.
// T: device scratch of >= n * n / 4 complex (the recursion's largest off-diagonal block).
void trinv_upper(const void* R, int64_t ldr, void* X, int64_t ldx, void* T, int n, cudaStream_t st);

// Hermitian eigendecomposition G = Z diag(theta) Z^H by block-cyclic two-sided Jacobi
// (64 x 64 subproblems solved in one CTA each, updates as 64 x 64 complex tile products).
// G: n x n (ld) device, destroyed.  theta: device n doubles ascending.  Z: device n x n (ldz).
// Returns the number of sweeps; throws NumericError if not converged.
// `work`: the caller's workspace slot (a handle owns one; allocated / grown on first use, freed by
// heev_work_release), so concurrent handles on one device never share buffers.
struct JacobiWork;
int heev_jacobi(void* G, int64_t ld, int n, double* theta, void* Z, int64_t ldz, cudaStream_t st, JacobiWork** work);
void heev_work_release(JacobiWork* work);

}  // namespace chase
