// Cholesky (G = R^H R, R upper) and upper-triangular inverse on the device, blocked with
// NB = 64: diagonal blocks in one CTA (shared memory), panels by substitution, trailing updates
// through the DMMA GEMM (zgemm); the inverse recursively (half-size off-diagonal blocks).  Used by CholQR2 (SURVEY §8
// row a7: "Gram -> Cholesky -> V <- V R^-1").
#include <algorithm>
#include "common.cuh"
#include "dense.h"
#include "linalg.h"
#include "zgemm.h"

namespace chase {

namespace {
constexpr int NB = 64;
constexpr int LDS = NB + 1;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {   // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

// Unblocked upper Cholesky of the nb x nb diagonal block at G (ld), in place; lower part zeroed.
__global__ void k_chol_diag(double2* G, int64_t ld, int nb, int* info) {
  extern __shared__ double2 A[];   // NB x LDS
  const int t = threadIdx.x, nt = blockDim.x;
  for (int idx = t; idx < nb * nb; idx += nt) {
    const int i = idx % nb, j = idx / nb;
    A[i * LDS + j] = (i <= j) ? G[i + (int64_t)j * ld] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int k = 0; k < nb; ++k) {
    if (t == 0) {
      const double d = A[k * LDS + k].x;
      double r;
      if (!(d > 0.0) || !isfinite(d)) {
        atomicExch(info, 1);
        r = 1.0;
      } else {
        r = sqrt(d);
      }
      A[k * LDS + k] = make_double2(r, 0.0);
    }
    __syncthreads();
    const double rkk = A[k * LDS + k].x;
    for (int j = k + 1 + t; j < nb; j += nt) {
      double2 v = A[k * LDS + j];
      A[k * LDS + j] = make_double2(v.x / rkk, v.y / rkk);
    }
    __syncthreads();
    const int m = nb - k - 1;
    for (int idx = t; idx < m * m; idx += nt) {
      const int i = k + 1 + idx % m, j = k + 1 + idx / m;
      if (i <= j) {
        const double2 u = cmulc(A[k * LDS + i], A[k * LDS + j]);
        A[i * LDS + j].x -= u.x;
        A[i * LDS + j].y -= u.y;
      }
    }
    __syncthreads();
  }
  for (int idx = t; idx < nb * nb; idx += nt) {
    const int i = idx % nb, j = idx / nb;
    G[i + (int64_t)j * ld] = A[i * LDS + j];
  }
}

// Panel: X[0:nb, j] <- R_kk^{-H} X[0:nb, j] for the columns right of the diagonal block.
__global__ void k_chol_panel(double2* G, int64_t ld, int nb, int ncols) {
  extern __shared__ double2 R[];   // NB x LDS
  const double2* Rg = G;
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int i = idx % nb, j = idx / nb;
    R[i * LDS + j] = Rg[i + (int64_t)j * ld];
  }
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  double2* x = G + (int64_t)(nb + j) * ld;   // column (block col offset nb + j), rows 0..nb
  double2 xs[NB];
#pragma unroll 1
  for (int i = 0; i < nb; ++i) {
    double2 s = x[i];
    for (int l = 0; l < i; ++l) {
      const double2 u = cmulc(R[l * LDS + i], xs[l]);
      s.x -= u.x;
      s.y -= u.y;
    }
    xs[i] = cdiv(s, R[i * LDS + i]);
  }
  for (int i = 0; i < nb; ++i) x[i] = xs[i];
}

// Inverse of each upper-triangular diagonal block of R (n x n) into X (same layout); the strictly
// lower part of every diagonal block of X is zeroed.
__global__ void k_trinv_diag(const double2* R, int64_t ldr, double2* X, int64_t ldx, int n) {
  extern __shared__ double2 Rs[];   // 2 x NB x LDS
  double2* Xs = Rs + NB * LDS;
  const int kb = blockIdx.x * NB;
  const int nb = min(NB, n - kb);
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int i = idx % nb, j = idx / nb;
    Rs[i * LDS + j] = R[(kb + i) + (int64_t)(kb + j) * ldr];
    Xs[i * LDS + j] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int j = threadIdx.x;
  if (j < nb) {
    Xs[j * LDS + j] = cdiv(make_double2(1.0, 0.0), Rs[j * LDS + j]);
    for (int i = j - 1; i >= 0; --i) {
      double2 s = make_double2(0.0, 0.0);
      for (int l = i + 1; l <= j; ++l) {
        const double2 u = cmul(Rs[i * LDS + l], Xs[l * LDS + j]);
        s.x += u.x;
        s.y += u.y;
      }
      const double2 v = cdiv(s, Rs[i * LDS + i]);
      Xs[i * LDS + j] = make_double2(-v.x, -v.y);
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int i = idx % nb, jj = idx / nb;
    X[(kb + i) + (int64_t)(kb + jj) * ldx] = Xs[i * LDS + jj];
  }
}
}  // namespace

bool cholesky_upper(void* Gv, int64_t ld, int n, int* d_info, cudaStream_t st) {
  double2* G = reinterpret_cast<double2*>(Gv);
  CHASE_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int), st));
  static unsigned long long attr = 0;
  const size_t smem = sizeof(double2) * NB * LDS;
  if (first_on_device(attr)) {
    CHASE_CUDA(cudaFuncSetAttribute(k_chol_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CHASE_CUDA(cudaFuncSetAttribute(k_chol_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  for (int kb = 0; kb < n; kb += NB) {
    const int nb = std::min(NB, n - kb);
    double2* Gkk = G + kb + (int64_t)kb * ld;
    k_chol_diag<<<1, 256, smem, st>>>(Gkk, ld, nb, d_info);
    CHASE_CHECK_LAUNCH();
    const int m = n - kb - nb;
    if (m <= 0) break;
    k_chol_panel<<<ceil_div(m, 64), 64, smem, st>>>(Gkk, ld, nb, m);
    CHASE_CHECK_LAUNCH();
    // trailing: G22 -= R12^H R12  (R12 = G[kb:kb+nb, kb+nb:] stored nb x m)
    ZgemmDesc d;
    d.M = m; d.N = m; d.K = nb; d.conjA = true;
    d.A = G + kb + (int64_t)(kb + nb) * ld; d.lda = ld;
    d.B = d.A; d.ldb = ld;
    d.C = G + (kb + nb) + (int64_t)(kb + nb) * ld; d.ldc = ld;
    d.alpha = -1.0; d.beta = 1.0;
    d.upper_only = true;          // only the upper triangle of the trailing matrix is ever read
    zgemm(d, st);
  }
  int info = 0;
  CHASE_CUDA(cudaMemcpyAsync(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost, st));
  CHASE_CUDA(cudaStreamSynchronize(st));
  return info == 0;
}

namespace {
// X = R^-1 on the leading n x n block, recursively (the diagonal NB-blocks of X are already
// inverted): X11 = R11^-1, X22 = R22^-1, X12 = -(X11 R12) X22.  Every level is two GEMMs over
// half-size blocks, so the products stay large (the column-by-column blocked form runs 2(n/NB)
// GEMMs of at most n x NB outputs -- 1..23 CTAs each at n = 3000).  T: >= n1 n2 scratch.
void trinv_rec(const double2* R, int64_t ldr, double2* X, int64_t ldx, double2* T, int n, cudaStream_t st) {
  if (n <= NB) return;
  const int n1 = ceil_div(ceil_div(n, NB), 2) * NB;       // a multiple of NB
  const int n2 = n - n1;
  trinv_rec(R, ldr, X, ldx, T, n1, st);
  trinv_rec(R + n1 + (int64_t)n1 * ldr, ldr, X + n1 + (int64_t)n1 * ldx, ldx, T, n2, st);
  ZgemmDesc d;                                             // T = X11 R12   (n1 x n2)
  d.M = n1; d.N = n2; d.K = n1;
  d.A = X; d.lda = ldx;
  d.B = R + (int64_t)n1 * ldr; d.ldb = ldr;
  d.C = T; d.ldc = n1;
  zgemm(d, st);
  ZgemmDesc e;                                             // X12 = -T X22
  e.M = n1; e.N = n2; e.K = n2;
  e.A = T; e.lda = n1;
  e.B = X + n1 + (int64_t)n1 * ldx; e.ldb = ldx;
  e.C = X + (int64_t)n1 * ldx; e.ldc = ldx;
  e.alpha = -1.0; e.beta = 0.0;
  zgemm(e, st);
}
}  // namespace

void trinv_upper(const void* Rv, int64_t ldr, void* Xv, int64_t ldx, void* T, int n, cudaStream_t st) {
  const double2* R = reinterpret_cast<const double2*>(Rv);
  double2* X = reinterpret_cast<double2*>(Xv);
  // the strictly lower block triangle of X must be 0: the GEMM steps read full squares of X
  zzero2d(X, ldx, n, n, st);
  const int nblk = ceil_div(n, NB);
  const size_t smem = 2 * sizeof(double2) * NB * LDS;
  static unsigned long long attr = 0;
  if (first_on_device(attr)) {
    CHASE_CUDA(cudaFuncSetAttribute(k_trinv_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  k_trinv_diag<<<nblk, NB, smem, st>>>(R, ldr, X, ldx, n);
  CHASE_CHECK_LAUNCH();
  trinv_rec(R, ldr, X, ldx, reinterpret_cast<double2*>(T), n, st);
}

}  // namespace chase
