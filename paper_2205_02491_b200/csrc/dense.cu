// Vector / small dense kernels (see dense.h).  HBM-bound: coalesced 16-byte accesses, block
// tree reductions in shared memory, fixed-order two-pass column reductions (deterministic).
#include <algorithm>
#include "common.cuh"
#include "dense.h"

namespace chase {

namespace {
constexpr int RT = 256;            // threads per reduction block
constexpr int MAX_CHUNKS = 64;     // row chunks per column in pass 1

__global__ void k_zcopy2d(double2* dst, int64_t ldd, const double2* src, int64_t lds, int64_t rows, int cols) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows, c = i / rows;
    dst[r + c * ldd] = src[r + c * lds];
  }
}

__global__ void k_zzero2d(double2* dst, int64_t ldd, int64_t rows, int cols) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows, c = i / rows;
    dst[r + c * ldd] = make_double2(0.0, 0.0);
  }
}

inline int grid_for(int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 32));
}

inline int chunks_for(int64_t rows) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(MAX_CHUNKS, (rows + 4095) / 4096));
}

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sh) {
  // sh: RT * NV doubles
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < NV; ++k) sh[k * RT + t] = v[k];
  __syncthreads();
  for (int s = RT / 2; s > 0; s >>= 1) {
    if (t < s) {
#pragma unroll
      for (int k = 0; k < NV; ++k) sh[k * RT + t] += sh[k * RT + t + s];
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = sh[k * RT];
}

// pass 1: part[(col * chunks + chunk) * 2 + {0,1}] = partial conj(x).y over the chunk
__global__ void k_col_dots_p1(const double2* X, int64_t ldx, const double2* Y, int64_t ldy, int64_t rows,
                              int chunks, double* part) {
  __shared__ double sh[2 * RT];
  const int col = blockIdx.x, chunk = blockIdx.y;
  const int64_t len = (rows + chunks - 1) / chunks;
  const int64_t r0 = chunk * len, r1 = min(rows, r0 + len);
  double v[2] = {0.0, 0.0};
  const double2* x = X + col * ldx;
  const double2* y = Y + col * ldy;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += RT) {
    const double2 a = x[r], b = y[r];
    v[0] += a.x * b.x + a.y * b.y;
    v[1] += a.x * b.y - a.y * b.x;
  }
  block_sum<2>(v, sh);
  if (threadIdx.x == 0) {
    part[((int64_t)col * chunks + chunk) * 2] = v[0];
    part[((int64_t)col * chunks + chunk) * 2 + 1] = v[1];
  }
}

__global__ void k_col_reduce_p2(const double* part, int chunks, int width, int ncols, double* out) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ncols) return;
  for (int w = 0; w < width; ++w) {
    double s = 0.0;
    for (int c = 0; c < chunks; ++c) s += part[((int64_t)col * chunks + c) * width + w];
    out[(int64_t)col * width + w] = s;
  }
}

__global__ void k_resid_p1(const double2* HV, int64_t ldh, const double2* V, int64_t ldv, const double* theta,
                           int64_t rows, int chunks, double* part) {
  __shared__ double sh[RT];
  const int col = blockIdx.x, chunk = blockIdx.y;
  const int64_t len = (rows + chunks - 1) / chunks;
  const int64_t r0 = chunk * len, r1 = min(rows, r0 + len);
  const double th = theta[col];
  double v[1] = {0.0};
  const double2* h = HV + col * ldh;
  const double2* x = V + col * ldv;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += RT) {
    const double2 a = h[r], b = x[r];
    const double dr = a.x - th * b.x, di = a.y - th * b.y;
    v[0] += dr * dr + di * di;
  }
  block_sum<1>(v, sh);
  if (threadIdx.x == 0) part[(int64_t)col * chunks + chunk] = v[0];
}

__global__ void k_hermitize(double2* G, int64_t ld, int n) {
  const int64_t total = (int64_t)n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    if (i > j) continue;
    if (i == j) {
      G[i + (int64_t)i * ld].y = 0.0;
      continue;
    }
    const double2 a = G[i + (int64_t)j * ld], b = G[j + (int64_t)i * ld];
    const double2 s = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
    G[i + (int64_t)j * ld] = s;
    G[j + (int64_t)i * ld] = make_double2(s.x, -s.y);
  }
}

__global__ void k_permute_cols(double2* dst, int64_t ldd, const double2* src, int64_t lds, int64_t rows,
                               const int* perm, int ncols) {
  const int64_t total = rows * ncols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows;
    const int c = (int)(i / rows);
    dst[r + c * ldd] = src[r + (int64_t)perm[c] * lds];
  }
}

__global__ void k_scale_cols_inv(double2* X, int64_t ld, int64_t rows, int ncols, const double* nrm2) {
  const int64_t total = rows * ncols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows;
    const int c = (int)(i / rows);
    const double n2 = nrm2[c];
    const double s = n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0;
    double2 v = X[r + c * ld];
    X[r + c * ld] = make_double2(v.x * s, v.y * s);
  }
}
__global__ void k_add_diag(double2* G, int64_t ld, int n, double s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) G[i + (int64_t)i * ld].x += s;
}
}  // namespace

void add_diag(void* G, int64_t ld, int n, double s, cudaStream_t st) {
  if (n <= 0) return;
  k_add_diag<<<(n + 255) / 256, 256, 0, st>>>((double2*)G, ld, n, s);
  CHASE_CHECK_LAUNCH();
}

void zcopy2d(void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows, int cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  if (ldd == rows && lds == rows) {
    CHASE_CUDA(cudaMemcpyAsync(dst, src, 16 * (size_t)rows * cols, cudaMemcpyDeviceToDevice, st));
    return;
  }
  k_zcopy2d<<<grid_for(rows * cols), 256, 0, st>>>((double2*)dst, ldd, (const double2*)src, lds, rows, cols);
  CHASE_CHECK_LAUNCH();
}

void zzero2d(void* dst, int64_t ldd, int64_t rows, int cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  if (ldd == rows) {
    CHASE_CUDA(cudaMemsetAsync(dst, 0, 16 * (size_t)rows * cols, st));
    return;
  }
  k_zzero2d<<<grid_for(rows * cols), 256, 0, st>>>((double2*)dst, ldd, rows, cols);
  CHASE_CHECK_LAUNCH();
}

size_t colreduce_scratch(int ncols) { return (size_t)ncols * MAX_CHUNKS * 2; }

void col_dots(const void* X, int64_t ldx, const void* Y, int64_t ldy, int64_t rows, int ncols, double* out,
              double* part, cudaStream_t st) {
  if (ncols <= 0) return;
  if (rows <= 0) {
    CHASE_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * 2 * ncols, st));
    return;
  }
  const int chunks = chunks_for(rows);
  k_col_dots_p1<<<dim3(ncols, chunks), RT, 0, st>>>((const double2*)X, ldx, (const double2*)Y, ldy, rows, chunks, part);
  CHASE_CHECK_LAUNCH();
  k_col_reduce_p2<<<(ncols + 127) / 128, 128, 0, st>>>(part, chunks, 2, ncols, out);
  CHASE_CHECK_LAUNCH();
}

void resid_norms2(const void* HV, int64_t ldh, const void* V, int64_t ldv, const double* theta, int64_t rows,
                  int ncols, double* out, double* part, cudaStream_t st) {
  if (ncols <= 0) return;
  if (rows <= 0) {
    CHASE_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * ncols, st));
    return;
  }
  const int chunks = chunks_for(rows);
  k_resid_p1<<<dim3(ncols, chunks), RT, 0, st>>>((const double2*)HV, ldh, (const double2*)V, ldv, theta, rows,
                                                 chunks, part);
  CHASE_CHECK_LAUNCH();
  k_col_reduce_p2<<<(ncols + 127) / 128, 128, 0, st>>>(part, chunks, 1, ncols, out);
  CHASE_CHECK_LAUNCH();
}

void hermitize(void* G, int64_t ld, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_hermitize<<<grid_for((int64_t)n * n), 256, 0, st>>>((double2*)G, ld, n);
  CHASE_CHECK_LAUNCH();
}

void permute_cols(void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows, const int* perm, int ncols,
                  cudaStream_t st) {
  if (rows <= 0 || ncols <= 0) return;
  k_permute_cols<<<grid_for(rows * ncols), 256, 0, st>>>((double2*)dst, ldd, (const double2*)src, lds, rows, perm,
                                                         ncols);
  CHASE_CHECK_LAUNCH();
}

void scale_cols_inv(void* X, int64_t ld, int64_t rows, int ncols, const double* nrm2, cudaStream_t st) {
  if (rows <= 0 || ncols <= 0) return;
  k_scale_cols_inv<<<grid_for(rows * ncols), 256, 0, st>>>((double2*)X, ld, rows, ncols, nrm2);
  CHASE_CHECK_LAUNCH();
}

}  // namespace chase
