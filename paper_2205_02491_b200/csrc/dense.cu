// Vector / small dense kernels (see dense.h).  HBM-bound: coalesced accesses, block tree
// reductions in shared memory, fixed-order two-pass column reductions (deterministic).
#include <algorithm>
#include "common.cuh"
#include "dense.h"
#include "scalar.cuh"

namespace chase {

namespace {
constexpr int RT = 256;            // threads per reduction block
constexpr int MAX_CHUNKS = 64;     // row chunks per column in pass 1

template <class T>
__global__ void k_copy2d(T* dst, int64_t ldd, const T* src, int64_t lds, int64_t rows, int cols) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows, c = i / rows;
    dst[r + c * ldd] = src[r + c * lds];
  }
}

template <class T>
__global__ void k_zero2d(T* dst, int64_t ldd, int64_t rows, int cols) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows, c = i / rows;
    dst[r + c * ldd] = SC<T>::zero();
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
template <class T>
__global__ void k_col_dots_p1(const T* X, int64_t ldx, const T* Y, int64_t ldy, int64_t rows, int chunks,
                              double* part) {
  __shared__ double sh[2 * RT];
  const int col = blockIdx.x, chunk = blockIdx.y;
  const int64_t len = (rows + chunks - 1) / chunks;
  const int64_t r0 = chunk * len, r1 = min(rows, r0 + len);
  double v[2] = {0.0, 0.0};
  const T* x = X + col * ldx;
  const T* y = Y + col * ldy;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += RT) {
    const T d = SC<T>::mulc(x[r], y[r]);
    v[0] += SC<T>::re(d);
    v[1] += SC<T>::im(d);
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

template <class T>
__global__ void k_resid_p1(const T* HV, int64_t ldh, const T* V, int64_t ldv, const double* theta, int64_t rows,
                           int chunks, double* part) {
  __shared__ double sh[RT];
  const int col = blockIdx.x, chunk = blockIdx.y;
  const int64_t len = (rows + chunks - 1) / chunks;
  const int64_t r0 = chunk * len, r1 = min(rows, r0 + len);
  const double th = theta[col];
  double v[1] = {0.0};
  const T* h = HV + col * ldh;
  const T* x = V + col * ldv;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += RT) v[0] += SC<T>::abs2(SC<T>::sub(h[r], SC<T>::scale(x[r], th)));
  block_sum<1>(v, sh);
  if (threadIdx.x == 0) part[(int64_t)col * chunks + chunk] = v[0];
}

template <class T>
__global__ void k_hermitize(T* G, int64_t ld, int n) {
  const int64_t total = (int64_t)n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    if (i > j) continue;
    if (i == j) {
      G[i + (int64_t)i * ld] = SC<T>::make(SC<T>::re(G[i + (int64_t)i * ld]), 0.0);
      continue;
    }
    const T s = SC<T>::scale(SC<T>::add(G[i + (int64_t)j * ld], SC<T>::conj(G[j + (int64_t)i * ld])), 0.5);
    G[i + (int64_t)j * ld] = s;
    G[j + (int64_t)i * ld] = SC<T>::conj(s);
  }
}

template <class T>
__global__ void k_permute_cols(T* dst, int64_t ldd, const T* src, int64_t lds, int64_t rows, const int* perm,
                               int ncols) {
  const int64_t total = rows * ncols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows;
    const int c = (int)(i / rows);
    dst[r + c * ldd] = src[r + (int64_t)perm[c] * lds];
  }
}

template <class T>
__global__ void k_add_diag(T* G, int64_t ld, int n, double s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) G[i + (int64_t)i * ld] = SC<T>::add(G[i + (int64_t)i * ld], SC<T>::make(s, 0.0));
}

__global__ void k_r2c(double2* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows, c = i / rows;
    dst[r + c * ldd] = make_double2(src[r + c * lds], 0.0);
  }
}

__global__ void k_c2r(double* dst, int64_t ldd, const double2* src, int64_t lds, int rows, int cols) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows, c = i / rows;
    dst[r + c * ldd] = src[r + c * lds].x;
  }
}
}  // namespace

template <class T>
void copy2d(void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows, int cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  if (ldd == rows && lds == rows) {
    CHASE_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * (size_t)rows * cols, cudaMemcpyDeviceToDevice, st));
    return;
  }
  k_copy2d<T><<<grid_for(rows * cols), 256, 0, st>>>((T*)dst, ldd, (const T*)src, lds, rows, cols);
  CHASE_CHECK_LAUNCH();
}

template <class T>
void zero2d(void* dst, int64_t ldd, int64_t rows, int cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  if (ldd == rows) {
    CHASE_CUDA(cudaMemsetAsync(dst, 0, sizeof(T) * (size_t)rows * cols, st));
    return;
  }
  k_zero2d<T><<<grid_for(rows * cols), 256, 0, st>>>((T*)dst, ldd, rows, cols);
  CHASE_CHECK_LAUNCH();
}

size_t colreduce_scratch(int ncols) { return (size_t)ncols * MAX_CHUNKS * 2; }

template <class T>
void col_dots(const void* X, int64_t ldx, const void* Y, int64_t ldy, int64_t rows, int ncols, double* out,
              double* part, cudaStream_t st) {
  if (ncols <= 0) return;
  if (rows <= 0) {
    CHASE_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * 2 * ncols, st));
    return;
  }
  const int chunks = chunks_for(rows);
  k_col_dots_p1<T><<<dim3(ncols, chunks), RT, 0, st>>>((const T*)X, ldx, (const T*)Y, ldy, rows, chunks, part);
  CHASE_CHECK_LAUNCH();
  k_col_reduce_p2<<<(ncols + 127) / 128, 128, 0, st>>>(part, chunks, 2, ncols, out);
  CHASE_CHECK_LAUNCH();
}

template <class T>
void resid_norms2(const void* HV, int64_t ldh, const void* V, int64_t ldv, const double* theta, int64_t rows,
                  int ncols, double* out, double* part, cudaStream_t st) {
  if (ncols <= 0) return;
  if (rows <= 0) {
    CHASE_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * ncols, st));
    return;
  }
  const int chunks = chunks_for(rows);
  k_resid_p1<T><<<dim3(ncols, chunks), RT, 0, st>>>((const T*)HV, ldh, (const T*)V, ldv, theta, rows, chunks, part);
  CHASE_CHECK_LAUNCH();
  k_col_reduce_p2<<<(ncols + 127) / 128, 128, 0, st>>>(part, chunks, 1, ncols, out);
  CHASE_CHECK_LAUNCH();
}

template <class T>
void hermitize(void* G, int64_t ld, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_hermitize<T><<<grid_for((int64_t)n * n), 256, 0, st>>>((T*)G, ld, n);
  CHASE_CHECK_LAUNCH();
}

template <class T>
void permute_cols(void* dst, int64_t ldd, const void* src, int64_t lds, int64_t rows, const int* perm, int ncols,
                  cudaStream_t st) {
  if (rows <= 0 || ncols <= 0) return;
  k_permute_cols<T><<<grid_for(rows * ncols), 256, 0, st>>>((T*)dst, ldd, (const T*)src, lds, rows, perm, ncols);
  CHASE_CHECK_LAUNCH();
}

template <class T>
void add_diag(void* G, int64_t ld, int n, double s, cudaStream_t st) {
  if (n <= 0) return;
  k_add_diag<T><<<(n + 255) / 256, 256, 0, st>>>((T*)G, ld, n, s);
  CHASE_CHECK_LAUNCH();
}

void real_to_complex(double2* dst, int64_t ldd, const double* src, int64_t lds, int rows, int cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  k_r2c<<<grid_for((int64_t)rows * cols), 256, 0, st>>>(dst, ldd, src, lds, rows, cols);
  CHASE_CHECK_LAUNCH();
}

void complex_to_real(double* dst, int64_t ldd, const double2* src, int64_t lds, int rows, int cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  k_c2r<<<grid_for((int64_t)rows * cols), 256, 0, st>>>(dst, ldd, src, lds, rows, cols);
  CHASE_CHECK_LAUNCH();
}

#define CHASE_INST(T)                                                                                       \
  template void copy2d<T>(void*, int64_t, const void*, int64_t, int64_t, int, cudaStream_t);                \
  template void zero2d<T>(void*, int64_t, int64_t, int, cudaStream_t);                                      \
  template void col_dots<T>(const void*, int64_t, const void*, int64_t, int64_t, int, double*, double*,     \
                            cudaStream_t);                                                                  \
  template void resid_norms2<T>(const void*, int64_t, const void*, int64_t, const double*, int64_t, int,    \
                                double*, double*, cudaStream_t);                                            \
  template void hermitize<T>(void*, int64_t, int, cudaStream_t);                                            \
  template void permute_cols<T>(void*, int64_t, const void*, int64_t, int64_t, const int*, int, cudaStream_t); \
  template void add_diag<T>(void*, int64_t, int, double, cudaStream_t);
CHASE_INST(double2)
CHASE_INST(double)
#undef CHASE_INST

}  // namespace chase
