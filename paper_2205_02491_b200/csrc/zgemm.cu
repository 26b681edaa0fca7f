#include <cstdlib>
// Host launcher for the TMA + DMMA complex GEMM (zgemm.cuh) and the tensor-map encoder.
#include "zgemm.h"
#include "zgemm.cuh"
#include "zgemm3m.cuh"
#include <algorithm>

namespace chase {

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {   // thread-safe one-time init
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CHASE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

void make_zmatrix_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                       int box_cols) {
  cuuint64_t dims[2] = {(cuuint64_t)(2 * rows), (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 16)};
  cuuint32_t box[2] = {16u, (cuuint32_t)box_cols};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = get_encode()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") rows=" +
                    std::to_string(rows) + " cols=" + std::to_string(cols) + " ld=" + std::to_string(ld));
}

bool make_zmatrix_tmap_chunked(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                               int box_cols, int box_chunks) {
  if (rows % 8 != 0) return false;
  cuuint64_t dims[3] = {16u, (cuuint64_t)cols, (cuuint64_t)(rows / 8)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 16), 128u};
  cuuint32_t box[3] = {16u, (cuuint32_t)box_cols, (cuuint32_t)box_chunks};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = get_encode()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BM, int BN, bool CONJ>
static void launch(const ZgemmDesc& d, cudaStream_t st) {
  using C_ = zg::Cfg<BM, BN>;
  CUtensorMap ta, tb;
  bool chunked = false;
  if (!CONJ) {
    chunked = make_zmatrix_tmap_chunked(&ta, d.A, d.M, d.K, d.lda, zg::BK, BM / 8);
    if (!chunked) make_zmatrix_tmap(&ta, d.A, d.M, d.K, d.lda, zg::BK);      // A: M x K
  } else {
    make_zmatrix_tmap(&ta, d.A, d.K, d.M, d.lda, BM);          // A: K x M (op = A^H)
  }
  make_zmatrix_tmap(&tb, d.B, d.K, d.N, d.ldb, BN);
  static unsigned long long attr_set = 0;
  if (first_on_device(attr_set)) {
    CHASE_CUDA(cudaFuncSetAttribute(zgemm_dmma_kernel<BM, BN, CONJ>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C_::SMEM));
  }
  ZgemmParams p;
  p.M = d.M; p.N = d.N; p.K = d.K;
  p.alpha = d.alpha; p.beta = d.beta; p.gamma = d.gamma;
  p.S = reinterpret_cast<const double2*>(d.S); p.lds = d.lds;
  p.shift_lo = d.shift_lo; p.shift_hi = d.shift_hi; p.shift_off = d.shift_off;
  p.C = reinterpret_cast<double2*>(d.C); p.ldc = d.ldc;
  p.a_chunked = chunked ? 1 : 0;
  p.upper_only = d.upper_only ? 1 : 0;
  p.b_upper = d.b_upper ? 1 : 0;
  const int grid = ceil_div(d.M, BM) * ceil_div(d.N, BN);
  zgemm_dmma_kernel<BM, BN, CONJ><<<grid, C_::THREADS, C_::SMEM, st>>>(ta, tb, p);
  CHASE_CHECK_LAUNCH();
}

template <class CFG, bool CONJ>
static void launch3m(const ZgemmDesc& d, cudaStream_t st) {
  CUtensorMap ta, tb;
  bool chunked = false;
  if (!CONJ) {
    chunked = make_zmatrix_tmap_chunked(&ta, d.A, d.M, d.K, d.lda, CFG::BK, CFG::BM / 8);
    if (!chunked) make_zmatrix_tmap(&ta, d.A, d.M, d.K, d.lda, CFG::BK);
  } else {
    make_zmatrix_tmap(&ta, d.A, d.K, d.M, d.lda, CFG::BM);
  }
  make_zmatrix_tmap(&tb, d.B, d.K, d.N, d.ldb, CFG::BN);
  static unsigned long long attr_set = 0;
  if (first_on_device(attr_set)) {
    CHASE_CUDA(cudaFuncSetAttribute(zgemm3m_dmma_kernel<CFG, CONJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)CFG::SMEM));
  }
  ZgemmParams p;
  p.M = d.M; p.N = d.N; p.K = d.K;
  p.alpha = d.alpha; p.beta = d.beta; p.gamma = d.gamma;
  p.S = reinterpret_cast<const double2*>(d.S); p.lds = d.lds;
  p.shift_lo = d.shift_lo; p.shift_hi = d.shift_hi; p.shift_off = d.shift_off;
  p.C = reinterpret_cast<double2*>(d.C); p.ldc = d.ldc;
  p.a_chunked = chunked ? 1 : 0;
  p.upper_only = d.upper_only ? 1 : 0;
  p.b_upper = d.b_upper ? 1 : 0;
  if (d.red) {
    if (d.upper_only) throw CudaError("fused all-reduce cannot skip tiles (upper_only)");
    p.red = *d.red;
  }
  static const int group_m = std::getenv("CHASE_ZGEMM_GROUP_M") ? std::atoi(std::getenv("CHASE_ZGEMM_GROUP_M")) : 0;
  p.group_m = group_m;
  const int grid = ceil_div(d.M, CFG::BM) * ceil_div(d.N, CFG::BN);
  zgemm3m_dmma_kernel<CFG, CONJ><<<grid, CFG::THREADS, CFG::SMEM, st>>>(ta, tb, p);
  CHASE_CHECK_LAUNCH();
}

int zgemm3m_tiles(int M, int N) { return ceil_div(M, Z3Default::BM) * ceil_div(N, Z3Default::BN); }

void zgemm(const ZgemmDesc& d0, cudaStream_t st) {
  if (d0.M <= 0 || d0.N <= 0) return;
  if (d0.K <= 0) throw CudaError("zgemm: K must be > 0");
  ZgemmDesc d = d0;
  if (!d.S) d.shift_lo = d.shift_hi = 0;
  if (d.use3m || d.red) {
    if (d.conjA) launch3m<Z3Default, true>(d, st); else launch3m<Z3Default, false>(d, st);
    return;
  }
  if (d.conjA) launch<128, 64, true>(d, st); else launch<128, 64, false>(d, st);
}

}  // namespace chase

// ------------------------------------------------------------------ skinny (L <= 8) product
namespace chase {
namespace {
constexpr int SK_T = 256;      // rows per CTA (one per thread)
constexpr int SK_KB = 128;     // k per shared-memory stage

inline int skinny_splits(int M, int K) {
  const int rb = ceil_div(M, SK_T);
  int s = std::max(1, (148 * 8) / std::max(1, rb));
  s = std::min(s, std::max(1, K / (2 * SK_KB)));
  return s;
}

__device__ __forceinline__ double2 ld_c(const double2* a) { return __ldg(a); }
__device__ __forceinline__ double2 ld_c(const float2* a) {
  const float2 v = __ldg(a);
  return make_double2(v.x, v.y);
}

// TA = double2 (complex double shard) or float2 (complex-single shard, FP64 accumulation)
template <int L, class TA>
__global__ void __launch_bounds__(SK_T) k_skinny(int M, int K, int kchunk, const TA* __restrict__ A,
                                                 int64_t lda, const double2* __restrict__ B, int64_t ldb,
                                                 double2* __restrict__ P) {
  __shared__ double2 Bs[SK_KB][L];
  const int m = blockIdx.x * SK_T + threadIdx.x;
  const int k0 = blockIdx.y * kchunk, k1 = min(K, k0 + kchunk);
  double ar[L], ai[L];
#pragma unroll
  for (int l = 0; l < L; ++l) ar[l] = ai[l] = 0.0;
  for (int kb = k0; kb < k1; kb += SK_KB) {
    const int kn = min(SK_KB, k1 - kb);
    __syncthreads();
    for (int e = threadIdx.x; e < SK_KB * L; e += SK_T) {
      const int kk = e % SK_KB, l = e / SK_KB;
      Bs[kk][l] = kk < kn ? B[(int64_t)(kb + kk) + (int64_t)l * ldb] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    if (m < M) {
      const TA* a = A + m + (int64_t)kb * lda;
#pragma unroll 4
      for (int kk = 0; kk < kn; ++kk) {
        const double2 h = ld_c(a + (int64_t)kk * lda);
#pragma unroll
        for (int l = 0; l < L; ++l) {
          const double2 b = Bs[kk][l];
          ar[l] = fma(h.x, b.x, ar[l]);
          ar[l] = fma(-h.y, b.y, ar[l]);
          ai[l] = fma(h.x, b.y, ai[l]);
          ai[l] = fma(h.y, b.x, ai[l]);
        }
      }
    }
  }
  if (m < M) {
#pragma unroll
    for (int l = 0; l < L; ++l) P[((int64_t)blockIdx.y * L + l) * M + m] = make_double2(ar[l], ai[l]);
  }
}

__global__ void k_skinny_reduce(int M, int L, int splits, double alpha, const double2* __restrict__ P,
                                double2* __restrict__ C, int64_t ldc) {
  const int64_t total = (int64_t)M * L;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i % M), l = (int)(i / M);
    double r = 0.0, im = 0.0;
    for (int s = 0; s < splits; ++s) {
      const double2 v = P[((int64_t)s * L + l) * M + m];
      r += v.x;
      im += v.y;
    }
    C[m + (int64_t)l * ldc] = make_double2(alpha * r, alpha * im);
  }
}
}  // namespace

size_t skinny_work_bytes(int M, int K, int L) { return 16 * (size_t)skinny_splits(M, K) * L * M; }

template <class TA>
static void skinny_launch(int M, int L, int K, const TA* Ad, int64_t lda, const double2* Bd, int64_t ldb, double2* P,
                          dim3 grid, int kchunk, cudaStream_t st) {
  switch (L) {
    case 1: k_skinny<1, TA><<<grid, SK_T, 0, st>>>(M, K, kchunk, Ad, lda, Bd, ldb, P); break;
    case 2: k_skinny<2, TA><<<grid, SK_T, 0, st>>>(M, K, kchunk, Ad, lda, Bd, ldb, P); break;
    case 3: k_skinny<3, TA><<<grid, SK_T, 0, st>>>(M, K, kchunk, Ad, lda, Bd, ldb, P); break;
    case 4: k_skinny<4, TA><<<grid, SK_T, 0, st>>>(M, K, kchunk, Ad, lda, Bd, ldb, P); break;
    case 8: k_skinny<8, TA><<<grid, SK_T, 0, st>>>(M, K, kchunk, Ad, lda, Bd, ldb, P); break;
    default: throw CudaError("zgemm_skinny: L must be 1, 2, 3, 4 or 8");
  }
}

void zgemm_skinny(int M, int L, int K, double alpha, const void* A, int64_t lda, const void* B, int64_t ldb,
                  void* C, int64_t ldc, void* work, cudaStream_t st, bool a_c64) {
  if (M <= 0 || L <= 0) return;
  if (L > 8) throw CudaError("zgemm_skinny: L must be <= 8");
  const int splits = skinny_splits(M, K);
  const int kchunk = ceil_div(K, splits);
  dim3 grid(ceil_div(M, SK_T), splits);
  auto* Bd = reinterpret_cast<const double2*>(B);
  auto* P = reinterpret_cast<double2*>(work);
  if (a_c64)
    skinny_launch(M, L, K, reinterpret_cast<const float2*>(A), lda, Bd, ldb, P, grid, kchunk, st);
  else
    skinny_launch(M, L, K, reinterpret_cast<const double2*>(A), lda, Bd, ldb, P, grid, kchunk, st);
  CHASE_CHECK_LAUNCH();
  const int64_t total = (int64_t)M * L;
  k_skinny_reduce<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, st>>>(
      M, L, splits, alpha, P, reinterpret_cast<double2*>(C), ldc);
  CHASE_CHECK_LAUNCH();
}
}  // namespace chase

// ------------------------------------------------------------------ real (f2) GEMM launcher
#include "dgemm.cuh"
namespace chase {
// Real tensor maps: dim 0 = rows (doubles, contiguous), dim 1 = cols; box {16 doubles, box_cols}.
static void make_dmatrix_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                              int box_cols) {
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {16u, (cuuint32_t)box_cols};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = get_encode()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (real) failed");
}

static bool make_dmatrix_tmap_chunked(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                                      int box_cols, int box_chunks) {
  if (rows % 16 != 0) return false;
  cuuint64_t dims[3] = {16u, (cuuint64_t)cols, (cuuint64_t)(rows / 16)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 8), 128u};
  cuuint32_t box[3] = {16u, (cuuint32_t)box_cols, (cuuint32_t)box_chunks};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = get_encode()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool TRANS, bool TMA>
static void launch_d(const ZgemmDesc& d, cudaStream_t st) {
  static unsigned long long attr_set = 0;
  if (first_on_device(attr_set)) {
    CHASE_CUDA(cudaFuncSetAttribute(dgemm_dmma_kernel<TRANS, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)DCfg::SMEM));
  }
  CUtensorMap ta{}, tb{};
  bool chunked = false;
  if (TMA) {
    if (!TRANS) {
      chunked = make_dmatrix_tmap_chunked(&ta, d.A, d.M, d.K, d.lda, DCfg::BK, DCfg::BM / 16);
      if (!chunked) make_dmatrix_tmap(&ta, d.A, d.M, d.K, d.lda, DCfg::BK);
    } else {
      make_dmatrix_tmap(&ta, d.A, d.K, d.M, d.lda, DCfg::BM);
    }
    make_dmatrix_tmap(&tb, d.B, d.K, d.N, d.ldb, DCfg::BN);
  }
  DgemmParams p;
  p.M = d.M; p.N = d.N; p.K = d.K;
  p.alpha = d.alpha; p.beta = d.beta; p.gamma = d.gamma;
  p.A = reinterpret_cast<const double*>(d.A); p.lda = d.lda;
  p.B = reinterpret_cast<const double*>(d.B); p.ldb = d.ldb;
  p.S = reinterpret_cast<const double*>(d.S); p.lds = d.lds;
  p.shift_lo = d.shift_lo; p.shift_hi = d.shift_hi; p.shift_off = d.shift_off;
  p.C = reinterpret_cast<double*>(d.C); p.ldc = d.ldc;
  p.upper_only = d.upper_only ? 1 : 0;
  p.b_upper = d.b_upper ? 1 : 0;
  p.a_chunked = chunked ? 1 : 0;
  if (d.red) {
    if (d.upper_only) throw CudaError("fused all-reduce cannot skip tiles (upper_only)");
    p.red = *d.red;
  }
  const int grid = ceil_div(d.M, DCfg::BM) * ceil_div(d.N, DCfg::BN);
  dgemm_dmma_kernel<TRANS, TMA><<<grid, DCfg::THREADS, DCfg::SMEM, st>>>(ta, tb, p);
  CHASE_CHECK_LAUNCH();
}

int dgemm_tiles(int M, int N) { return ceil_div(M, DCfg::BM) * ceil_div(N, DCfg::BN); }

void dgemm(const ZgemmDesc& d0, cudaStream_t st) {
  if (d0.M <= 0 || d0.N <= 0) return;
  if (d0.K <= 0) throw CudaError("dgemm: K must be > 0");
  ZgemmDesc d = d0;
  if (!d.S) d.shift_lo = d.shift_hi = 0;
  // TMA needs 16-byte aligned bases and leading dimensions that are a multiple of 16 bytes
  const bool tma = (reinterpret_cast<uintptr_t>(d.A) % 16 == 0) && (reinterpret_cast<uintptr_t>(d.B) % 16 == 0) &&
                   (d.lda % 2 == 0) && (d.ldb % 2 == 0);
  if (d.conjA) {
    if (tma) launch_d<true, true>(d, st); else launch_d<true, false>(d, st);
  } else {
    if (tma) launch_d<false, true>(d, st); else launch_d<false, false>(d, st);
  }
}
}  // namespace chase

// ------------------------------------------------------------------ real skinny (Lanczos, f2)
namespace chase {
namespace {
template <int L>
__global__ void __launch_bounds__(SK_T) k_skinny_real(int M, int K, int kchunk, const double* __restrict__ A,
                                                      int64_t lda, const double* __restrict__ B, int64_t ldb,
                                                      double* __restrict__ P) {
  __shared__ double Bs[SK_KB][L];
  const int m = blockIdx.x * SK_T + threadIdx.x;
  const int k0 = blockIdx.y * kchunk, k1 = min(K, k0 + kchunk);
  double ar[L];
#pragma unroll
  for (int l = 0; l < L; ++l) ar[l] = 0.0;
  for (int kb = k0; kb < k1; kb += SK_KB) {
    const int kn = min(SK_KB, k1 - kb);
    __syncthreads();
    for (int e = threadIdx.x; e < SK_KB * L; e += SK_T) {
      const int kk = e % SK_KB, l = e / SK_KB;
      Bs[kk][l] = kk < kn ? B[(int64_t)(kb + kk) + (int64_t)l * ldb] : 0.0;
    }
    __syncthreads();
    if (m < M) {
      const double* a = A + m + (int64_t)kb * lda;
#pragma unroll 4
      for (int kk = 0; kk < kn; ++kk) {
        const double h = __ldg(a + (int64_t)kk * lda);
#pragma unroll
        for (int l = 0; l < L; ++l) ar[l] = fma(h, Bs[kk][l], ar[l]);
      }
    }
  }
  if (m < M) {
#pragma unroll
    for (int l = 0; l < L; ++l) P[((int64_t)blockIdx.y * L + l) * M + m] = ar[l];
  }
}

__global__ void k_skinny_reduce_real(int M, int L, int splits, double alpha, const double* __restrict__ P,
                                     double* __restrict__ C, int64_t ldc) {
  const int64_t total = (int64_t)M * L;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i % M), l = (int)(i / M);
    double r = 0.0;
    for (int s = 0; s < splits; ++s) r += P[((int64_t)s * L + l) * M + m];
    C[m + (int64_t)l * ldc] = alpha * r;
  }
}
}  // namespace

void dgemm_skinny(int M, int L, int K, double alpha, const void* A, int64_t lda, const void* B, int64_t ldb,
                  void* C, int64_t ldc, void* work, cudaStream_t st) {
  if (M <= 0 || L <= 0) return;
  const int splits = skinny_splits(M, K);
  const int kchunk = ceil_div(K, splits);
  dim3 grid(ceil_div(M, SK_T), splits);
  auto* Ad = reinterpret_cast<const double*>(A);
  auto* Bd = reinterpret_cast<const double*>(B);
  auto* P = reinterpret_cast<double*>(work);
  switch (L) {
    case 1: k_skinny_real<1><<<grid, SK_T, 0, st>>>(M, K, kchunk, Ad, lda, Bd, ldb, P); break;
    case 2: k_skinny_real<2><<<grid, SK_T, 0, st>>>(M, K, kchunk, Ad, lda, Bd, ldb, P); break;
    case 3: k_skinny_real<3><<<grid, SK_T, 0, st>>>(M, K, kchunk, Ad, lda, Bd, ldb, P); break;
    case 4: k_skinny_real<4><<<grid, SK_T, 0, st>>>(M, K, kchunk, Ad, lda, Bd, ldb, P); break;
    case 8: k_skinny_real<8><<<grid, SK_T, 0, st>>>(M, K, kchunk, Ad, lda, Bd, ldb, P); break;
    default: throw CudaError("dgemm_skinny: L must be 1, 2, 3, 4 or 8");
  }
  CHASE_CHECK_LAUNCH();
  const int64_t total = (int64_t)M * L;
  k_skinny_reduce_real<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, st>>>(
      M, L, splits, alpha, P, reinterpret_cast<double*>(C), ldc);
  CHASE_CHECK_LAUNCH();
}
}  // namespace chase
