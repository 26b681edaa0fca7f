// Host launcher for the TMA + DMMA complex GEMM (zgemm.cuh) and the tensor-map encoder.
#include "zgemm.h"
#include "zgemm.cuh"

namespace chase {

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CHASE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
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

template <int BM, int BN, bool CONJ>
static void launch(const ZgemmDesc& d, cudaStream_t st) {
  using C_ = zg::Cfg<BM, BN>;
  CUtensorMap ta, tb;
  if (!CONJ)
    make_zmatrix_tmap(&ta, d.A, d.M, d.K, d.lda, zg::BK);      // A: M x K
  else
    make_zmatrix_tmap(&ta, d.A, d.K, d.M, d.lda, BM);          // A: K x M (op = A^H)
  make_zmatrix_tmap(&tb, d.B, d.K, d.N, d.ldb, BN);
  static bool attr_set = false;
  if (!attr_set) {
    CHASE_CUDA(cudaFuncSetAttribute(zgemm_dmma_kernel<BM, BN, CONJ>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C_::SMEM));
    attr_set = true;
  }
  ZgemmParams p;
  p.M = d.M; p.N = d.N; p.K = d.K;
  p.alpha = d.alpha; p.beta = d.beta; p.gamma = d.gamma;
  p.S = reinterpret_cast<const double2*>(d.S); p.lds = d.lds;
  p.shift_lo = d.shift_lo; p.shift_hi = d.shift_hi; p.shift_off = d.shift_off;
  p.C = reinterpret_cast<double2*>(d.C); p.ldc = d.ldc;
  const int grid = ceil_div(d.M, BM) * ceil_div(d.N, BN);
  zgemm_dmma_kernel<BM, BN, CONJ><<<grid, C_::THREADS, C_::SMEM, st>>>(ta, tb, p);
  CHASE_CHECK_LAUNCH();
}

void zgemm(const ZgemmDesc& d, cudaStream_t st) {
  if (d.M <= 0 || d.N <= 0) return;
  if (d.K <= 0) throw CudaError("zgemm: K must be > 0");
  if (!d.S) {
    ZgemmDesc e = d;
    e.shift_lo = e.shift_hi = 0;
    if (d.conjA) launch<128, 64, true>(e, st); else launch<128, 64, false>(e, st);
    return;
  }
  if (d.conjA) launch<128, 64, true>(d, st); else launch<128, 64, false>(d, st);
}

}  // namespace chase
