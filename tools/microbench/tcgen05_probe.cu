// tcgen05 (5th-gen tensor core) TF32 probe for sm_100a: validates the UMMA shared-memory and
// instruction descriptor encodings, TMEM alloc / MMA / commit / ld, with an MN-major A (column-major
// M x K, as the H shard in the forward filter step) and a K-major B (column-major K x N, as V).
// One CTA: C[128 x 64] = A[128 x K] * B[K x 64], K = 64 (8 MMAs of K = 8).  Prints max rel error.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int M = 128, N = 64, K = 64;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, int lbo_mode = 0, int layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)(lbo_mode & 1) << 52;
  d |= (uint64_t)(layout & 7) << 61;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                 // version = 1 (sm100)
  return d;
}

__global__ void probe(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tAk,
                      const __grid_constant__ CUtensorMap tB, float* C, int mode) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = sm;                 // 4 m-chunks x (64 k x 128 B) = 32 KB
  unsigned char* sB = sm + 32768;         // 2 k-chunks x (64 n x 128 B) = 16 KB
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_tma)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_mma)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar_tma)), "r"(49152));
    if (mode & 1) {
      for (int c = 0; c < 4; ++c)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su32(sA + c * 8192)), "l"((uint64_t)&tA), "r"(32 * c), "r"(0), "r"(su32(&bar_tma)) : "memory");
    } else {   // A row-major (K-major): box 32 k x 128 m per k-chunk -> [k-chunk][m][32 k]
      for (int c = 0; c < 2; ++c)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su32(sA + c * 16384)), "l"((uint64_t)&tAk), "r"(32 * c), "r"(0), "r"(su32(&bar_tma)) : "memory");
    }
    for (int c = 0; c < 2; ++c)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sB + c * 8192)), "l"((uint64_t)&tB), "r"(32 * c), "r"(0), "r"(su32(&bar_tma)) : "memory");
  }
  // wait TMA
  asm volatile("{ .reg .pred P; W1: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W1; }" ::"r"(su32(&bar_tma)));
  if (threadIdx.x == 0 && mode >= 99) {
    const float* fa = (const float*)sA; const float* fb = (const float*)sB;
    printf("smem A %f %f %f | B %f %f %f | tmem %u\n", fa[0], fa[1], fa[33], fb[0], fb[1], fb[33], tmem_base);
  }
  if (warp == 0) {
    uint32_t is_leader;
    asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(is_leader));
    if (is_leader) {
    // instruction descriptor: F32 accum, TF32 A/B, A MN-major, B K-major, N=64, M=128
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((mode & 1 ? 1u : 0u) << 15) | (0u << 16) |
                     ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int kk = 0; kk < K / 8; ++kk) {
      // A (MN-major, SW128): atom = 128 B of m x 8 k-rows; LBO = stride between m-atoms (8 KB box),
      // SBO = stride between 8-k groups (1 KB)
      const int v = mode >> 1;
      // MN-major tf32 needs the 128B-swizzle-with-32B-atoms layout (UMMA layout type 1, TMA
      // SWIZZLE_128B_ATOM_32B): atom = 128 B of m x 4 k-rows
      const uint64_t da = (mode & 1) ? (v == 0 ? sdesc(su32(sA) + kk * 1024, 8192, 512, 0, 1)
                                       : v == 1 ? sdesc(su32(sA) + kk * 1024, 512, 8192, 0, 1)
                                       : sdesc(su32(sA) + kk * 1024, 8192, 1024, 0, 1))
                                     : sdesc(su32(sA) + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024);
      // B (K-major, SW128): rows of 32 k; SBO = 8 rows (1 KB); K = 8 tf32 = 32 B per MMA
      const uint64_t db = sdesc(su32(sB) + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024);
      const uint32_t acc = kk > 0 ? 1u : 0u;
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                   ::"r"(tmem_base), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar_mma)));
    }
    __syncwarp();
  }
  asm volatile("{ .reg .pred P; W2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W2; }" ::"r"(su32(&bar_mma)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w reads TMEM lanes 32w..32w+31 (rows), 64 columns
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    const uint32_t taddr = tmem_base + ((uint32_t)(32 * warp) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int m = 32 * warp + lane;
    if (mode >= 99 && threadIdx.x == 0 && c0 == 0) printf("tmem r0 %08x %f\n", r[0], __uint_as_float(r[0]));
    for (int j = 0; j < 16; ++j) C[m + (c0 + j) * M] = __uint_as_float(r[j]);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(64));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}

static void tmap(CUtensorMap* m, void* base, uint64_t rows, uint64_t cols, uint32_t box_cols,
                 CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  cuuint64_t dims[2] = {rows, cols};
  cuuint64_t str[1] = {rows * 4};
  cuuint32_t box[2] = {32, box_cols};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("tmap fail %d\n", (int)r); exit(1); }
}

int main() {
  std::vector<float> A(M * K), B(K * N), C(M * N);
  srand(1);
  for (auto& x : A) x = (rand() / (float)RAND_MAX) - 0.5f;
  for (auto& x : B) x = (rand() / (float)RAND_MAX) - 0.5f;
  float *dA, *dB, *dC;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dC, C.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  std::vector<float> Ak(M * K);
  for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) Ak[k + m * K] = A[m + k * M];
  float* dAk; CK(cudaMalloc(&dAk, Ak.size() * 4));
  CK(cudaMemcpy(dAk, Ak.data(), Ak.size() * 4, cudaMemcpyHostToDevice));
  CUtensorMap tA, tAk, tB;
  tmap(&tAk, dAk, K, M, M);   // A^T col-major K x M (k contiguous): box 32 k x 128 m
  tmap(&tA, dA, M, K, K, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);   // A col-major M x K: box 32 m x 64 k
  tmap(&tB, dB, K, N, N);     // B col-major K x N (k contiguous): box 32 k x 64 n
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024));
  for (int mode = 0; mode <= 5; ++mode) {
    if (mode == 2 || mode == 4) continue;
    CK(cudaMemset(dC, 0, C.size() * 4));
    probe<<<1, 128, 50 * 1024>>>(tA, tAk, tB, dC, mode);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[m + k * M] * B[k + n * K];
        maxerr = fmax(maxerr, fabs(ref - C[m + n * M]));
        maxref = fmax(maxref, fabs(ref));
      }
    printf("{\"mode\":%d,\"probe\":\"tcgen05 tf32 A x K-major B\",", mode); printf("\"max_abs_err\":%.3e,\"max_ref\":%.3e,\"rel\":%.3e,\"C00\":%.6f}\n",
           maxerr, maxref, maxerr / maxref, C[0]);
  }
  return 0;
}
