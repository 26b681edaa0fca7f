// tcgen05 kind::i8 probe: is an MN-major (M-contiguous) int8 A operand accepted on sm_100a, and
// with which descriptor?  One CTA: C[128 x 64] = A[128 x K] B[K x 64], K = 128, A stored [k][m]
// (m contiguous, as a column-major H read as the forward operand), B K-major.  Tries LBO/SBO
// variants; prints max abs error vs the CPU product for each (0 = exact = usable).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
constexpr int M = 128, N = 64, K = 128;
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, int layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}
__global__ void probe(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, int* C, int lbo, int sbo, int kstep) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = sm;            // [k 0..127][m 128 B]  = 16 KB
  unsigned char* sB = sm + 16384;    // [n 0..63][k 128 B]   = 8 KB
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
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar_tma)), "r"(16384 + 8192));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(sA)), "l"((uint64_t)&tA), "r"(0), "r"(0), "r"(su32(&bar_tma)) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(sB)), "l"((uint64_t)&tB), "r"(0), "r"(0), "r"(su32(&bar_tma)) : "memory");
  }
  asm volatile("{ .reg .pred P; W1: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W1; }" ::"r"(su32(&bar_tma)));
  if (warp == 0) {
    uint32_t leader;
    asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(leader));
    if (leader) {
      // S32 accum, s8 A / B, A MN-major (bit 15), B K-major, N = 64, M = 128
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
      for (int kk = 0; kk < K / 32; ++kk) {
        const uint64_t da = sdesc(su32(sA) + kk * kstep, lbo, sbo, 2);
        const uint64_t db = sdesc(su32(sB) + kk * 32, 16, 1024, 2);
        const uint32_t acc = kk > 0 ? 1u : 0u;
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                     ::"r"(tmem_base), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar_mma)));
    }
    __syncwarp();
  }
  asm volatile("{ .reg .pred P; W2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W2; }" ::"r"(su32(&bar_mma)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem_base + ((uint32_t)(32 * warp) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int m = 32 * warp + lane;
    for (int j = 0; j < 16; ++j) C[m + (c0 + j) * M] = (int)r[j];
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(64));
}
static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}
static void tmap(CUtensorMap* m, void* base, uint64_t inner, uint64_t outer, uint32_t box_inner, uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t str[1] = {inner};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("tmap fail %d\n", (int)r); exit(1); }
}
int main() {
  std::vector<int8_t> A(M * K), B(K * N);   // A stored [k][m] (m contiguous); B stored [n][k]
  srand(3);
  for (auto& x : A) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : B) x = (int8_t)(rand() % 255 - 127);
  int8_t *dA, *dB; int* dC;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dC, 4 * M * N));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CUtensorMap tA, tB;
  tmap(&tA, dA, M, K, 128, K);   // [k][m]: inner m (128 B), outer k
  tmap(&tB, dB, K, N, 128, N);   // [n][k]: inner k
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 30 * 1024));
  std::vector<int> C(M * N);
  const int variants[][3] = {{16, 1024, 4096}, {1024, 16, 4096}, {0, 1024, 4096}, {8192, 1024, 4096}, {128, 1024, 4096}, {1024, 128, 4096}};
  for (auto& v : variants) {
    CK(cudaMemset(dC, 0, 4 * M * N));
    probe<<<1, 128, 30 * 1024>>>(tA, tB, dC, v[0], v[1], v[2]);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("{\"lbo\":%d,\"sbo\":%d,\"error\":\"%s\"}\n", v[0], v[1], cudaGetErrorString(e)); return 0; }
    CK(cudaMemcpy(C.data(), dC, 4 * M * N, cudaMemcpyDeviceToHost));
    long long maxerr = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        long long ref = 0;
        for (int k = 0; k < K; ++k) ref += (long long)A[m + k * M] * B[k + n * K];
        maxerr = std::max(maxerr, std::llabs(ref - C[m + n * M]));
      }
    printf("{\"lbo\":%d,\"sbo\":%d,\"kstep\":%d,\"max_abs_err\":%lld,\"C00\":%d}\n", v[0], v[1], v[2], maxerr, C[0]);
  }
  return 0;
}
