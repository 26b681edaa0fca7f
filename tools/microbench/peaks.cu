// Roofline denominators for the filter kernels, measured on the B200 (sm_100a) they run on
// ("measured sustained DMMA FP64 peak ... >= 4 s back-to-back" and "TF32 dense
// peak ... measure it"):
//   * FP64 tensor: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), the only FP64 tensor path on sm_100a;
//   * TF32 tensor: tcgen05.mma.cta_group::1.kind::tf32, M = 128, N = 256, K = 8, operands in
//     128-B-swizzled shared memory (random data, so the power draw is realistic), accumulators in
//     TMEM, issued back to back by one elected thread per SM with double-buffered commits.
// For each: "burst" = one ~60 ms launch after 3 s idle; "sustained" = back-to-back launches for
// >= 6 s, rate over the last 4 s (median of the per-launch rates there).  One JSON line each;
// tools/microbench/run_peaks.sh records nvidia-smi clocks alongside.
#include <cuda_runtime.h>
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <thread>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  return d;
}

constexpr int TM = 128, TN = 256;
constexpr int GROUP = 32;                    // MMAs per commit group

// KIND 0: kind::tf32 (F32 accumulate); KIND 1: kind::i8 (signed int8 A/B, S32 accumulate).  Both
// read 32-byte K slices of the 128-byte swizzled rows (8 tf32 or 32 int8 per MMA).
template <int KIND>
__global__ void __launch_bounds__(128, 1) mma_loop(int groups, float* out) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = sm;                    // 128 rows x 128 B (32 tf32 of k), K-major, SW128
  unsigned char* sB = sm + TM * 128;         // 256 rows x 128 B
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  // random operands (a hash of the byte offset): realistic toggling in the datapath (for i8 the
  // same words read as four int8 values each)
  uint32_t* w = reinterpret_cast<uint32_t*>(sm);
  for (int i = threadIdx.x; i < (TM + TN) * 32; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + blockIdx.x * 40503u;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    w[i] = 0x3f000000u | (x & 0x007fffffu) | ((x & 1u) << 31);    // +-[0.5, 1)
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    uint32_t leader;
    asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(leader));
    if (leader) {
      // tf32: F32 accumulate (1 << 4), TF32 A / B (2 << 7, 2 << 10); i8: S32 accumulate (2 << 4),
      // signed 8-bit A / B (1 << 7, 1 << 10); both K-major, N = 256, M = 128
      const uint32_t idesc = (KIND == 0 ? ((1u << 4) | (2u << 7) | (2u << 10)) : ((2u << 4) | (1u << 7) | (1u << 10))) |
                             ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
      uint32_t phase[2] = {0, 0};
      for (int g = 0; g < groups; ++g) {
        const int b = g & 1;
        if (g >= 2) {                          // group g-2 done before its barrier is reused
          asm volatile("{ .reg .pred P; W1: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W1; }"
                       ::"r"(su32(&bar[b])), "r"(phase[b]));
          phase[b] ^= 1;
        }
#pragma unroll 4
        for (int i = 0; i < GROUP; ++i) {
          const int kk = i & 3;                // K = 8 tf32 = 32 B steps inside the 128-B rows
          const uint64_t da = sdesc(su32(sA) + kk * 32, 16, 1024);
          const uint64_t db = sdesc(su32(sB) + kk * 32, 16, 1024);
          const uint32_t acc = (g > 0 || i > 0) ? 1u : 0u;
          if constexpr (KIND == 0)
            asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                         ::"r"(tmem_base), "l"(da), "l"(db), "r"(idesc), "r"(acc));
          else
            asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                         ::"r"(tmem_base), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[b])));
      }
      for (int b = 0; b < 2 && b < groups; ++b)
        asm volatile("{ .reg .pred P; W2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W2; }"
                     ::"r"(su32(&bar[(groups - 1 - b) & 1])), "r"(phase[(groups - 1 - b) & 1]));
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    uint32_t r0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r0) : "r"(tmem_base));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (__uint_as_float(r0) == 12345.0f) out[0] = 1.0f;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TN));
  }
}

template <class Launch>
static int measure(const char* name, double flop_per_launch, Launch launch, double burst_ms_target) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();                                       // warm-up (module load, clocks up)
  cudaDeviceSynchronize();
  std::this_thread::sleep_for(std::chrono::seconds(3));     // idle: burst starts from a cool, uncapped GPU
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float bms = 0.f;
  cudaEventElapsedTime(&bms, e0, e1);
  const double burst = flop_per_launch / (bms * 1e-3) / 1e12;
  std::vector<float> ms;
  std::vector<double> t_end;
  const auto t0 = std::chrono::steady_clock::now();
  double el = 0.0;
  while (el < 6.5) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float m = 0.f;
    cudaEventElapsedTime(&m, e0, e1);
    ms.push_back(m);
    el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    t_end.push_back(el);
  }
  std::vector<double> rates;
  double win = 0.0;
  for (size_t i = 0; i < ms.size(); ++i)
    if (t_end[i] >= el - 4.0) { rates.push_back(flop_per_launch / (ms[i] * 1e-3) / 1e12); win += ms[i] * 1e-3; }
  std::sort(rates.begin(), rates.end());
  const double sustained = rates[rates.size() / 2];
  const cudaError_t err = cudaGetLastError();
  printf("{\"kernel\":\"%s\",\"burst_tflops\":%.3f,\"burst_ms\":%.2f,\"sustained_tflops\":%.3f,"
         "\"sustained_window_s\":%.2f,\"sustained_total_s\":%.2f,\"launches\":%zu,\"min_tflops\":%.3f,\"max_tflops\":%.3f,"
         "\"status\":\"%s\"}\n",
         name, burst, bms, sustained, win, el, ms.size(), rates.front(), rates.back(), cudaGetErrorString(err));
  fflush(stdout);
  (void)burst_ms_target;
  return err == cudaSuccess ? 0 : 1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d = nullptr;
  CK(cudaMalloc(&d, 64));
  // FP64 DMMA: 148 x 2 CTAs of 8 warps, 8 independent DMMA.8x8x4 (512 flop each) per iteration
  {
    const int warps = 8, iters = 240000;
    const double flop = 2.0 * sms * warps * 8.0 * iters * 512.0;
    if (measure("dmma_m8n8k4_f64", flop, [&] { dmma_loop<<<sms * 2, warps * 32>>>((double*)d, iters); }, 60)) return 1;
  }
  // TF32 tcgen05: one CTA per SM, 2 x 128 x 256 x 8 flop per MMA
  {
    const int smem = (TM + TN) * 128 + 1024;
    CK(cudaFuncSetAttribute(mma_loop<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int groups = 30000;
    const double flop = 2.0 * TM * TN * 8.0 * GROUP * groups * sms;
    if (measure("tcgen05_mma_kind_tf32_m128n256k8", flop, [&] { mma_loop<0><<<sms, 128, smem>>>(groups, d); }, 60)) return 1;
  }
  // INT8 tcgen05 (the Ozaki-scheme FP64 emulation's engine): 2 x 128 x 256 x 32 ops per MMA
  {
    const int smem = (TM + TN) * 128 + 1024;
    CK(cudaFuncSetAttribute(mma_loop<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int groups = 60000;
    const double ops = 2.0 * TM * TN * 32.0 * GROUP * groups * sms;
    if (measure("tcgen05_mma_kind_i8_m128n256k32", ops, [&] { mma_loop<1><<<sms, 128, smem>>>(groups, d); }, 60)) return 1;
  }
  return 0;
}
