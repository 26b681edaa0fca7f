// Real-double GEMM with the fused Chebyshev-step epilogue: the real-symmetric variant (
// the paper's own experiments are real symmetric).
//
//   C[M x N] = alpha * op(A) * B  -  alpha*gamma * S[shift rows]  +  beta * C,  op(A) = A or A^T
//
// FP64 DMMA.8x8x4 (one MMA per real multiply-add).  8 warps of 64 (m) x 32 (n) accumulators
// (128 registers) on a 128 x 128 CTA tile, BK = 32 real k per stage, 3-stage ring.  Operand tiles
// are staged with cp.async (8-byte, zero-filled out of bounds): real shards may have odd leading
// dimensions and odd row offsets, which TMA's 16-byte alignment rules exclude.  Shared memory uses
// the same XOR-128B swizzle as the TMA path: 128-byte rows of 16 doubles, 16-byte chunk index XOR
// (row % 8).  With the k permutation kk(t, s) = 2 s + (t & 1) + 8 (t >> 1) the 16 lanes of a
// half-warp read 8 distinct chunks x 2 halves (conflict-free) for B and transposed A; forward-A
// rows hold 16 m values and are read 2-way conflicted (8 of 12 fragment loads per 32 DMMAs).
#pragma once
#include "common.cuh"
#include "tma.cuh"
#include "zgemm.h"
#include "zgemm.cuh"

namespace chase {

struct DCfg {
  static constexpr int WM = 2, WN = 4, STAGES = 3;
  static constexpr int BM = 64 * WM, BN = 32 * WN, BK = 32;
  static constexpr int NWARPS = WM * WN, THREADS = NWARPS * 32;
  static constexpr uint32_t A_BYTES = BM * BK * 8, B_BYTES = BK * BN * 8, STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 2 * STAGES * 8 + 1024;
};

struct DgemmParams {
  int M, N, K;
  double alpha, beta, gamma;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  const double* S;
  int64_t lds;
  int shift_lo, shift_hi;
  int64_t shift_off;
  double* C;
  int64_t ldc;
  int upper_only;
  int b_upper;
  int a_chunked;        // TMA path: forward A as one 3-D box (M % 16 == 0)
  PeerRed red;          // f1: fused all-reduce over peer memory (buffers hold doubles; red.n <= 1: off)
};

namespace dg {
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, bool pred) {
  const int sz = pred ? 8 : 0;   // src-size 0 -> zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// byte offset of element (row r of 128 B, index x in [0,16)) in a swizzled tile
__device__ __forceinline__ uint32_t soff(int r, int x) {
  return (uint32_t)(r * 128 + ((((x >> 1) ^ (r & 7))) << 4) + ((x & 1) << 3));
}
}  // namespace dg

// USE_TMA: operands 16-byte aligned with even leading dimensions -> TMA boxes filled by thread 0
// into an mbarrier ring (as zgemm.cuh); otherwise cooperative 8-byte cp.async with a
// __syncthreads ring.  Both produce the identical swizzled shared-memory layout.
template <bool TRANS_A, bool USE_TMA>
__global__ void __launch_bounds__(DCfg::THREADS, 1)
    dgemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      DgemmParams p) {
  constexpr int WN = DCfg::WN, STAGES = DCfg::STAGES, BM = DCfg::BM, BN = DCfg::BN, BK = DCfg::BK;
  constexpr int THREADS = DCfg::THREADS;
  constexpr uint32_t A_BYTES = DCfg::A_BYTES, STAGE_BYTES = DCfg::STAGE_BYTES;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int tiles_n = (p.N + BN - 1) / BN;
  const int tiles_m = (p.M + BM - 1) / BM;
  constexpr int GROUP_M = 8;
  const int per_group = GROUP_M * tiles_n;
  const int group = blockIdx.x / per_group;
  const int first_m = group * GROUP_M;
  const int gsize = min(tiles_m - first_m, GROUP_M);
  const int in_group = blockIdx.x % per_group;
  const int m0 = (first_m + in_group % gsize) * BM;
  const int n0 = (in_group / gsize) * BN;
  if (p.upper_only && m0 >= n0 + BN) return;
  const int KT = p.b_upper ? (min(p.K, n0 + BN) + BK - 1) / BK : (p.K + BK - 1) / BK;
  const uint32_t smem_base = smem_u32(smem);

  // cooperative staging of k-tile kt into slot kt % STAGES
  auto stage_load = [&](int kt) {
    const uint32_t sa = smem_base + (kt % STAGES) * STAGE_BYTES;
    const uint32_t sb = sa + A_BYTES;
    const int k0 = kt * BK;
    // A: BM x BK elements
#pragma unroll 2
    for (int it = 0; it < (BM * BK) / THREADS; ++it) {
      const int e = tid + it * THREADS;
      if constexpr (!TRANS_A) {
        // A col-major M x K (m contiguous): smem [BM/16][BK][16 m]
        const int m = e % BM, k = e / BM;
        const int gm = m0 + m, gk = k0 + k;
        const bool ok = gm < p.M && gk < p.K;
        const double* src = p.A + (ok ? (int64_t)gm + (int64_t)gk * p.lda : 0);
        dg::cp_async8(sa + dg::soff((m >> 4) * BK + k, m & 15), src, ok);
      } else {
        // A col-major K x M (k contiguous), op = A^T: smem [BK/16][BM][16 k]
        const int k = e % BK, m = e / BK;
        const int gm = m0 + m, gk = k0 + k;
        const bool ok = gm < p.M && gk < p.K;
        const double* src = p.A + (ok ? (int64_t)gk + (int64_t)gm * p.lda : 0);
        dg::cp_async8(sa + dg::soff((k >> 4) * BM + m, k & 15), src, ok);
      }
    }
    // B: BK x BN, col-major (k contiguous): smem [BK/16][BN][16 k]
#pragma unroll 2
    for (int it = 0; it < (BK * BN) / THREADS; ++it) {
      const int e = tid + it * THREADS;
      const int k = e % BK, n = e / BK;
      const int gk = k0 + k, gn = n0 + n;
      const bool ok = gk < p.K && gn < p.N;
      const double* src = p.B + (ok ? (int64_t)gk + (int64_t)gn * p.ldb : 0);
      dg::cp_async8(sb + dg::soff((k >> 4) * BN + n, k & 15), src, ok);
    }
  };

  auto tma_issue = [&](int kt) {
    const int s = kt % STAGES;
    unsigned char* sa = smem + s * STAGE_BYTES;
    unsigned char* sb = sa + A_BYTES;
    mbar_arrive_expect_tx(full + s, STAGE_BYTES);
    const int k0 = kt * BK;
    if constexpr (!TRANS_A) {
      if (p.a_chunked) {
        tma_load_3d(sa, &tmA, 0, k0, m0 / 16, full + s);
      } else {
#pragma unroll
        for (int c = 0; c < BM / 16; ++c) tma_load_2d(sa + c * (BK * 128), &tmA, m0 + 16 * c, k0, full + s);
      }
    } else {
#pragma unroll
      for (int kc = 0; kc < BK / 16; ++kc) tma_load_2d(sa + kc * (BM * 128), &tmA, k0 + 16 * kc, m0, full + s);
    }
#pragma unroll
    for (int kc = 0; kc < BK / 16; ++kc) tma_load_2d(sb + kc * (BN * 128), &tmB, k0 + 16 * kc, n0, full + s);
  };
  if constexpr (USE_TMA) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(full + s, 1);
        mbar_init(empty + s, DCfg::NWARPS);
      }
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      for (int kt = 0; kt < STAGES - 1 && kt < KT; ++kt) tma_issue(kt);
    }
  } else {
#pragma unroll
    for (int kt = 0; kt < STAGES - 1; ++kt) {
      if (kt < KT) stage_load(kt);
      dg::cp_commit();
    }
  }

  const int wm = warp / WN, wn = warp % WN;
  const int g = lane >> 2, t = lane & 3;
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    if constexpr (USE_TMA) {
      if (threadIdx.x == 0 && kt + STAGES - 1 < KT) {
        if (kt >= 1) mbar_wait(empty + (kt - 1) % STAGES, ((kt - 1) / STAGES) & 1);
        tma_issue(kt + STAGES - 1);
      }
      mbar_wait(full + kt % STAGES, (kt / STAGES) & 1);
    } else {
      dg::cp_wait<STAGES - 2>();
      __syncthreads();                         // tile kt visible; slot of tile kt-1 free
      if (kt + STAGES - 1 < KT) stage_load(kt + STAGES - 1);
      dg::cp_commit();
    }
    const uint32_t sa = smem_base + (kt % STAGES) * STAGE_BYTES;
    const uint32_t sb = sa + A_BYTES;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int kc = ks >> 2;
      const int kk = 2 * (ks & 3) + (t & 1) + 8 * (t >> 1);
      double a[8], b[4];
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        if constexpr (!TRANS_A) {
          const int m = wm * 64 + mt * 8 + g;
          a[mt] = dg::lds64(sa + dg::soff((m >> 4) * BK + kc * 16 + kk, m & 15));
        } else {
          a[mt] = dg::lds64(sa + dg::soff(kc * BM + wm * 64 + mt * 8 + g, kk));
        }
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) b[nt] = dg::lds64(sb + dg::soff(kc * BN + wn * 32 + nt * 8 + g, kk));
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) zg::dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
    }
    if constexpr (USE_TMA) {
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + kt % STAGES);
    }
  }
  if constexpr (!USE_TMA) dg::cp_wait<0>();

  const double ag = p.alpha * p.gamma;
  const bool fused = p.red.n > 1;
  double* dst = fused ? reinterpret_cast<double*>(p.red.stage[p.red.me]) + p.red.off : p.C;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    const int m = m0 + wm * 64 + mt * 8 + g;
    if (m >= p.M) continue;
    const bool shifted = (m >= p.shift_lo) && (m < p.shift_hi);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = n0 + wn * 32 + nt * 8 + 2 * t + j;
        if (n >= p.N) continue;
        double v = p.alpha * acc[mt][nt][j];
        if (shifted) v -= ag * p.S[(int64_t)m + p.shift_off + (int64_t)n * p.lds];
        const int64_t o = (int64_t)m + (int64_t)n * p.ldc;
        if (p.beta != 0.0) v += p.beta * p.C[o];
        dst[o] = v;
      }
    }
  }
  if (!fused) return;
  // ---- f1 (see zgemm3m.cuh): last of the n ranks to arrive on this tile reduces and broadcasts
  __shared__ int s_last;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned old = atomicAdd_system(p.red.ctr + blockIdx.x, 1u);
    s_last = ((old + 1u) % (unsigned)p.red.n) == 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence_system();
#pragma unroll 2
  for (int mt = 0; mt < 8; ++mt) {
    const int m = m0 + wm * 64 + mt * 8 + g;
    if (m >= p.M) continue;
    for (int nt = 0; nt < 4; ++nt) {
      for (int j = 0; j < 2; ++j) {
        const int n = n0 + wn * 32 + nt * 8 + 2 * t + j;
        if (n >= p.N) continue;
        const int64_t o = p.red.off + (int64_t)m + (int64_t)n * p.ldc;
        double a = __ldcg(reinterpret_cast<const double*>(p.red.stage[0]) + o);
        for (int r = 1; r < p.red.n; ++r) a += __ldcg(reinterpret_cast<const double*>(p.red.stage[r]) + o);
        for (int r = 0; r < p.red.n; ++r) reinterpret_cast<double*>(p.red.out[r])[o] = a;
      }
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < p.red.n) atomicAdd_system(p.red.done[threadIdx.x], 1u);
}

}  // namespace chase
