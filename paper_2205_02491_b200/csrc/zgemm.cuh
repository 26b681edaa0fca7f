// Complex-double GEMM with the fused Chebyshev-step epilogue -- the filter's hot kernel.
//
//   C[M x N] = alpha * op(A) * B  -  alpha*gamma * S[shift rows]  +  beta * C
//
// op(A) = A (A column-major M x K, "forward" W = H V, Eq. w=av) or
//       = A^H (A column-major K x M, "backward" V = H^H W, Eq. v=aw + the A^T trick).
// B column-major K x N.  The shift term realises A-hat = A - gamma I on the
// rows where the global diagonal crosses this shard (intersection I_ij), without touching H.
// beta * C is the three-term recurrence's beta_i V_{i-1} term written in place
// ("W = A V + W", Fig. 1a).
//
// B200 design: FP64 tensor cores are only reachable through the warp-level DMMA.8x8x4
// (mma.sync m8n8k4 f64); tcgen05 has no f64 kind.  Complex arithmetic is mapped onto real MMAs
// (4M: Cr += Ar Br - Ai Bi, Ci += Ar Bi + Ai Br).  Operand tiles are staged by TMA
// (cp.async.bulk.tensor, SWIZZLE_128B) into a 4-stage mbarrier ring filled by one producer warp;
// 8 consumer warps each own a 32x32 complex accumulator tile in registers.  One 16-byte LDS
// delivers the (re, im) pair of one element, and the k-index permutation k = 8*kc + 2*t + s
// (t = lane%4) makes every fragment read bank-conflict free under the 128-B swizzle.
#pragma once
#include "common.cuh"
#include "tma.cuh"
#include "zgemm.h"

namespace chase {

struct ZgemmParams {
  int M, N, K;
  double alpha, beta, gamma;
  // shift term: rows m in [shift_lo, shift_hi) get  -alpha*gamma*S[m + shift_off, n]
  const double2* S;
  int64_t lds;
  int shift_lo, shift_hi;
  int64_t shift_off;
  double2* C;
  int64_t ldc;
  int a_chunked;        // forward A loaded by one 3-D TMA box (M % 8 == 0) instead of BM/8 2-D boxes
  int upper_only;       // skip output tiles strictly below the diagonal
  int b_upper;          // B is upper triangular: k-loop stops at the tile's last column
  PeerRed red;          // f1: fused all-reduce over peer memory (red.n <= 1: off)
  int group_m;          // 3M kernel tile rasterisation: M tiles per group (0: default 12)
};

namespace zg {
constexpr int BK = 16;      // complex k per stage (two 8-element swizzle chunks)
constexpr int STAGES = 4;

template <int BM, int BN>
struct Cfg {
  static constexpr int WM = BM / 32, WN = BN / 32, NWARPS = WM * WN;
  static constexpr int THREADS = NWARPS * 32;
  static constexpr uint32_t A_BYTES = BM * BK * 16;
  static constexpr uint32_t B_BYTES = BK * BN * 16;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 2 * STAGES * 8 + 1024;
};

// Not volatile: the compiler may interleave the DMMAs of one k4 step with the fragment loads of
// the next (software pipelining).  The shared-memory load carries a "memory" clobber so it stays
// ordered after the mbarrier wait that publishes the TMA data.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 lds128(uint32_t addr) {
  double2 v;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}
}  // namespace zg

template <int BM, int BN, bool CONJ_A>
__global__ void __launch_bounds__(zg::Cfg<BM, BN>::THREADS, 1)
    zgemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, ZgemmParams p) {
  using C_ = zg::Cfg<BM, BN>;
  constexpr int BK = zg::BK, STAGES = zg::STAGES;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C_::STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grouped rasterisation: a wave of 148 CTAs covers ~8 m-tiles x ~18 n-tiles, so concurrently
  // resident CTAs share both A row-panels and B column-panels in L2
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
  // structure flags: upper_only skips tiles strictly below the diagonal (Hermitian results whose
  // lower triangle is never read, e.g. Gram matrices for Cholesky); b_upper truncates the k-loop
  // at the tile's last column when B is upper triangular (V R^{-1}).
  if (p.upper_only && m0 >= n0 + BN) return;
  const int KT = p.b_upper ? (min(p.K, n0 + BN) + BK - 1) / BK : (p.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, C_::NWARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // Thread 0 doubles as the TMA producer (a 9th warp would cap registers at 168/thread, since
  // registers are split per SM sub-partition).  Tile kt lands in slot kt % STAGES.
  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    unsigned char* sa = smem + s * C_::STAGE_BYTES;
    unsigned char* sb = sa + C_::A_BYTES;
    mbar_arrive_expect_tx(full + s, C_::STAGE_BYTES);
    const int k0 = kt * BK;
    if constexpr (!CONJ_A) {
      // A col-major M x K -> smem [BM/8][BK][8 m]: one 3-D box, or one 2-D box per 8-row chunk
      if (p.a_chunked) {
        tma_load_3d(sa, &tmA, 0, k0, m0 / 8, full + s);
      } else {
#pragma unroll
        for (int c = 0; c < BM / 8; ++c)
          tma_load_2d(sa + c * (BK * 128), &tmA, 2 * (m0 + 8 * c), k0, full + s);
      }
    } else {
      // A col-major K x M, op = A^H -> smem [BK/8][BM][8 k]
#pragma unroll
      for (int kc = 0; kc < BK / 8; ++kc)
        tma_load_2d(sa + kc * (BM * 128), &tmA, 2 * (k0 + 8 * kc), m0, full + s);
    }
#pragma unroll
    for (int kc = 0; kc < BK / 8; ++kc)
      tma_load_2d(sb + kc * (BN * 128), &tmB, 2 * (k0 + 8 * kc), n0, full + s);
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int kt = 0; kt < STAGES - 1 && kt < KT; ++kt) issue(kt);
  }

  // -------------------------------------------------------------------- MMA consumer warps
  const int wm = warp / C_::WN, wn = warp % C_::WN;
  const int g = lane >> 2, t = lane & 3;
  double cr[4][4][2], ci[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

  const uint32_t smem_base = smem_u32(smem);
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    if (threadIdx.x == 0 && kt + STAGES - 1 < KT) {
      // refill the slot last used by tile kt-1 once every warp has released it
      if (kt >= 1) mbar_wait(empty + (kt - 1) % STAGES, ((kt - 1) / STAGES) & 1);
      issue(kt + STAGES - 1);
    }
    mbar_wait(full + s, (kt / STAGES) & 1);
    const uint32_t sa = smem_base + s * C_::STAGE_BYTES;
    const uint32_t sb = sa + C_::A_BYTES;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int kc = ks >> 1;
      const int kk = 2 * t + (ks & 1);           // k within the 8-element chunk
      double2 a[4], b[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        if constexpr (!CONJ_A) {
          const int row = (wm * 4 + mt) * BK + kc * 8 + kk;       // [m-chunk][k] rows of 128 B
          a[mt] = zg::lds128(sa + row * 128 + ((g ^ (row & 7)) << 4));
        } else {
          const int row = kc * BM + wm * 32 + mt * 8 + g;         // [k-chunk][m] rows of 128 B
          a[mt] = zg::lds128(sa + row * 128 + ((kk ^ g) << 4));
          a[mt].y = -a[mt].y;                                      // conj
        }
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int row = kc * BN + wn * 32 + nt * 8 + g;
        b[nt] = zg::lds128(sb + row * 128 + ((kk ^ g) << 4));
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const double nbi = -b[nt].y;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          zg::dmma(cr[mt][nt][0], cr[mt][nt][1], a[mt].x, b[nt].x);
          zg::dmma(ci[mt][nt][0], ci[mt][nt][1], a[mt].x, b[nt].y);
          zg::dmma(cr[mt][nt][0], cr[mt][nt][1], a[mt].y, nbi);
          zg::dmma(ci[mt][nt][0], ci[mt][nt][1], a[mt].y, b[nt].x);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }

  // ------------------------------------------------------------------ fused epilogue
  const double ag = p.alpha * p.gamma;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int m = m0 + wm * 32 + mt * 8 + g;
    if (m >= p.M) continue;
    const bool shifted = (m >= p.shift_lo) && (m < p.shift_hi);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = n0 + wn * 32 + nt * 8 + 2 * t + j;
        if (n >= p.N) continue;
        double vr = p.alpha * cr[mt][nt][j];
        double vi = p.alpha * ci[mt][nt][j];
        if (shifted) {
          const double2 sv = p.S[(int64_t)m + p.shift_off + (int64_t)n * p.lds];
          vr -= ag * sv.x;
          vi -= ag * sv.y;
        }
        double2* cp = p.C + (int64_t)m + (int64_t)n * p.ldc;
        if (p.beta != 0.0) {
          const double2 cv = *cp;
          vr += p.beta * cv.x;
          vi += p.beta * cv.y;
        }
        *cp = make_double2(vr, vi);
      }
    }
  }
}

}  // namespace chase
