// Complex-double GEMM with the fused Chebyshev-step epilogue, 3M (Gauss) variant.
//
// Same contract as zgemm.cuh (C = alpha op(A) B - alpha gamma S[shift rows] + beta C), but the
// complex product is formed from three real products per k (Karatsuba/Gauss "3M", Higham §23.2.4):
//   T1 = Ar Br,  T2 = Ai Bi,  T3 = (Ar + Ai)(Br + Bi);   Cr = T1 - T2,  Ci = T3 - T1 - T2.
// 3 DMMA.8x8x4 per complex 8x8x4 step instead of 4 -> 4/3 of the FP64 tensor peak in complex
// flops.  3M is normwise backward stable (|error| <= c u ||A|| ||B||) but not componentwise; the
// parity tests hold it to the same 1e-13 relative Frobenius bar as 4M.
//
// Tiling: warps of 32 (m) x 16 (n) complex with three accumulator sets (96 registers per thread);
// default CTA 96 x 64 with 12 warps (3 per SM sub-partition) and a 5-stage TMA ring of 40 KB stages
// (SWIZZLE_128B, same conflict-free fragment addressing and k-permutation as zgemm.cuh).
#pragma once
#include "common.cuh"
#include "tma.cuh"
#include "zgemm.cuh"

namespace chase {

template <int WM_, int WN_, int STAGES_>
struct Z3Cfg {
  static constexpr int WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int BM = 32 * WM, BN = 16 * WN, BK = 16;
  static constexpr int NWARPS = WM * WN, THREADS = NWARPS * 32;
  static constexpr uint32_t A_BYTES = BM * BK * 16, B_BYTES = BK * BN * 16, STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 2 * STAGES * 8 + 1024;
};
// default: 12 warps (3 per SM sub-partition) on a 96 x 64 CTA tile, 5 stages of 40 KB
using Z3Default = Z3Cfg<3, 4, 5>;

template <class CFG, bool CONJ_A>
__global__ void __launch_bounds__(CFG::THREADS, 1)
    zgemm3m_dmma_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, ZgemmParams p) {
  constexpr int WM = CFG::WM, WN = CFG::WN, STAGES = CFG::STAGES, BM = CFG::BM, BN = CFG::BN, BK = CFG::BK;
  constexpr int NWARPS = CFG::NWARPS;
  constexpr uint32_t A_BYTES = CFG::A_BYTES, STAGE_BYTES = CFG::STAGE_BYTES;
  (void)WM;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = (p.N + BN - 1) / BN;
  const int tiles_m = (p.M + BM - 1) / BM;
  const int GROUP_M = p.group_m > 0 ? p.group_m : 12;
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
      mbar_init(empty + s, NWARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    unsigned char* sa = smem + s * STAGE_BYTES;
    unsigned char* sb = sa + A_BYTES;
    mbar_arrive_expect_tx(full + s, STAGE_BYTES);
    const int k0 = kt * BK;
    if constexpr (!CONJ_A) {
      if (p.a_chunked) {
        tma_load_3d(sa, &tmA, 0, k0, m0 / 8, full + s);
      } else {
#pragma unroll
        for (int c = 0; c < BM / 8; ++c)
          tma_load_2d(sa + c * (BK * 128), &tmA, 2 * (m0 + 8 * c), k0, full + s);
      }
    } else {
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

  const int wm = warp / WN, wn = warp % WN;
  const int g = lane >> 2, t = lane & 3;
  double t1[4][2][2], t2[4][2][2], t3[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) t1[i][j][e] = t2[i][j][e] = t3[i][j][e] = 0.0;

  const uint32_t smem_base = smem_u32(smem);
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    if (threadIdx.x == 0 && kt + STAGES - 1 < KT) {
      if (kt >= 1) mbar_wait(empty + (kt - 1) % STAGES, ((kt - 1) / STAGES) & 1);
      issue(kt + STAGES - 1);
    }
    mbar_wait(full + s, (kt / STAGES) & 1);
    const uint32_t sa = smem_base + s * STAGE_BYTES;
    const uint32_t sb = sa + A_BYTES;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int kc = ks >> 1;
      const int kk = 2 * t + (ks & 1);
      double2 a[4], b[2];
      double as[4], bs[2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        if constexpr (!CONJ_A) {
          const int row = (wm * 4 + mt) * BK + kc * 8 + kk;
          a[mt] = zg::lds128(sa + row * 128 + ((g ^ (row & 7)) << 4));
        } else {
          const int row = kc * BM + wm * 32 + mt * 8 + g;
          a[mt] = zg::lds128(sa + row * 128 + ((kk ^ g) << 4));
          a[mt].y = -a[mt].y;
        }
        as[mt] = a[mt].x + a[mt].y;
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int row = kc * BN + wn * 16 + nt * 8 + g;
        b[nt] = zg::lds128(sb + row * 128 + ((kk ^ g) << 4));
        bs[nt] = b[nt].x + b[nt].y;
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          zg::dmma(t1[mt][nt][0], t1[mt][nt][1], a[mt].x, b[nt].x);
          zg::dmma(t2[mt][nt][0], t2[mt][nt][1], a[mt].y, b[nt].y);
          zg::dmma(t3[mt][nt][0], t3[mt][nt][1], as[mt], bs[nt]);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }

  const double ag = p.alpha * p.gamma;
  const bool fused = p.red.n > 1;
  // without f1 the result goes to C; with f1 this rank's partial goes to its staging buffer
  double2* dst = fused ? p.red.stage[p.red.me] + p.red.off : p.C;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int m = m0 + wm * 32 + mt * 8 + g;
    if (m >= p.M) continue;
    const bool shifted = (m >= p.shift_lo) && (m < p.shift_hi);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = n0 + wn * 16 + nt * 8 + 2 * t + j;
        if (n >= p.N) continue;
        const double cr = t1[mt][nt][j] - t2[mt][nt][j];
        const double ci = t3[mt][nt][j] - t1[mt][nt][j] - t2[mt][nt][j];
        double vr = p.alpha * cr;
        double vi = p.alpha * ci;
        if (shifted) {
          const double2 sv = p.S[(int64_t)m + p.shift_off + (int64_t)n * p.lds];
          vr -= ag * sv.x;
          vi -= ag * sv.y;
        }
        const int64_t o = (int64_t)m + (int64_t)n * p.ldc;
        if (p.beta != 0.0) {
          const double2 cv = p.C[o];
          vr += p.beta * cv.x;
          vi += p.beta * cv.y;
        }
        dst[o] = make_double2(vr, vi);
      }
    }
  }
  if (!fused) return;
  // ---- f1: arrive on this tile's counter; the last of the n ranks reduces and broadcasts
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
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int m = m0 + wm * 32 + mt * 8 + g;
    if (m >= p.M) continue;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = n0 + wn * 16 + nt * 8 + 2 * t + j;
        if (n >= p.N) continue;
        const int64_t o = p.red.off + (int64_t)m + (int64_t)n * p.ldc;
        double2 acc = __ldcg(p.red.stage[0] + o);                  // comm-rank order: same bits everywhere
        for (int r = 1; r < p.red.n; ++r) {
          const double2 v = __ldcg(p.red.stage[r] + o);
          acc.x += v.x;
          acc.y += v.y;
        }
        for (int r = 0; r < p.red.n; ++r) p.red.out[r][o] = acc;
      }
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < p.red.n) atomicAdd_system(p.red.done[threadIdx.x], 1u);
}

}  // namespace chase
