// f4 research branch: the complex-double filter step with its
// FP64 products emulated on the INT8 tensor cores (tcgen05.mma kind::i8) by the Ozaki scheme
// (error-free splitting into int8 slices, exact int32 products, FP64 recombination).
//
// Arithmetic.  A complex product C = A B runs as Gauss's 3M on real matrices, T1 = Ar Br,
// T2 = Ai Bi, T3 = (Ar + Ai)(Br + Bi); Re C = T1 - T2, Im C = T3 - T1 - T2 (as in zgemm3m.cuh).
// Each real product P = X Y is emulated: every row m of X is scaled by 2^-e_m (e_m = frexp
// exponent of the row's max |x|, so |x| 2^-e_m < 1) and cut into S truncated 7-bit slices,
//   x 2^-e_m = sum_{s=1..S} a_s 2^-7s + r,   a_s in [-127, 127] (int8),  |r| < 2^-7S,
// every column n of Y likewise (exponent f_n, slices b_t).  Then
//   P_mn = 2^(e_m + f_n) sum_{s+t <= S+1} 2^-7(s+t) (A_s B_t)_mn  + O(S 2^-7S) |X||Y| (normwise),
// the (A_s B_t) are exact int32 tensor-core products, and terms of equal d = s + t share one
// int32 accumulator (up to floor((2^31 - 1) / (127^2 K)) products per accumulator, so the sum is
// exact).  With S = 7 the truncation error is ~2^-49 |X||Y| per entry, below the FP64 step bar
// of 1e-13 by two orders of magnitude.
//
// Data.  The H shard is equilibrated (H_P = D_r Hhat_P D_c, power-of-two row and column scalings,
// diagonal excluded) and Hhat_P sliced ONCE per API call into int8 [slice][j][i] (columns of H,
// i contiguous): the backward step (A = H^H) reads it as a K-major operand, the forward step
// (A = H) as an MN-major one (tcgen05 transpose bit), and the scalings fold into the B operand
// (D_c X forward, D_r W backward) and the output rows.  Every step slices its block X (columns
// contiguous in k), TMA-loaded as 128-byte swizzled rows.
//
// Kernel (oz_gemm_kernel): persistent CTA pairs (tcgen05 cta_group::2), 256 x 256 output tiles,
// 192 threads per CTA: warp 0 TMA producer into a 6-stage ring (16 KB of A rows + 16 KB of B
// columns per CTA and stage), one elected lane of the leader's warp 1 issues 4
// tcgen05.mma.kind::i8 (M = 256, N = 256, K = 32) per stage into one of two 256-column int32
// TMEM accumulators (all slice pairs of the launch accumulate into it), warps 2-5 drain it
// (tcgen05.ld 32x32b) and add 2^-7d x acc into the FP64 accumulator of the real product while
// the next tile accumulates.  Tiles are rastered N-fastest, so concurrently running pairs share
// each A panel (the large H slices) through L2.
// The final oz_combine kernel forms the 3M combination with the exponent scalings and the fused
// step epilogue  Y = alpha (C - gamma E X) + beta Y.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <type_traits>
#include <vector>
#include "dense.h"
#include "handle.h"
#include "tma.cuh"

namespace chase {

namespace oz {
constexpr int BM = 128, BN = 256, BK = 128;            // per CTA: 128 rows; per MMA: 256 x 256; BK int8 (= bytes)
constexpr uint32_t A_BYTES = BM * BK, B_BYTES = (BN / 2) * BK;   // 16 KB of A rows, 16 KB of B columns per sub-tile
constexpr int THREADS = 192;
constexpr int MAX_PAIRS = 8;
constexpr uint32_t TCOLS = 512;                         // all of TMEM: NS = 1 two 256-col buffers, NS = 2 one 512-col
// NS = 256-column sub-tiles per pair tile (1: 256 x 256 tiles, double-buffered accumulators --
// the default; 2: 256 x 512 tiles, one accumulator: each A k block feeds two MMAs, so the TMA
// writes per MAC drop from 60 to 44 B/clk/SM and a round re-reads half as many B panels, but it
// measured 15 % slower -- the exposed drain and the 4-stage ring cost more; CHASE_OZ_NS=2)
template <int NS> struct Shape {
  static constexpr uint32_t STAGE_BYTES = A_BYTES + NS * B_BYTES;
  static constexpr int STAGES = NS == 1 ? 6 : 4;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 1024;
  static constexpr int BNT = NS * BN;                    // tile width
  static constexpr int NBUF = 2 / NS;                    // TMEM accumulator buffers
};

struct Params {
  int M, N, K;
  int npairs;
  int sa[MAX_PAIRS], tb[MAX_PAIRS];    // slice index of A and of B for every pair of the launch
  double scale;                        // 2^-7d
  double* out;                         // FP64 accumulator of the real product (M x N, ld ldo)
  int64_t ldo;
  int accumulate;                      // 0: out = scale acc; 1: out += scale acc
  int hint;                            // 1: L2 evict_first for A (streamed), evict_last for B (re-read)
  unsigned* sync;                      // round barrier counter (zeroed per launch); null = no barrier
  int amn;                             // 1: A is MN-major (slices [k][m], m contiguous: the forward step)
  int dbg;                             // experiments only (CHASE_OZ_DBG): 1 = drain without the FP64 RMW,
                                       // 2 = every k block re-loads k block 0 (no HBM streaming)
  int snake;                           // 1: odd rounds walk K backwards (B's last k windows still in L2)
  uint8_t* rout;                       // CRT mode: the product mod `modulus`, one byte per output (ld ldo)
  int modulus;
};

__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {   // K-major, SWIZZLE_128B, 8-row groups 1 KB apart
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// MN-major A (int8, SWIZZLE_128B): one 128-byte m atom (the CTA's 128 rows) per k row, 8-row
// groups 1 KB apart; one MMA (K = 32) spans 32 k rows = 4 KB (validated by
// tools/microbench/i8_mn_probe.cu: bit-exact against the CPU product)
__device__ __forceinline__ uint64_t sdesc_mn(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa0(uint32_t addr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(0));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_3d_pair(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_3d_pair_hint(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint32_t bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAITOZ:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONEOZ;\n"
      "bra LAB_WAITOZ;\n"
      "DONEOZ:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void commit_both(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}

// Persistent CTA-pair kernel (cluster of 2, tcgen05 cta_group::2): every pair walks the 256 x 256
// output tiles t = pair, pair + npair, ... (N fastest, so concurrently running pairs share A
// panels in L2).  Per tile and k block of 128, each CTA stages its 128 A rows and its half (128
// columns) of B for every slice pair of the launch; the leader's MMA warp issues 4
// tcgen05.mma.cta_group::2.kind::i8 (M = 256, N = 256, K = 32) per stage into one of two
// 256-column TMEM accumulators, so the drain of tile t overlaps the MMAs of tile t + 1.  Drain:
// 4 warps per CTA (TMEM lane quadrant = warp % 4), 16 columns at a time, 2^-7d x acc added
// into the FP64 output.
template <int NS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, Params p) {
  constexpr uint32_t STAGE_BYTES = Shape<NS>::STAGE_BYTES;
  constexpr int STAGES = Shape<NS>::STAGES, BNT = Shape<NS>::BNT, NBUF = Shape<NS>::NBUF;
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES], empty[STAGES], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int tiles_n = (p.N + BNT - 1) / BNT, tiles_m = (p.M + 2 * BM - 1) / (2 * BM);
  const int pair = blockIdx.x >> 1, npair = gridDim.x >> 1;
  const int KT = (p.K + BK - 1) / BK;
  // Static L2-aware schedule: the pairs form groups of tiles_n; group g walks the m tiles
  // g, g + ngroups, ... and pair j of the group always takes n tile j, so the tiles_n pairs that
  // read one A panel run it in lockstep and share it through L2 (a round-robin walk lets them
  // drift apart: measured 13x the A traffic at 12 n tiles).  Pairs beyond ngroups x tiles_n idle.
  const bool grouped = tiles_n <= npair;
  const int ngroups = grouped ? npair / tiles_n : 1;
  const int g = pair / tiles_n, jn = pair % tiles_n;
  const bool active = !grouped || g < ngroups;
  // tile r of this pair: (m tile, n tile); ntile() = number of tiles
  auto ntile = [&]() -> int {
    if (!active) return 0;
    if (grouped) return g < tiles_m ? (tiles_m - 1 - g) / ngroups + 1 : 0;
    const int T = tiles_n * tiles_m;
    return pair < T ? (T - 1 - pair) / npair + 1 : 0;
  };
  auto tile_mn = [&](int r, int& tmi, int& tni) {
    if (grouped) { tmi = g + r * ngroups; tni = jn; }
    else { const int t = pair + r * npair; tmi = t / tiles_n; tni = t % tiles_n; }
  };
  const int NT = ntile();

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + b, 1);
      mbar_init(acc_empty + b, 8);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tA);
      tma_prefetch_desc(&tB);
      uint64_t pol_a = 0, pol_b = 0;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_a));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_b));
      int it = 0;
      unsigned target = 0;
      for (int r = 0; r < NT; ++r) {
        if (p.sync && grouped && r > 0) {
          // Round barrier of the producers (performance only): every CTA starts loading round r
          // together, so the pairs stream the A and B k windows in step and share them through L2
          // (B, re-read by every m round, does not fit L2; without the barrier the pairs drift
          // apart over a launch -- measured 35 GB vs 13 GB of DRAM reads per launch).  The
          // results never depend on it: a CTA that waits longer than 50 ms (e.g. not all CTAs
          // resident because another kernel shares the GPU) stops synchronising and carries on.
          target += 2u * (unsigned)tiles_n * (unsigned)min(ngroups, tiles_m - r * ngroups);
          atomicAdd(p.sync, 1u);
          unsigned long long t0, t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          unsigned v;
          while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.sync) : "memory");
            if (v >= target) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 > 50000000ull) { p.sync = nullptr; break; }
          }
        }
        int tmi, tni;
        tile_mn(r, tmi, tni);
        const int m0 = tmi * 2 * BM + (int)rank * BM;
        const int nh = tni * BNT + (int)rank * (BN / 2);      // this CTA's half of sub-tile 0
        // Boustrophedon K order: every round streams all of B's k windows (B does not fit L2), so
        // odd rounds walk K backwards and start on the windows the previous round read last, which
        // L2 still holds.  The int32 sums are exact, so the order never changes a result bit.
        const bool back = p.snake && grouped && (r & 1);
        for (int kt0 = 0; kt0 < KT; ++kt0) {
          const int kt = back ? KT - 1 - kt0 : kt0;
          for (int q = 0; q < p.npairs; ++q, ++it) {
            const int s = it % STAGES;
            if (it >= STAGES) mbar_wait(empty + s, ((it / STAGES) - 1) & 1);
            const uint32_t st = smem_u32(sm + s * STAGE_BYTES);
            const uint32_t fb = mapa0(smem_u32(full + s));
            if (rank == 0) mbar_arrive_expect_tx(full + s, 2 * STAGE_BYTES);
            // A box {128, 128, 1}: K-major coordinates (k, m), MN-major (m, k)
            const int kb = (p.dbg & 2) ? 0 : kt * BK;
            const int ac0 = p.amn ? m0 : kb, ac1 = p.amn ? kb : m0;
            if (p.hint) {
              tma_3d_pair_hint(st, &tA, ac0, ac1, p.sa[q], fb, pol_a);
#pragma unroll
              for (int sub = 0; sub < NS; ++sub)
                tma_3d_pair_hint(st + A_BYTES + sub * B_BYTES, &tB, kb, nh + sub * BN, p.tb[q], fb, pol_b);
            } else {
              tma_3d_pair(st, &tA, ac0, ac1, p.sa[q], fb);
#pragma unroll
              for (int sub = 0; sub < NS; ++sub)
                tma_3d_pair(st + A_BYTES + sub * B_BYTES, &tB, kb, nh + sub * BN, p.tb[q], fb);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      uint32_t leader;
      asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(leader));
      // S32 accumulate, signed int8 A and B, both K-major, N = 256, M = 256 (pair)
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((p.amn ? 1u : 0u) << 15) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((2 * BM) >> 4) << 24);
      int it = 0, tl = 0;
      for (int r = 0; r < NT; ++r, ++tl) {
        const int b = tl % NBUF;
        if (tl >= NBUF) {
          wait_cluster(acc_empty + b, ((tl / NBUF) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint32_t td = tm + (uint32_t)b * BNT;
        for (int j = 0; j < KT * p.npairs; ++j, ++it) {
          const int s = it % STAGES;
          mbar_wait(full + s, (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (leader) {
            const uint32_t sa = smem_u32(sm + s * STAGE_BYTES), sb = sa + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 32; ++kk) {
              const uint32_t acc = (j > 0 || kk > 0) ? 1u : 0u;
              const uint64_t da = p.amn ? sdesc_mn(sa + kk * 4096) : sdesc(sa + kk * 32);
#pragma unroll
              for (int sub = 0; sub < NS; ++sub)
                asm volatile(
                    "{ .reg .pred q; setp.ne.b32 q, %4, 0; tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, q; }"
                    ::"r"(td + sub * BN), "l"(da), "l"(sdesc(sb + sub * B_BYTES + kk * 32)), "r"(idesc), "r"(acc));
            }
            commit_both(empty + s);
          }
          __syncwarp();
        }
        if (leader) commit_both(acc_full + b);
        __syncwarp();
      }
    }
  } else {
    const int quad = warp & 3;
    const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
    int tl = 0;
    for (int r = 0; r < NT; ++r, ++tl) {
      const int b = tl % NBUF;
      int tmi, tni;
      tile_mn(r, tmi, tni);
      const int row = tmi * 2 * BM + (int)rank * BM + 32 * quad + lane;
      const int n0 = tni * BNT;
      mbar_wait(acc_full + b, (tl / NBUF) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t base = tm + lane_off + (uint32_t)b * BNT;
      for (int c0 = 0; c0 < BNT; c0 += 16) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(base + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (p.rout) {
          if (row < p.M) {
            const double m = (double)p.modulus, inv_m = 1.0 / m;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int n = n0 + c0 + j;
              if (n < p.N) {
                const double a = (double)(int)r[j];            // exact int32 product
                double t = fma(-rint(a * inv_m), m, a);        // exact, |t| <= 1.5 m
                if (t < 0.0) t += m;
                if (t < 0.0) t += m;
                if (t >= m) t -= m;
                p.rout[(int64_t)row + (int64_t)n * p.ldo] = (uint8_t)(int)t;
              }
            }
          }
        } else if (row < p.M && !(p.dbg & 1)) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = n0 + c0 + j;
            if (n < p.N) {
              double* o = p.out + (int64_t)row + (int64_t)n * p.ldo;
              const double v = p.scale * (double)(int)r[j];
              *o = p.accumulate ? *o + v : v;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) {
        const uint32_t bar = mapa0(smem_u32(acc_empty + b));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(TCOLS));
}

// ------------------------------------------------------------------------------- slicing
// exponent e with 128 max 2^-e < 127.5 (so the first round-to-nearest slice stays in int8),
// 0 for an all-zero line
__device__ __forceinline__ int line_exp(double mx) {
  int e = 0;
  if (mx > 0.0) {
    frexp(mx, &e);
    if (ldexp(mx, 7 - e) >= 127.5) ++e;
  }
  return e;
}

// S round-to-nearest 7-bit slices of v (|v| 128 < 127.5): a_s = rint(r 2^7), r <- r 2^7 - a_s
// (exact in FP64).  |a_1| <= 127, |a_s| <= 64 after that; the remainder is <= 2^-7S / 2 and,
// unlike truncation, unbiased (measured: ~7x smaller product error than truncated slices).
template <int S>
__device__ __forceinline__ void cut(double v, int8_t (&a)[S]) {
#pragma unroll
  for (int s = 0; s < S; ++s) {
    v *= 128.0;
    const double t = rint(v);
    a[s] = (int8_t)(int)t;
    v -= t;
  }
}

// ---- Ozaki scheme II (CRT; option oz_crt): instead of slices, the 52-bit integer
// A' = rint(v 2^52) of every scaled value (|v| < 1) is stored as its residues modulo 16 pairwise
// coprime moduli <= 256 (symmetric, |r| <= 128); one int8 GEMM per modulus gives A'B' mod m_i
// exactly (|r_a r_b| K <= 2^14 K < 2^31 for K <= 131071), and Garner's algorithm rebuilds A'B'
// (|A'B'| <= K 2^104 < M / 2, M = prod m_i ~ 2^125) exactly before one FP64 rounding.
constexpr int NMOD = 16;
__host__ __device__ constexpr int crt_mod(int i) {
  constexpr int m[NMOD] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};
  return m[i];
}
constexpr int CRT_BITS = 52;
constexpr double CRT_SCALE = double(1LL << CRT_BITS);            // 2^52

__device__ __forceinline__ void crt_cut(double v, int8_t (&a)[NMOD]) {
  const double A = rint(v * CRT_SCALE);                    // 2^52 v, |A| < 2^52: exact integer
#pragma unroll
  for (int i = 0; i < NMOD; ++i) {
    const int mi = crt_mod(i);
    const double m = (double)mi;
    const double hi = mi == 256 ? 127.0 : 0.5 * (m - 1.0), lo = mi == 256 ? -128.0 : -hi;
    const double q = rint(A * (1.0 / m));                  // within one of A / m
    double r = fma(-q, m, A);                              // exact (|q m| < 2^53), |r| <= 1.5 m
    if (r > hi) r -= m;
    if (r < lo) r += m;
    if (r > hi) r -= m;
    a[i] = (int8_t)(int)r;
  }
}

// The NP real matrices the products run on: complex (NP = 3, Gauss's 3M): re, im, re + sg im
// (sg = -1 for the B operand of the backward step, see ozaki_step_t); real symmetric (NP = 1).
template <class T> struct Comp;
template <> struct Comp<double2> {
  static constexpr int NP = 3;
  __device__ static void get(double2 v, double sg, double (&c)[3]) {
    c[0] = v.x;
    c[1] = v.y;
    c[2] = v.x + sg * v.y;
  }
  __device__ static double2 zero() { return make_double2(0.0, 0.0); }
};
template <> struct Comp<double> {
  static constexpr int NP = 1;
  __device__ static void get(double v, double, double (&c)[1]) { c[0] = v; }
  __device__ static double zero() { return 0.0; }
};

// Lines contiguous in memory (columns of a column-major matrix): line c of `rows` values at
// X + c ld, each value k first scaled by 2^(ksg kexp[P kexp_ld + k]) if kexp is given (the
// equilibration of the shard, see ozaki_step_t).  Writes, for every real component P (Comp),
// slices out[(P S + s) * plane + c * ldk + k] and exponents e[P * lines + c].  One CTA per line.
// diag != INT_MIN: the element k = c + diag of line c lies on the global diagonal of H; it is left
// out of the slices (zero) and added exactly in FP64 by oz_combine (diagonal split: the dominant
// diagonal of a Hermitian H would otherwise set the line's exponent and cost the off-diagonal
// entries their low bits).
template <int S, class T>
__global__ void __launch_bounds__(256) oz_slice_lines(const T* X, int64_t ld, int rows, int lines, int sg3,
                                                      int diag, const int* kexp, int kexp_ld, int ksg, int8_t* out,
                                                      int64_t ldk, int64_t plane, int* e) {
  constexpr int NP = Comp<T>::NP;
  const int c = blockIdx.x;
  const T* x = X + (int64_t)c * ld;
  const double sg = sg3 < 0 ? -1.0 : 1.0;
  const int kd = diag == INT_MIN ? -1 : c + diag;
  auto load = [&](int k, double (&v)[NP]) {
    Comp<T>::get(x[k], sg, v);
    if (kexp) {
#pragma unroll
      for (int P = 0; P < NP; ++P) v[P] = ldexp(v[P], ksg * kexp[P * kexp_ld + k]);
    }
  };
  double mx[NP];
#pragma unroll
  for (int P = 0; P < NP; ++P) mx[P] = 0.0;
  for (int k = threadIdx.x; k < rows; k += 256) {
    if (k == kd) continue;
    double v[NP];
    load(k, v);
#pragma unroll
    for (int P = 0; P < NP; ++P) mx[P] = fmax(mx[P], fabs(v[P]));
  }
  __shared__ double sm[NP][8];
#pragma unroll
  for (int P = 0; P < NP; ++P) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx[P] = fmax(mx[P], __shfl_xor_sync(0xffffffffu, mx[P], o));
    if ((threadIdx.x & 31) == 0) sm[P][threadIdx.x >> 5] = mx[P];
  }
  __syncthreads();
  __shared__ int ex[NP];
  if (threadIdx.x < NP) {
    double m = 0.0;
    for (int w = 0; w < 8; ++w) m = fmax(m, sm[threadIdx.x][w]);
    ex[threadIdx.x] = line_exp(m);
    e[threadIdx.x * lines + c] = ex[threadIdx.x];
  }
  __syncthreads();
  double sc[NP];
#pragma unroll
  for (int P = 0; P < NP; ++P) sc[P] = ldexp(1.0, -ex[P]);
  if constexpr (S == NMOD) {
    // scheme II: the 4 values of a thread loaded once, then one real component at a time (16
    // residue words live at once instead of 48: occupancy)
    for (int k4 = threadIdx.x * 4; k4 < (int)ldk; k4 += 256 * 4) {
      double vv[4][NP];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int k = k4 + kk;
        if (k < rows && k != kd) {
          load(k, vv[kk]);
        } else {
#pragma unroll
          for (int P = 0; P < NP; ++P) vv[kk][P] = 0.0;
        }
      }
      int8_t* o = out + (int64_t)c * ldk + k4;
#pragma unroll
      for (int P = 0; P < NP; ++P) {
        uint32_t packed[NMOD];
#pragma unroll
        for (int i = 0; i < NMOD; ++i) packed[i] = 0;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          int8_t a[NMOD];
          crt_cut(vv[kk][P] * sc[P], a);
#pragma unroll
          for (int i = 0; i < NMOD; ++i) packed[i] |= (uint32_t)(uint8_t)a[i] << (8 * kk);
        }
#pragma unroll
        for (int i = 0; i < NMOD; ++i) *reinterpret_cast<uint32_t*>(o + (int64_t)(P * NMOD + i) * plane) = packed[i];
      }
    }
    return;
  }
  // 4 consecutive k per thread: one 4-byte store per slice (ldk % 128 == 0)
  for (int k4 = threadIdx.x * 4; k4 < (int)ldk; k4 += 256 * 4) {
    uint32_t packed[NP][S];
#pragma unroll
    for (int P = 0; P < NP; ++P)
#pragma unroll
      for (int s = 0; s < S; ++s) packed[P][s] = 0;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int k = k4 + kk;
      double v[NP];
      if (k < rows && k != kd) {
        load(k, v);
      } else {
#pragma unroll
        for (int P = 0; P < NP; ++P) v[P] = 0.0;
      }
      int8_t a[NP][S];
#pragma unroll
      for (int P = 0; P < NP; ++P) {
        if constexpr (S == NMOD) crt_cut(v[P] * sc[P], a[P]);   // scheme II: residues
        else cut<S>(v[P] * sc[P], a[P]);
      }
#pragma unroll
      for (int P = 0; P < NP; ++P)
#pragma unroll
        for (int s = 0; s < S; ++s) packed[P][s] |= (uint32_t)(uint8_t)a[P][s] << (8 * kk);
    }
    int8_t* o = out + (int64_t)c * ldk + k4;
#pragma unroll
    for (int P = 0; P < NP; ++P)
#pragma unroll
      for (int s = 0; s < S; ++s) *reinterpret_cast<uint32_t*>(o + (int64_t)(P * S + s) * plane) = packed[P][s];
  }
}

// Row maxima (rows of H for the forward A operand) per real component, as order-preserving bit
// patterns of non-negative doubles via atomicMax.
template <class T>
__global__ void oz_row_max(const T* H, int64_t ld, int rows, int cols, int diag, unsigned long long* mx) {
  constexpr int NP = Comp<T>::NP;
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= rows) return;
  const int c0 = blockIdx.y * 256, c1 = min(cols, c0 + 256);
  double m[NP];
#pragma unroll
  for (int P = 0; P < NP; ++P) m[P] = 0.0;
  for (int j = c0; j < c1; ++j) {
    if (j == i + diag) continue;                      // diagonal split (see oz_slice_lines)
    double v[NP];
    Comp<T>::get(H[i + (int64_t)j * ld], 1.0, v);
#pragma unroll
    for (int P = 0; P < NP; ++P) m[P] = fmax(m[P], fabs(v[P]));
  }
#pragma unroll
  for (int P = 0; P < NP; ++P) atomicMax(mx + P * rows + i, (unsigned long long)__double_as_longlong(m[P]));
}

// row exponents of the equilibration: r[P][i] from the row maxima (line_exp)
template <class T>
__global__ void oz_row_exp(const unsigned long long* mx, int rows, int* r) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= rows) return;
#pragma unroll
  for (int P = 0; P < Comp<T>::NP; ++P) r[P * rows + i] = line_exp(__longlong_as_double((long long)mx[P * rows + i]));
}

// Y = alpha (C - gamma E X) + beta Y from the FP64 real products with their exponents (complex:
// the three products of 3M, Re C = T1 - T2, Im C = T3 - T1 - T2; real: C = T1).  Rows m in
// [dlo, dhi) carry the diagonal split and the shift: + alpha (hdiag[m] - gamma) X[m + doff].
__device__ __forceinline__ double2 c_fma(double a, double2 v, double2 acc) {
  return make_double2(acc.x + a * v.x, acc.y + a * v.y);
}
template <class T>
__global__ void oz_combine(const double* T_, int64_t ldt, int64_t tplane, const int* eA, int M, const int* fB, int N,
                           T* Y, int64_t ldy, double alpha, double beta, int beta_on, const T* X, int64_t ldx,
                           const double2* hdiag, int dlo, int dhi, int64_t doff, double gamma, int dir) {
  const int64_t total = (int64_t)M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(idx % M), n = (int)(idx / M);
    const int64_t o = (int64_t)m + (int64_t)n * ldt;
    T* y = Y + (int64_t)m + (int64_t)n * ldy;
    const double t1 = ldexp(T_[o], eA[m] + fB[n]);
    if constexpr (Comp<T>::NP == 3) {
      const double t2 = ldexp(T_[tplane + o], eA[M + m] + fB[N + n]);
      const double t3 = ldexp(T_[2 * tplane + o], eA[2 * M + m] + fB[2 * N + n]);
      // forward (H X): Re = T1 - T2, Im = T3 - T1 - T2 with T3 = (Hr + Hi)(Xr + Xi);
      // backward (H^H W): Re = T1 + T2, Im = T1 - T2 - T3 with T3 = (Hr + Hi)(Wr - Wi)
      double re, im;
      if (dir == 0) { re = alpha * (t1 - t2); im = alpha * (t3 - t1 - t2); }
      else { re = alpha * (t1 + t2); im = alpha * (t1 - t2 - t3); }
      if (m >= dlo && m < dhi) {
        const double2 x = X[(int64_t)m + doff + (int64_t)n * ldx];
        const double2 hd = hdiag[m];
        const double dr = hd.x - gamma;
        re += alpha * (dr * x.x - hd.y * x.y);
        im += alpha * (dr * x.y + hd.y * x.x);
      }
      if (beta_on) {
        const double2 yo = *y;
        re += beta * yo.x;
        im += beta * yo.y;
      }
      *y = make_double2(re, im);
    } else {
      double v = alpha * t1;
      if (m >= dlo && m < dhi) v += alpha * (hdiag[m].x - gamma) * X[(int64_t)m + doff + (int64_t)n * ldx];
      if (beta_on) v += beta * *y;
      *y = v;
    }
  }
}

// Scheme II reconstruction: the NMOD residues of one real product (byte planes of M x N, ld M,
// written by the GEMM drain) -> Garner's mixed-radix digits (balanced: the representation of
// A'B' in (-M/2, M/2), exact) -> A'B' by Horner in 64/128-bit integers -> FP64 ->
// times 2^-104 into T (ld ldt), where oz_combine picks it up like a slice-scheme accumulator.
__host__ __device__ constexpr int inv_mod(int a, int m) {   // a^-1 mod m (gcd(a, m) = 1)
  int t = 0, nt = 1, r = m, nr = a % m;
  while (nr != 0) {
    const int qq = r / nr;
    int tmp = t - qq * nt; t = nt; nt = tmp;
    tmp = r - qq * nr; r = nr; nr = tmp;
  }
  return t < 0 ? t + m : t;
}
__host__ __device__ constexpr int pmod(int i, int j) {      // (m_0 ... m_{i-1}) mod m_j
  int p = 1;
  for (int k = 0; k < i; ++k) p = p * (crt_mod(k) % crt_mod(j)) % crt_mod(j);
  return p;
}
// Garner digit J: v_J = (c_J - sum_{i<J} v_i P_i) P_J^-1 mod m_J (balanced), where
// R[J] = sum_{i<J} v_i (P_i mod m_J) is accumulated as the digits appear (|R| < 2^19).
template <int J, int K>
struct CrtUpd {
  __device__ __forceinline__ static void run(int vj, int (&R)[NMOD]) {
    constexpr int pm = pmod(J, K);
    R[K] += vj * pm;
    CrtUpd<J, K + 1>::run(vj, R);
  }
};
template <int J>
struct CrtUpd<J, NMOD> {
  __device__ __forceinline__ static void run(int, int (&)[NMOD]) {}
};
template <int J>
struct CrtDig {
  __device__ __forceinline__ static void run(const uint8_t* c, int64_t iplane, int64_t idx, int (&v)[NMOD],
                                             int (&R)[NMOD]) {
    constexpr int mj = crt_mod(J);
    constexpr int invp = inv_mod(pmod(J, J), mj);
    constexpr int hi = mj == 256 ? 127 : (mj - 1) / 2;
    int t = ((int)c[(int64_t)J * iplane + idx] - R[J]) % mj;
    if (t < 0) t += mj;
    t = (t * invp) % mj;
    const int vj = t > hi ? t - mj : t;
    v[J] = vj;
    CrtUpd<J, J + 1>::run(vj, R);
    CrtDig<J + 1>::run(c, iplane, idx, v, R);
  }
};
template <>
struct CrtDig<NMOD> {
  __device__ __forceinline__ static void run(const uint8_t*, int64_t, int64_t, int (&)[NMOD], int (&)[NMOD]) {}
};

__global__ void __launch_bounds__(256) oz_crt(const uint8_t* C, int64_t iplane, int M, int N, double* T, int64_t ldt) {
  const int64_t total = (int64_t)M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    int v[NMOD], R[NMOD];
#pragma unroll
    for (int j = 0; j < NMOD; ++j) R[j] = 0;
    CrtDig<0>::run(C, iplane, idx, v, R);
    // Horner in exact integers (|A'B'| < 2^124): the top 7 digits in 64 bits (|x| < 2^62), the
    // rest in 128; then FP64 as hi 2^64 + lo (exact whenever A'B' is representable, else within
    // one ulp -- the 128-bit software conversion costs several times more)
    long long x64 = v[NMOD - 1];
#pragma unroll
    for (int j = NMOD - 2; j >= NMOD - 7; --j) x64 = x64 * crt_mod(j) + v[j];
    __int128 x = x64;
#pragma unroll
    for (int j = NMOD - 8; j >= 0; --j) x = x * crt_mod(j) + v[j];
    const bool neg = x < 0;
    const unsigned __int128 ax = neg ? (unsigned __int128)(-x) : (unsigned __int128)x;   // (on the
    const unsigned long long xh = (unsigned long long)(ax >> 64);                       // magnitude:
    const unsigned long long xl = (unsigned long long)ax;                               // lo <= 53 bits
    const double xa = fma((double)xh, 18446744073709551616.0, (double)xl);              // when exact)
    const double xd = neg ? -xa : xa;
    const int m = (int)(idx % M), n = (int)(idx / M);
    T[(int64_t)m + (int64_t)n * ldt] = xd * (1.0 / (CRT_SCALE * CRT_SCALE));   // 2^-104
  }
}

// the diagonal element of output row m (forward: H[m][m + off]; backward: conj(H[m - off][m])),
// zero where row m does not cross the global diagonal (off = r0 - c0)
__device__ __forceinline__ double2 as_c(double2 v) { return v; }
__device__ __forceinline__ double2 as_c(double v) { return make_double2(v, 0.0); }
template <class T>
__global__ void oz_diag(const T* H, int64_t ld, int p, int q, int dir, int off, double2* d) {
  const int m = blockIdx.x * 256 + threadIdx.x;
  const int lines = dir == 0 ? p : q;
  if (m >= lines) return;
  double2 v = make_double2(0.0, 0.0);
  if (dir == 0) {
    const int j = m + off;
    if (j >= 0 && j < q) v = as_c(H[m + (int64_t)j * ld]);
  } else {
    const int i = m - off;
    if (i >= 0 && i < p) { v = as_c(H[i + (int64_t)m * ld]); v.y = -v.y; }
  }
  d[m] = v;
}

// 3-D int8 tensor map over [slice][line][ldk] (dims {K, lines, slices}), box {128, box_lines, 1}
void make_slice_tmap(CUtensorMap* map, const int8_t* base, int64_t K, int64_t lines, int64_t ldk, int slices,
                     int box_lines) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    CHASE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)lines, (cuuint64_t)slices};
  cuuint64_t strides[2] = {(cuuint64_t)ldk, (cuuint64_t)(ldk * lines)};
  cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_lines, 1};
  cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (ozaki slices) failed: " + std::to_string((int)r));
}

inline int64_t ldk_of(int64_t K) { return (K + 127) / 128 * 128; }   // 16-B TMA strides, whole k tiles
}  // namespace oz

// ------------------------------------------------------------------------------------ host
using OzShard = chase_handle::OzShard;    // the shard's slice set (cached on the handle within one API call)

static int oz_slices_opt(chase_handle* h) {      // planes per real component: slices, or NMOD residues
  return h->opt.oz_crt ? oz::NMOD : std::min(8, std::max(0, h->opt.fp64_emulation));
}

template <int S, class T>
static void slice_lines(const T* X, int64_t ld, int rows, int lines, int sg3, int diag, const int* kexp, int kexp_ld,
                        int ksg, int8_t* out, int64_t ldk, int64_t plane, int* e, cudaStream_t st) {
  if (lines <= 0) return;
  oz::oz_slice_lines<S, T><<<lines, 256, 0, st>>>(X, ld, rows, lines, sg3, diag, kexp, kexp_ld, ksg, out, ldk, plane,
                                                  e);
  CHASE_CHECK_LAUNCH();
}

template <class F>
static void with_S(int S, F&& f) {
  switch (S) {
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 5: f(std::integral_constant<int, 5>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    case 7: f(std::integral_constant<int, 7>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    case oz::NMOD: f(std::integral_constant<int, oz::NMOD>{}); break;
    default: throw UsageError("fp64_emulation: slices must be 3..8");
  }
}

// The shard's slice set, shared by both step directions (equilibrated Ozaki splitting): per real
// component P, row exponents r[P][i] (row maxima of |H_P|, diagonal excluded) and column
// exponents c[P][j] (column maxima of |H_P| 2^-r_i) give H_P = D_r Hhat_P D_c with
// 128 |hhat| < 127.5 in every row and column; Hhat_P is cut into S slices stored [j][i] (i
// contiguous), which the backward step reads as a K-major operand (A = H^H: row j, k = i) and the
// forward step as an MN-major one (A = H: m = i, k = j).  21 B per complex element in all (the
// round-1 design kept one set per direction: 42 B).  The diagonal of the split is kept per
// direction (forward: H[m][m + off]; backward: conj(H[m - off][m])).
// Slices of a stored p x q matrix (column-major, ld) into z; split = true takes the global
// diagonal out (local (i, i + off), off = r0 - c0) and records it for the combine.
template <class T>
static void oz_slice_matrix(chase_handle* h, OzShard& z, const void* H, int64_t ldh, int64_t p, int64_t q, bool split,
                            int64_t off) {
  constexpr int NP = oz::Comp<T>::NP;
  const int S = oz_slices_opt(h);
  const int64_t ldk = oz::ldk_of(p);
  if (S == oz::NMOD) {
    // test hook: a residue set larger than CHASE_OZ_CRT_MAXBYTES behaves as if it did not fit
    const char* cap_e = std::getenv("CHASE_OZ_CRT_MAXBYTES");
    const double cap = cap_e ? std::atof(cap_e) : 0.0;
    if (cap > 0.0 && (double)NP * S * q * ldk > cap) throw std::bad_alloc();
  }
  z.slices.alloc((size_t)NP * S * q * ldk);
  // exps: r [NP][p] | c [NP][q] | row maxima (u64) [NP][p]
  const size_t ri = (size_t)NP * p, ci = (size_t)NP * q;
  z.exps.alloc(sizeof(int) * (ri + ci) + 16 + sizeof(unsigned long long) * ri);
  int* r = z.exps.as<int>();
  int* c = r + ri;
  unsigned long long* mx = reinterpret_cast<unsigned long long*>(z.exps.as<char>() + ((sizeof(int) * (ri + ci) + 15) & ~size_t(15)));
  const T* Hz = reinterpret_cast<const T*>(H);
  // diagonal split: the global diagonal of H sits at local (i, i + off) = (j - off, j)
  const int row_diag = split ? (int)off : (1 << 30), col_diag = split ? (int)-off : INT_MIN;
  CHASE_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned long long) * ri, h->stream));
  oz::oz_row_max<T><<<dim3(ceil_div(p, 256), ceil_div(q, 256)), 256, 0, h->stream>>>(Hz, ldh, (int)p, (int)q,
                                                                                     row_diag, mx);
  CHASE_CHECK_LAUNCH();
  oz::oz_row_exp<T><<<ceil_div(p, 256), 256, 0, h->stream>>>(mx, (int)p, r);
  CHASE_CHECK_LAUNCH();
  with_S(S, [&](auto Sc) {
    slice_lines<decltype(Sc)::value, T>(Hz, ldh, (int)p, (int)q, 1, col_diag, r, (int)p, -1, z.slices.as<int8_t>(),
                                        ldk, (int64_t)q * ldk, c, h->stream);
  });
  if (split) {
    z.diag.alloc(sizeof(double2) * (size_t)(p + q));
    oz::oz_diag<T><<<ceil_div(p, 256), 256, 0, h->stream>>>(Hz, ldh, (int)p, (int)q, 0, (int)off, z.diag.as<double2>());
    CHASE_CHECK_LAUNCH();
    oz::oz_diag<T><<<ceil_div(q, 256), 256, 0, h->stream>>>(Hz, ldh, (int)p, (int)q, 1, (int)off,
                                                            z.diag.as<double2>() + p);
    CHASE_CHECK_LAUNCH();
  }
  z.S = S;
}

// the shard's slice set (cached within one API call, see invalidate_shard_caches)
template <class T>
static const OzShard& oz_shard(chase_handle* h, const void* H, int64_t ldh) {
  OzShard& z = h->oz_fwd;
  const int S = oz_slices_opt(h);
  if (z.src == H && z.ld == ldh && z.S == S && z.slices.p) return z;
  oz_slice_matrix<T>(h, z, H, ldh, h->grid.rows.len, h->grid.cols.len, true, h->grid.rows.start - h->grid.cols.start);
  z.src = H;
  z.ld = ldh;
  return z;
}

// Y = alpha (op(H) X - gamma E X) + beta Y  (one rank's local part of a fused step; T = double2
// complex Hermitian, T = double real symmetric)
// shard = true: A is the handle's H shard (cached slices, diagonal split, shift); false: a general
// GEMM C = alpha op(A) B + beta C (A sliced for this call, no split, no shift)
template <class T>
static void ozaki_step_t(chase_handle* h, const ZgemmDesc& d, bool shard) {
  constexpr int NP = oz::Comp<T>::NP;
  const int S = oz_slices_opt(h);
  const int dir = d.conjA ? 1 : 0;
  // stored A: shard p x q, or op(A)^{(H)} dims: conjA stores K x M, plain stores M x K
  const int64_t pp = shard ? h->grid.rows.len : (d.conjA ? d.K : d.M);
  const int64_t qq = shard ? h->grid.cols.len : (d.conjA ? d.M : d.K);
  if (!shard) oz_slice_matrix<T>(h, h->oz_g, d.A, d.lda, pp, qq, false, 0);
  const OzShard& A = shard ? oz_shard<T>(h, d.A, d.lda) : h->oz_g;
  const int* r_exp = A.exps.as<int>();
  const int* c_exp = r_exp + (size_t)NP * pp;
  const int M = d.M, N = d.N, K = d.K;
  if (M <= 0 || N <= 0) return;
  cudaStream_t st = h->stream;
  // B operand: the block X (columns contiguous in k)
  const int64_t ldkb = oz::ldk_of(K);
  h->oz_b.alloc((size_t)NP * S * N * ldkb + sizeof(int) * NP * (size_t)N + 64);
  int8_t* bsl = h->oz_b.as<int8_t>();
  int* fB = reinterpret_cast<int*>(bsl + (size_t)NP * S * N * ldkb);
  // B' = D X: forward scales X's rows (k = j) by 2^c_j, backward W's rows (k = i) by 2^r_i; the
  // backward's third component is Wr - Wi (see oz_combine)
  with_S(S, [&](auto Sc) {
    slice_lines<decltype(Sc)::value, T>(reinterpret_cast<const T*>(d.B), d.ldb, K, N, dir == 0 ? 1 : -1, INT_MIN,
                                        dir == 0 ? c_exp : r_exp, dir == 0 ? (int)qq : (int)pp, 1, bsl, ldkb,
                                        (int64_t)N * ldkb, fB, st);
  });
  // FP64 accumulators of the real products
  h->oz_t.alloc(sizeof(double) * NP * (size_t)M * N);
  double* Tacc = h->oz_t.as<double>();
  static unsigned long long attr1 = 0, attr2 = 0;
  if (first_on_device(attr1))
    CHASE_CUDA(cudaFuncSetAttribute(oz::oz_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)oz::Shape<1>::SMEM));
  if (first_on_device(attr2))
    CHASE_CUDA(cudaFuncSetAttribute(oz::oz_gemm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)oz::Shape<2>::SMEM));
  static const int ns_env = [] { const char* e = std::getenv("CHASE_OZ_NS"); return e ? std::atoi(e) : 0; }();
  // 256 x 512 tiles (NS = 2) measured slower at the bench shape (87-89 vs 104-105 TFLOP/s: one
  // accumulator leaves the drain exposed and 4 stages hide less latency), so NS = 1 is the default
  const int ns = ns_env == 2 && N > oz::BN ? 2 : 1;
  const int64_t ldka = oz::ldk_of(pp);           // slices [j][i], row length ldk(p)
  int cap = oz::MAX_PAIRS;                                  // pairs per launch (see the packing below)
  static const int cap_env = [] { const char* e = std::getenv("CHASE_OZ_PAIRS"); return e ? std::atoi(e) : 0; }();
  if (cap_env > 0) cap = std::min(cap, cap_env);          // tuning knob: slice pairs per launch
  static const int hint_env = [] { const char* e = std::getenv("CHASE_OZ_HINT"); return e ? std::atoi(e) : 0; }();
  static const int dbg_env = [] { const char* e = std::getenv("CHASE_OZ_DBG"); return e ? std::atoi(e) : 0; }();
  static const int sync_env = [] { const char* e = std::getenv("CHASE_OZ_SYNC"); return e ? std::atoi(e) : 1; }();
  static const int snake_env = [] { const char* e = std::getenv("CHASE_OZ_SNAKE"); return e ? std::atoi(e) : 1; }();
  h->oz_sync.alloc(256);
  if (16129LL * K > 2147483647LL) throw UsageError("fp64_emulation: K > 133143 needs K chunking (not built)");
  const bool crt = S == oz::NMOD;
  if (crt && 16384LL * K > 2147483647LL) throw UsageError("oz_crt: K > 131071 needs K chunking (not built)");
  uint8_t* Ibuf = nullptr;
  if (crt) {
    h->oz_i.alloc((size_t)oz::NMOD * M * N);
    Ibuf = h->oz_i.as<uint8_t>();
  }
  const int ptiles = ceil_div(M, 2 * oz::BM) * ceil_div(N, ns * oz::BN);
  int sms = 148;
  {
    int dev = 0;
    CHASE_CUDA(cudaGetDevice(&dev));
    CHASE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int grid = 2 * std::min(ptiles, sms / 2);            // persistent: one CTA pair per 2 SMs
  for (int P = 0; P < NP; ++P) {
    CUtensorMap ta, tb;
    // [P][s][j][i]: dims {p (i, inner), q (j), S}; box {128, 128, 1} serves both directions
    oz::make_slice_tmap(&ta, A.slices.as<int8_t>() + (size_t)P * S * qq * ldka, pp, qq, ldka, S, oz::BM);
    oz::make_slice_tmap(&tb, bsl + (size_t)P * S * N * ldkb, K, N, ldkb, S, oz::BN / 2);
    bool first = true;
    if (crt) {
      // scheme II: one launch per modulus (residue plane i of A times plane i of B), then Garner
      for (int i = 0; i < oz::NMOD; ++i) {
        oz::Params prm{};
        prm.M = M; prm.N = N; prm.K = K;
        prm.npairs = 1;
        prm.sa[0] = i;
        prm.tb[0] = i;
        prm.scale = 1.0;
        prm.out = nullptr;
        prm.rout = Ibuf + (size_t)i * M * N;
        prm.modulus = oz::crt_mod(i);
        prm.ldo = M;
        prm.amn = dir == 0 ? 1 : 0;
        prm.snake = snake_env;
        prm.sync = nullptr;
        if (sync_env && !h->colocated) {
          CHASE_CUDA(cudaMemsetAsync(h->oz_sync.p, 0, 64, st));
          prm.sync = h->oz_sync.as<unsigned>();
        }
        oz::oz_gemm_kernel<1><<<grid, oz::THREADS, oz::Shape<1>::SMEM, st>>>(ta, tb, prm);
        CHASE_CHECK_LAUNCH();
      }
      oz::oz_crt<<<148 * 8, 256, 0, st>>>(Ibuf, (int64_t)M * N, M, N, Tacc + (size_t)P * M * N, M);
      CHASE_CHECK_LAUNCH();
      continue;
    }
    for (int dsum = 2; dsum <= S + 1; ++dsum) {
      std::vector<std::pair<int, int>> pairs;
      for (int s = 1; s < dsum; ++s)
        if (s <= S && dsum - s <= S) pairs.push_back({s - 1, dsum - s - 1});
      // pack the group's pairs into launches whose int32 sums stay exact: |a_1| <= 127 and
      // |a_s| <= 64 (s >= 2, round-to-nearest slices), so a pair contributes at most
      // m_s m_t K per output and a launch may hold pairs while sum m_s m_t K <= 2^31 - 1
      // (at K = 30000 every d group fits one launch: 7 launches per real product)
      auto mag = [](int s0) { return s0 == 0 ? 127LL : 64LL; };
      for (size_t b0 = 0, b1; b0 < pairs.size(); b0 = b1) {
        long long bound = 0;
        for (b1 = b0; b1 < pairs.size() && (int)(b1 - b0) < cap; ++b1) {
          const long long add = mag(pairs[b1].first) * mag(pairs[b1].second) * (long long)K;
          if (b1 > b0 && bound + add > 2147483647LL) break;
          bound += add;
        }
        oz::Params prm{};
        prm.M = M; prm.N = N; prm.K = K;
        prm.npairs = (int)(b1 - b0);
        for (int q = 0; q < prm.npairs; ++q) {
          prm.sa[q] = pairs[b0 + q].first;
          prm.tb[q] = pairs[b0 + q].second;
        }
        prm.scale = std::ldexp(1.0, -7 * dsum);
        prm.out = Tacc + (size_t)P * M * N;
        prm.ldo = M;
        prm.accumulate = first ? 0 : 1;
        prm.hint = hint_env;
        prm.amn = dir == 0 ? 1 : 0;
        prm.dbg = dbg_env;
        prm.snake = snake_env;
        prm.sync = nullptr;
        if (sync_env && !h->colocated) {     // co-located ranks share the SMs: no round barrier
          CHASE_CUDA(cudaMemsetAsync(h->oz_sync.p, 0, 64, st));
          prm.sync = h->oz_sync.as<unsigned>();
        }
        first = false;
        if (ns == 2) oz::oz_gemm_kernel<2><<<grid, oz::THREADS, oz::Shape<2>::SMEM, st>>>(ta, tb, prm);
        else oz::oz_gemm_kernel<1><<<grid, oz::THREADS, oz::Shape<1>::SMEM, st>>>(ta, tb, prm);
        CHASE_CHECK_LAUNCH();
      }
    }
  }
  const int* eA = dir == 0 ? r_exp : c_exp;        // output row exponents
  // intersection rows of this direction (the diagonal split and the shift live there)
  const Grid& g = h->grid;
  const int64_t r0 = g.rows.start, c0 = g.cols.start, p = g.rows.len, q = g.cols.len;
  int dlo, dhi;
  int64_t doff;
  if (dir == 0) {
    dlo = (int)std::max<int64_t>(0, c0 - r0); dhi = (int)std::min<int64_t>(p, c0 + q - r0); doff = r0 - c0;
  } else {
    dlo = (int)std::max<int64_t>(0, r0 - c0); dhi = (int)std::min<int64_t>(q, r0 + p - c0); doff = c0 - r0;
  }
  if (!shard) dlo = dhi = 0;                            // no split, no shift
  oz::oz_combine<T><<<148 * 8, 256, 0, st>>>(Tacc, M, (int64_t)M * N, eA, M, fB, N, reinterpret_cast<T*>(d.C), d.ldc,
                                             d.alpha, d.beta, d.beta != 0.0 ? 1 : 0, reinterpret_cast<const T*>(d.B),
                                             d.ldb, shard ? A.diag.as<double2>() + (dir == 0 ? 0 : pp) : nullptr, dlo,
                                             std::max(dlo, dhi), doff, d.gamma, dir);
  CHASE_CHECK_LAUNCH();
}

void ozaki_step(chase_handle* h, const ZgemmDesc& d) {
  if (h->real()) ozaki_step_t<double>(h, d, true);
  else ozaki_step_t<double2>(h, d, true);
}

void ozaki_gemm(chase_handle* h, const ZgemmDesc& d) {
  if (d.S || d.red || d.b_upper) throw std::logic_error("ozaki_gemm: plain products only");
  if (h->real()) ozaki_step_t<double>(h, d, false);
  else ozaki_step_t<double2>(h, d, false);
}

void ozaki_release(chase_handle* h) {
  for (OzShard* z : {&h->oz_fwd, &h->oz_g}) {
    z->slices.release();
    z->exps.release();
    z->diag.release();
    z->src = nullptr;
  }
  h->oz_b.release();
  h->oz_t.release();
  h->oz_i.release();
  h->oz_sync.release();
}

}  // namespace chase
