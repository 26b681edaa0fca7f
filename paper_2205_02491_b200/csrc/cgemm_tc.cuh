// Complex-single fused filter step on the 5th-generation tensor cores (tcgen05, kind::tf32) with
// the 3xTF32 split ("c64 uses tcgen05 kind::tf32, 3xTF32 split for FP32 accuracy,
// with FP32 accumulation").
//
// Complex arithmetic is mapped onto real TF32 MMAs through the storage itself (no operand copies
// of H):
//   forward  W = H V : A = H viewed as a REAL (2M x K) matrix (complex rows interleaved re/im,
//            MN-major), B1 = Re V, B2 = Im V (planar K x N, K-major).  D1 = A B1, D2 = A B2 hold
//            (Hr Vr, Hi Vr) and (Hr Vi, Hi Vi) on even/odd TMEM lanes, so
//            Re W[m] = D1[2m] - D2[2m+1], Im W[m] = D1[2m+1] + D2[2m]   (one lane-pair shuffle);
//            the real row index IS the interleaved storage index of W.
//   backward V = H^H W : A = H columns as a REAL (M x 2K) K-major matrix, B1 = W interleaved
//            (2K x N), B2 = (-i W) interleaved: D1 = Re V, D2 = Im V directly.
// 3xTF32: x = hi + lo with hi = tf32 truncation (what the MMA reads from an fp32 word) and
// lo = RN_tf32(x - hi); D += A_hi B_hi + A_hi B_lo + A_lo B_hi (the lo*lo term is ~2^-24 relative).
// H_lo is computed once per shard; the epilogues write the lo / rotated copies the NEXT step
// consumes, so every operand arrives by TMA.
//
// Roles (320 threads, 1 CTA per 128-row x BN-column tile): thread 0 issues TMA into a 2-4 stage
// mbarrier ring, one elected lane of warp 1 issues 3 tcgen05.mma (M=128, N=2 BN: B1 and B2 sit
// side by side in shared memory, so one MMA reads each A tile once for both) per 8-deep k step
// into the two BN-column TMEM accumulators of the current K chunk and commits each stage back to
// its `empty` barrier; warps 2-9 drain finished chunks (tcgen05.ld 32x32b, lane quadrant =
// warp % 4, column half = (warp - 2) / 4) into FP32 registers and run the fused epilogue.
#pragma once
#include <cstdint>
#include "common.cuh"
#include "tma.cuh"
#include "zgemm.h"

namespace chase {

// f1 for complex single: the same last-arriver tile reduction as the complex-double GEMM
// (zgemm.h PeerRed), here on fp32 staging; the reducer also writes the derived operand formats
// (rotated / lo copies) into every replica.
struct C64Red {
  int n = 0, me = 0;
  float* stage[kMaxPeers] = {};    // staging buffer of every comm rank
  float* base[kMaxPeers] = {};     // operand-format buffer of every comm rank (c64w fwd / c64v bwd)
  int64_t o0 = 0, o1 = 0, o0lo = 0, o1lo = 0;   // offsets (floats) of Y0 / Y1 / Y0lo / Y1lo from base
  int64_t plane = 0;               // staging offset (floats) of the backward's Im plane
  unsigned* ctr = nullptr;
  unsigned* done[kMaxPeers] = {};
};

struct C64Params {
  int M, N, K;             // output rows (complex: fwd counts real rows 2*M_complex), cols, k (real MMA k)
  float alpha, beta, gamma;
  // shift source and beta/output in the step's formats (see cgemm_tc.cu)
  const float* S0;          // fwd: Re X plane; bwd: X interleaved
  const float* S1;          // fwd: Im X plane
  int64_t lds;
  int shift_lo, shift_hi;   // complex output rows carrying the shift
  int64_t shift_off;
  float* Y0;                // fwd: W interleaved (real rows); bwd: Re V plane
  float* Y1;                // fwd: (-i W) interleaved;        bwd: Im V plane
  float* Y0lo;              // lo copies (may be null)
  float* Y1lo;
  int64_t ldy;              // in floats (fwd: 2*p rows; bwd: q)
  int beta_on;
  int kc_stages;            // K chunk (in BK stages) per fresh TMEM accumulator; 0 = default
  int raster_group;         // pair kernel tile order: 0 = N fastest; g > 0 = groups of g M pairs, M fastest
  C64Red red;               // f1 (pair kernel): fused all-reduce over peer memory when red.n > 1
};

namespace tc {
constexpr int BMR = 128;   // real rows per tile (fwd: 64 complex rows; bwd: 128 complex rows)
constexpr int BK = 32;     // real k per stage (one 128-byte row of tf32)
constexpr uint32_t A_BYTES = BMR * BK * 4;            // 16 KB
template <int BN>
struct Cfg {
  // B1 | B2 adjacent (one N = 2 BN operand), then their lo copies: one MMA per (hi/lo) pair
  static constexpr uint32_t B_BYTES = BK * BN * 4;
  static constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 4 * B_BYTES;
  static constexpr int STAGES = (220 * 1024) / STAGE_BYTES > 4 ? 4 : (220 * 1024) / STAGE_BYTES;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 1024;
};
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
  d |= (uint64_t)(layout & 7) << 61;        // 2 = SWIZZLE_128B, 1 = SWIZZLE_128B_BASE32B
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
               ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
}

// x = hi + lo with hi = trunc_tf32(x) (what the MMA reads from the fp32 word).  lo is stored
// pre-rounded to TF32 with round-to-nearest-even, so the MMA reads it exactly and the dropped
// remainder (<= 2^-12 |lo|) is unbiased; a truncated lo would bias every product toward zero by
// ~2^-23 relative (measured: 2e-6 relative HQ error at K = 4000 before this rounding).
__device__ __forceinline__ float tf32_rn(float y) {
  uint32_t b = __float_as_uint(y);
  b += 0xFFFu + ((b >> 13) & 1u);
  return __uint_as_float(b & 0xFFFFE000u);
}
__device__ __forceinline__ float tf32_lo(float x) {
  return tf32_rn(x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u));
}
}  // namespace tc

// f1 epilogue (pair kernel, 8 drain warps = 256 threads, named barrier 1): stage this rank's
// partial, arrive on the tile counter, and if last sum the partials in comm-rank order and store
// the sum into every replica (the rotated / lo copies are rebuilt locally after the step: one
// remote array instead of four).
__device__ __forceinline__ void drain_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <bool FWD, int HN>
__device__ __forceinline__ void c64_epilogue_fused(const C64Params& p, int row, int nbase, const float (&a1)[HN],
                                                   const float (&a2)[HN]) {
  const C64Red& R = p.red;
  const float ag = p.alpha * p.gamma;
  float* st = R.stage[R.me];
  const bool odd = (row & 1);
#pragma unroll
  for (int j = 0; j < HN; ++j) {
    const int n = nbase + j;
    const bool ok = n < p.N && row < p.M;
    const int64_t o = (int64_t)row + (int64_t)n * p.ldy;
    if constexpr (FWD) {
      const float d2p = __shfl_xor_sync(0xffffffffu, a2[j], 1);
      float v = (odd ? (a1[j] + d2p) : (a1[j] - d2p)) * p.alpha;
      const int mc = row >> 1;
      if (ok) {
        if (mc >= p.shift_lo && mc < p.shift_hi) {
          const float* src = odd ? p.S1 : p.S0;
          v -= ag * src[(int64_t)mc + p.shift_off + (int64_t)n * p.lds];
        }
        if (p.beta_on) v += p.beta * p.Y0[o];
        st[o] = v;
      }
    } else {
      if (ok) {
        float vr = p.alpha * a1[j], vi = p.alpha * a2[j];
        if (row >= p.shift_lo && row < p.shift_hi) {
          const float* src = p.S0 + 2 * ((int64_t)row + p.shift_off) + 2 * (int64_t)n * p.lds;
          vr -= ag * src[0];
          vi -= ag * src[1];
        }
        if (p.beta_on) {
          vr += p.beta * p.Y0[o];
          vi += p.beta * p.Y1[o];
        }
        st[o] = vr;
        st[R.plane + o] = vi;
      }
    }
  }
  __shared__ int s_last;
  __threadfence_system();
  drain_bar();
  if (threadIdx.x == 64) {
    const unsigned old = atomicAdd_system(R.ctr + blockIdx.x, 1u);
    s_last = ((old + 1u) % (unsigned)R.n) == 0u;
  }
  drain_bar();
  if (!s_last) return;
  __threadfence_system();
#pragma unroll 4
  for (int j = 0; j < HN; ++j) {
    const int n = nbase + j;
    const bool ok = n < p.N && row < p.M;
    const int64_t o = (int64_t)row + (int64_t)n * p.ldy;
    if constexpr (FWD) {
      float v = 0.f;
      if (ok) {
        v = __ldcg(R.stage[0] + o);
        for (int r = 1; r < R.n; ++r) v += __ldcg(R.stage[r] + o);
      }
      const float vp = __shfl_xor_sync(0xffffffffu, v, 1);
      (void)vp;
      if (ok)
        for (int r = 0; r < R.n; ++r) R.base[r][R.o0 + o] = v;   // derived formats: rebuilt locally
    } else if (ok) {
      float vr = __ldcg(R.stage[0] + o), vi = __ldcg(R.stage[0] + R.plane + o);
      for (int r = 1; r < R.n; ++r) {
        vr += __ldcg(R.stage[r] + o);
        vi += __ldcg(R.stage[r] + R.plane + o);
      }
      for (int r = 0; r < R.n; ++r) {
        R.base[r][R.o0 + o] = vr;
        R.base[r][R.o1 + o] = vi;
      }
    }
  }
  __threadfence_system();
  drain_bar();
  if (threadIdx.x >= 64 && threadIdx.x < 64 + R.n) atomicAdd_system(R.done[threadIdx.x - 64], 1u);
}

// fused epilogue from the drained FP32 accumulators of one thread (one row, HN columns of each of
// D1 / D2): shift on the intersection rows, scale, beta term, and the next step's operand formats
template <bool FWD, int HN>
__device__ __forceinline__ void c64_epilogue(const C64Params& p, int row, int nbase, const float (&a1)[HN],
                                             const float (&a2)[HN]) {
  const float ag = p.alpha * p.gamma;
#pragma unroll
  for (int j = 0; j < HN; ++j) {
    const int n = nbase + j;
    const float d1 = a1[j], d2 = a2[j];
    if constexpr (FWD) {
      // even lane (real row 2m): Re W = D1[2m] - D2[2m+1]; odd lane: Im W = D1[2m+1] + D2[2m]
      const float d2p = __shfl_xor_sync(0xffffffffu, d2, 1);
      const bool odd = (row & 1);
      float v = odd ? (d1 + d2p) : (d1 - d2p);
      v *= p.alpha;
      const int mc = row >> 1;                         // complex row
      if (n < p.N && row < p.M) {
        if (mc >= p.shift_lo && mc < p.shift_hi) {
          const float* src = odd ? p.S1 : p.S0;        // planar Re / Im of X
          v -= ag * src[(int64_t)mc + p.shift_off + (int64_t)n * p.lds];
        }
        float* y = p.Y0 + (int64_t)row + (int64_t)n * p.ldy;
        if (p.beta_on) v += p.beta * *y;
      }
      // rotated copy -i W: (Im, -Re) -> even lane takes Im from its partner, odd lane -Re
      const float vp = __shfl_xor_sync(0xffffffffu, v, 1);
      if (n < p.N && row < p.M) {
        const int64_t o = (int64_t)row + (int64_t)n * p.ldy;
        p.Y0[o] = v;
        const float rot = odd ? -vp : vp;
        if (p.Y1) p.Y1[o] = rot;
        if (p.Y0lo) p.Y0lo[o] = tc::tf32_lo(v);
        if (p.Y1lo) p.Y1lo[o] = tc::tf32_lo(rot);
      }
    } else {
      if (n < p.N && row < p.M) {
        float vr = p.alpha * d1, vi = p.alpha * d2;
        if (row >= p.shift_lo && row < p.shift_hi) {
          const float* src = p.S0 + 2 * ((int64_t)row + p.shift_off) + 2 * (int64_t)n * p.lds;   // interleaved X
          vr -= ag * src[0];
          vi -= ag * src[1];
        }
        const int64_t o = (int64_t)row + (int64_t)n * p.ldy;
        if (p.beta_on) {
          vr += p.beta * p.Y0[o];
          vi += p.beta * p.Y1[o];
        }
        p.Y0[o] = vr;
        p.Y1[o] = vi;
        if (p.Y0lo) p.Y0lo[o] = tc::tf32_lo(vr);
        if (p.Y1lo) p.Y1lo[o] = tc::tf32_lo(vi);
      }
    }
  }
}

// FWD = true: forward step (A MN-major from H, output W interleaved + rotated + lo copies)
// FWD = false: backward step (A K-major from H's columns, output V planar + lo planes)
//
// Accumulation: the tensor core's FP32 accumulator loses precision with every MMA added into it
// (measured step error, K = 1200: 1.3e-7 / 1.9e-7 / 3.0e-7 / 5.3e-7 / 1.9e-6 for chunks of
// 32 / 64 / 128 / 256 / 1024 real k -- linear in the chunk length; unchunked it reached 5e-6 at
// K = 1200 and grows with K).  The K loop is therefore cut into chunks of 128 (64 costs ~4 % of
// throughput for 1.9e-7 instead of 3.0e-7; 32 costs ~10 %): every chunk starts
// a fresh TMEM accumulator (double-buffered, 2 x 2BN columns), and 8 epilogue warps drain the
// finished chunk into FP32 registers with round-to-nearest adds while the next chunk accumulates.
constexpr int C64_THREADS = 320;       // warp 0 TMA, warp 1 MMA, warps 2..9 chunk drain + epilogue
constexpr int C64_KC_STAGES = 4;       // chunk = 4 stages x BK 32 = 128 real k (error ~ linear in chunk length)

template <bool FWD, int BN>
__global__ void __launch_bounds__(C64_THREADS, 1)
    c64_step_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tAlo,
                    const __grid_constant__ CUtensorMap tB1, const __grid_constant__ CUtensorMap tB1lo,
                    const __grid_constant__ CUtensorMap tB2, const __grid_constant__ CUtensorMap tB2lo,
                    C64Params p) {
  using namespace tc;
  constexpr uint32_t B_BYTES = Cfg<BN>::B_BYTES, STAGE_BYTES = Cfg<BN>::STAGE_BYTES;
  constexpr int STAGES = Cfg<BN>::STAGES;
  const int CH = p.kc_stages > 0 ? p.kc_stages : C64_KC_STAGES;
  constexpr uint32_t TCOLS = 4 * BN;     // 2 chunk buffers x (D1 | D2)
  constexpr int HN = BN / 2;             // columns per epilogue warp (per accumulator)
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES], empty[STAGES], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = (p.N + BN - 1) / BN;
  const int m0 = (blockIdx.x / tiles_n) * BMR;     // real-row (fwd) / complex-row (bwd) tile origin
  const int n0 = (blockIdx.x % tiles_n) * BN;
  const int KT = (p.K + BK - 1) / BK;
  const int NCH = (KT + CH - 1) / CH;

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
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      tma_prefetch_desc(&tA);
      tma_prefetch_desc(&tB1);
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) mbar_wait(empty + s, ((kt / STAGES) - 1) & 1);
        unsigned char* st = sm + s * STAGE_BYTES;
        mbar_arrive_expect_tx(full + s, STAGE_BYTES);
        const int k0 = kt * BK;
        if constexpr (FWD) {
          // A MN-major: 4 boxes of 32 real rows x BK k -> [row-chunk][k][32 floats] (128B, 32B atoms)
#pragma unroll
          for (int c = 0; c < BMR / 32; ++c) {
            tma_load_2d(st + c * (BK * 128), &tA, m0 + 32 * c, k0, full + s);
            tma_load_2d(st + A_BYTES + c * (BK * 128), &tAlo, m0 + 32 * c, k0, full + s);
          }
        } else {
          // A K-major: one box of BK real k x 128 rows -> [row][32 floats]
          tma_load_2d(st, &tA, k0, m0, full + s);
          tma_load_2d(st + A_BYTES, &tAlo, k0, m0, full + s);
        }
        unsigned char* sb = st + 2 * A_BYTES;
        tma_load_2d(sb, &tB1, k0, n0, full + s);
        tma_load_2d(sb + B_BYTES, &tB2, k0, n0, full + s);
        tma_load_2d(sb + 2 * B_BYTES, &tB1lo, k0, n0, full + s);
        tma_load_2d(sb + 3 * B_BYTES, &tB2lo, k0, n0, full + s);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    uint32_t leader;
    asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(leader));
    // instruction descriptor: F32 accumulate, TF32 A/B, A major (fwd MN / bwd K), B K-major, N, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((FWD ? 1u : 0u) << 15) |
                           ((uint32_t)((2 * BN) >> 3) << 17) | ((uint32_t)(BMR >> 4) << 24);
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % STAGES;
      const int chunk = kt / CH, b = chunk & 1;
      const bool chunk_start = (kt % CH) == 0;
      if (chunk_start && chunk >= 2) {                     // buffer b drained (chunk - 2)?
        mbar_wait(acc_empty + b, ((chunk >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
      mbar_wait(full + s, (kt / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (leader) {
        const uint32_t st = smem_u32(sm + s * STAGE_BYTES);
        const uint32_t sa = st, salo = st + A_BYTES, sb = st + 2 * A_BYTES;
        const uint32_t td = tm + (uint32_t)b * 2 * BN;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          uint64_t da, dal;
          if constexpr (FWD) {
            da = sdesc(sa + kk * 1024, BK * 128, 512, 1);
            dal = sdesc(salo + kk * 1024, BK * 128, 512, 1);
          } else {
            da = sdesc(sa + kk * 32, 16, 1024, 2);
            dal = sdesc(salo + kk * 32, 16, 1024, 2);
          }
          // [B1 | B2] as one K-major operand of 2 BN rows: D[:, 0:BN) = A B1, D[:, BN:2BN) = A B2
          const uint64_t db = sdesc(sb + kk * 32, 16, 1024, 2);
          const uint64_t dbl = sdesc(sb + 2 * B_BYTES + kk * 32, 16, 1024, 2);
          const uint32_t acc = (chunk_start && kk == 0) ? 0u : 1u;
          tc::mma_tf32(td, da, db, idesc, acc);             // D = A_hi B_hi
          tc::mma_tf32(td, da, dbl, idesc, 1u);             //   + A_hi B_lo
          tc::mma_tf32(td, dal, db, idesc, 1u);             //   + A_lo B_hi
        }
        tc::commit(empty + s);                              // smem slot free once these MMAs retire
        if ((kt % CH) == CH - 1 || kt == KT - 1) tc::commit(acc_full + b);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------------ drain + epilogue (8 warps)
    const int quad = warp & 3;                       // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;                // column half of each accumulator
    const int row = m0 + 32 * quad + lane;           // real row (fwd) / complex row (bwd)
    const uint32_t lane_base = tm + ((uint32_t)(32 * quad) << 16) + (uint32_t)(half * HN);
    float a1[HN], a2[HN];
#pragma unroll
    for (int j = 0; j < HN; ++j) a1[j] = a2[j] = 0.f;
    for (int chunk = 0; chunk < NCH; ++chunk) {
      const int b = chunk & 1;
      mbar_wait(acc_full + b, (chunk >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t base = lane_base + (uint32_t)b * 2 * BN;
#pragma unroll
      for (int c0 = 0; c0 < HN; c0 += 16) {
        uint32_t r1[16], r2[16];
        tc::ld16(base + c0, r1);
        tc::ld16(base + BN + c0, r2);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          a1[c0 + j] += __uint_as_float(r1[j]);
          a2[c0 + j] += __uint_as_float(r2[j]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + b);
    }
    c64_epilogue<FWD, HN>(p, row, n0 + half * HN, a1, a2);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(TCOLS));
}

// ============================================================================================
// CTA-pair variant (tcgen05 cta_group::2): the two CTAs of a cluster share one M = 256 x N = 2BN
// MMA.  Each CTA stages its own 128 A rows and HALF of [B1 | B2] (rank 0: B1, rank 1: B2), so per
// CTA a stage is 64 KB instead of 96 KB (3 stages fit) and the L2 -> SM tile traffic drops by 1/3.
// The leader (rank 0) issues the MMAs; both CTAs' TMA loads complete on the leader's `full`
// barrier; MMA commits are multicast to both CTAs' `empty` / `acc_full` barriers; the 16 drain
// warps of the pair arrive on the leader's `acc_empty`.  Each CTA's TMEM holds its 128 rows of
// D = [A B1 | A B2], so the drain / epilogue code is the single-CTA one.
namespace tc2 {
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* m, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void arrive_cluster(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAITC:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONEC;\n"
      "bra LAB_WAITC;\n"
      "DONEC:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p; }"
               ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_both(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
}  // namespace tc2

template <int BN>
struct Cfg2 {
  static constexpr uint32_t B_BYTES = tc::BK * BN * 4;                       // one CTA's B half
  static constexpr uint32_t STAGE_BYTES = 2 * tc::A_BYTES + 2 * B_BYTES;   // A hi/lo + B half hi/lo
  static constexpr int STAGES = (220 * 1024) / STAGE_BYTES > 4 ? 4 : (220 * 1024) / STAGE_BYTES;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 1024;
};

template <bool FWD, int BN, bool RED>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(C64_THREADS, 1)
    c64_step_kernel2(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tAlo,
                     const __grid_constant__ CUtensorMap tB1, const __grid_constant__ CUtensorMap tB1lo,
                     const __grid_constant__ CUtensorMap tB2, const __grid_constant__ CUtensorMap tB2lo,
                     C64Params p) {
  using namespace tc;
  constexpr uint32_t B_BYTES = Cfg2<BN>::B_BYTES, STAGE_BYTES = Cfg2<BN>::STAGE_BYTES;
  constexpr int STAGES = Cfg2<BN>::STAGES;
  const int CH = p.kc_stages > 0 ? p.kc_stages : C64_KC_STAGES;
  constexpr uint32_t TCOLS = 4 * BN;
  constexpr int HN = BN / 2;
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES], empty[STAGES], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc2::cluster_rank();
  const int tiles_n = (p.N + BN - 1) / BN;
  const int pair = blockIdx.x >> 1;
  int pm, pn;
  if (p.raster_group > 0) {
    // groups of `raster_group` M pairs; inside a group M fastest, then N
    const int tiles_mp = (p.M + 2 * BMR - 1) / (2 * BMR);
    const int per_group = p.raster_group * tiles_n;
    const int grp = pair / per_group, first = grp * p.raster_group;
    const int gsize = min(tiles_mp - first, p.raster_group);
    const int in = pair % per_group;
    pm = first + in % gsize;
    pn = in / gsize;
  } else {
    pm = pair / tiles_n;
    pn = pair % tiles_n;
  }
  const int m0 = pm * (2 * BMR) + (int)rank * BMR;
  const int n0 = pn * BN;
  const int KT = (p.K + BK - 1) / BK;
  const int NCH = (KT + CH - 1) / CH;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + b, 1);
      mbar_init(acc_empty + b, 16);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  tc2::cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer (both CTAs)
      tma_prefetch_desc(&tA);
      tma_prefetch_desc(rank == 0 ? &tB1 : &tB2);
      const CUtensorMap* tb = rank == 0 ? &tB1 : &tB2;
      const CUtensorMap* tbl = rank == 0 ? &tB1lo : &tB2lo;
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) mbar_wait(empty + s, ((kt / STAGES) - 1) & 1);
        const uint32_t st = smem_u32(sm + s * STAGE_BYTES);
        const uint32_t fb = tc2::mapa(smem_u32(full + s), 0);
        if (rank == 0) mbar_arrive_expect_tx(full + s, 2 * STAGE_BYTES);
        const int k0 = kt * BK;
        if constexpr (FWD) {
#pragma unroll
          for (int c = 0; c < BMR / 32; ++c) {
            tc2::tma_load_2d_pair(st + c * (BK * 128), &tA, m0 + 32 * c, k0, fb);
            tc2::tma_load_2d_pair(st + A_BYTES + c * (BK * 128), &tAlo, m0 + 32 * c, k0, fb);
          }
        } else {
          tc2::tma_load_2d_pair(st, &tA, k0, m0, fb);
          tc2::tma_load_2d_pair(st + A_BYTES, &tAlo, k0, m0, fb);
        }
        tc2::tma_load_2d_pair(st + 2 * A_BYTES, tb, k0, n0, fb);
        tc2::tma_load_2d_pair(st + 2 * A_BYTES + B_BYTES, tbl, k0, n0, fb);
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // -------------------------------------------------------------- MMA issuer (leader CTA)
      uint32_t leader;
      asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(leader));
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((FWD ? 1u : 0u) << 15) |
                             ((uint32_t)((2 * BN) >> 3) << 17) | ((uint32_t)((2 * BMR) >> 4) << 24);
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        const int chunk = kt / CH, b = chunk & 1;
        const bool chunk_start = (kt % CH) == 0;
        if (chunk_start && chunk >= 2) {
          tc2::wait_cluster(acc_empty + b, ((chunk >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        mbar_wait(full + s, (kt / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (leader) {
          const uint32_t st = smem_u32(sm + s * STAGE_BYTES);
          const uint32_t sa = st, salo = st + A_BYTES, sb = st + 2 * A_BYTES;
          const uint32_t td = tm + (uint32_t)b * 2 * BN;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            uint64_t da, dal;
            if constexpr (FWD) {
              da = sdesc(sa + kk * 1024, BK * 128, 512, 1);
              dal = sdesc(salo + kk * 1024, BK * 128, 512, 1);
            } else {
              da = sdesc(sa + kk * 32, 16, 1024, 2);
              dal = sdesc(salo + kk * 32, 16, 1024, 2);
            }
            const uint64_t db = sdesc(sb + kk * 32, 16, 1024, 2);
            const uint64_t dbl = sdesc(sb + B_BYTES + kk * 32, 16, 1024, 2);
            const uint32_t acc = (chunk_start && kk == 0) ? 0u : 1u;
            tc2::mma_tf32(td, da, db, idesc, acc);
            tc2::mma_tf32(td, da, dbl, idesc, 1u);
            tc2::mma_tf32(td, dal, db, idesc, 1u);
          }
          tc2::commit_both(empty + s);
          if ((kt % CH) == CH - 1 || kt == KT - 1) tc2::commit_both(acc_full + b);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------------ drain + epilogue (8 warps)
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = m0 + 32 * quad + lane;
    const uint32_t lane_base = tm + ((uint32_t)(32 * quad) << 16) + (uint32_t)(half * HN);
    float a1[HN], a2[HN];
#pragma unroll
    for (int j = 0; j < HN; ++j) a1[j] = a2[j] = 0.f;
    for (int chunk = 0; chunk < NCH; ++chunk) {
      const int b = chunk & 1;
      mbar_wait(acc_full + b, (chunk >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t base = lane_base + (uint32_t)b * 2 * BN;
#pragma unroll
      for (int c0 = 0; c0 < HN; c0 += 16) {
        uint32_t r1[16], r2[16];
        tc::ld16(base + c0, r1);
        tc::ld16(base + BN + c0, r2);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          a1[c0 + j] += __uint_as_float(r1[j]);
          a2[c0 + j] += __uint_as_float(r2[j]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) tc2::arrive_cluster(tc2::mapa(smem_u32(acc_empty + b), 0));
    }
    if constexpr (RED)
      c64_epilogue_fused<FWD, HN>(p, row, n0 + half * HN, a1, a2);
    else
      c64_epilogue<FWD, HN>(p, row, n0 + half * HN, a1, a2);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  tc2::cluster_sync();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(TCOLS));
}

// ============================================================================================
// Persistent CTA-pair variant (the default, no fused reduction).  L2-aware static schedule: the
// n tiles are cut into segments of gw (a divisor of tiles_n chosen on the host so that a round's
// a x gw tile block, a = npair / gw, reads the fewest A and B panels per tile); the pairs form
// a = npair / gw groups of gw, group g walks the m tiles g, g + a, ... of segment 0, then of
// segment 1, ..., and pair j of the group always takes n tile seg gw + j.  The gw pairs of a group
// stream one A panel (the big H shard) in lockstep, and a round barrier of the TMA producers
// (50 ms timeout: performance only, never correctness) keeps the groups in step, so the B panels
// of the segment are shared too.  (Panels are K long -- far beyond L2 at large shards -- so a
// round costs a + gw panel reads: 17 for 8 x 9 vs 34 for 2 x 32 at N = 170000 / 2 x 2.)  The chunk
// accumulators stay double-buffered across tiles (global chunk counter), so the next tile's first
// chunk overlaps this tile's epilogue.  sync: round-barrier counter (zeroed per launch) or null.
template <bool FWD, int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(C64_THREADS, 1)
    c64_step_kernel_p(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tAlo,
                      const __grid_constant__ CUtensorMap tB1, const __grid_constant__ CUtensorMap tB1lo,
                      const __grid_constant__ CUtensorMap tB2, const __grid_constant__ CUtensorMap tB2lo,
                      C64Params p, unsigned* sync, int gw) {
  using namespace tc;
  constexpr uint32_t B_BYTES = Cfg2<BN>::B_BYTES, STAGE_BYTES = Cfg2<BN>::STAGE_BYTES;
  constexpr int STAGES = Cfg2<BN>::STAGES;
  const int CH = p.kc_stages > 0 ? p.kc_stages : C64_KC_STAGES;
  constexpr uint32_t TCOLS = 4 * BN;
  constexpr int HN = BN / 2;
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES], empty[STAGES], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc2::cluster_rank();
  const int tiles_n = (p.N + BN - 1) / BN, tiles_m = (p.M + 2 * BMR - 1) / (2 * BMR);
  const int pair = blockIdx.x >> 1, npair = gridDim.x >> 1;
  const int nseg = tiles_n / gw, ngroups = npair / gw;
  const int g = pair / gw, jn = pair % gw;
  // m tiles of group gg per segment, and this pair's tile count
  auto cnt = [&](int gg) { return gg < tiles_m ? (tiles_m - 1 - gg) / ngroups + 1 : 0; };
  const int NT = g < ngroups ? nseg * cnt(g) : 0;
  auto tile_mn = [&](int r, int& tmi, int& tni) {
    const int c = cnt(g);
    tmi = g + (r % c) * ngroups;
    tni = (r / c) * gw + jn;
  };
  const int KT = (p.K + BK - 1) / BK;
  const int NCH = (KT + CH - 1) / CH;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + b, 1);
      mbar_init(acc_empty + b, 16);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  tc2::cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tA);
      tma_prefetch_desc(rank == 0 ? &tB1 : &tB2);
      const CUtensorMap* tb = rank == 0 ? &tB1 : &tB2;
      const CUtensorMap* tbl = rank == 0 ? &tB1lo : &tB2lo;
      int it = 0;
      unsigned target = 0;
      for (int r = 0; r < NT; ++r) {
        if (sync && r > 0) {
          // arrivals at round r: the CTAs of the groups that still have an r-th tile
          int act = 0;
          for (int gg = 0; gg < ngroups; ++gg) act += (nseg * cnt(gg) > r) ? 1 : 0;
          target += 2u * (unsigned)gw * (unsigned)act;
          atomicAdd(sync, 1u);
          unsigned long long t0, t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          unsigned v;
          while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sync) : "memory");
            if (v >= target) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 > 50000000ull) { sync = nullptr; break; }
          }
        }
        int tmi, tni;
        tile_mn(r, tmi, tni);
        const int m0 = tmi * (2 * BMR) + (int)rank * BMR;
        const int n0 = tni * BN;
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(empty + s, ((it / STAGES) - 1) & 1);
          const uint32_t st = smem_u32(sm + s * STAGE_BYTES);
          const uint32_t fb = tc2::mapa(smem_u32(full + s), 0);
          if (rank == 0) mbar_arrive_expect_tx(full + s, 2 * STAGE_BYTES);
          const int k0 = kt * BK;
          if constexpr (FWD) {
#pragma unroll
            for (int c = 0; c < BMR / 32; ++c) {
              tc2::tma_load_2d_pair(st + c * (BK * 128), &tA, m0 + 32 * c, k0, fb);
              tc2::tma_load_2d_pair(st + A_BYTES + c * (BK * 128), &tAlo, m0 + 32 * c, k0, fb);
            }
          } else {
            tc2::tma_load_2d_pair(st, &tA, k0, m0, fb);
            tc2::tma_load_2d_pair(st + A_BYTES, &tAlo, k0, m0, fb);
          }
          tc2::tma_load_2d_pair(st + 2 * A_BYTES, tb, k0, n0, fb);
          tc2::tma_load_2d_pair(st + 2 * A_BYTES + B_BYTES, tbl, k0, n0, fb);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      uint32_t leader;
      asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(leader));
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((FWD ? 1u : 0u) << 15) |
                             ((uint32_t)((2 * BN) >> 3) << 17) | ((uint32_t)((2 * BMR) >> 4) << 24);
      int it = 0, gc = 0;
      for (int r = 0; r < NT; ++r) {
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int s = it % STAGES;
          const bool chunk_start = (kt % CH) == 0;
          const int cg = gc + kt / CH, b = cg & 1;            // global chunk index
          if (chunk_start && cg >= 2) {
            tc2::wait_cluster(acc_empty + b, ((cg >> 1) - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
          }
          mbar_wait(full + s, (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (leader) {
            const uint32_t st = smem_u32(sm + s * STAGE_BYTES);
            const uint32_t sa = st, salo = st + A_BYTES, sb = st + 2 * A_BYTES;
            const uint32_t td = tm + (uint32_t)b * 2 * BN;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              uint64_t da, dal;
              if constexpr (FWD) {
                da = sdesc(sa + kk * 1024, BK * 128, 512, 1);
                dal = sdesc(salo + kk * 1024, BK * 128, 512, 1);
              } else {
                da = sdesc(sa + kk * 32, 16, 1024, 2);
                dal = sdesc(salo + kk * 32, 16, 1024, 2);
              }
              const uint64_t db = sdesc(sb + kk * 32, 16, 1024, 2);
              const uint64_t dbl = sdesc(sb + B_BYTES + kk * 32, 16, 1024, 2);
              const uint32_t acc = (chunk_start && kk == 0) ? 0u : 1u;
              tc2::mma_tf32(td, da, db, idesc, acc);
              tc2::mma_tf32(td, da, dbl, idesc, 1u);
              tc2::mma_tf32(td, dal, db, idesc, 1u);
            }
            tc2::commit_both(empty + s);
            if ((kt % CH) == CH - 1 || kt == KT - 1) tc2::commit_both(acc_full + b);
          }
          __syncwarp();
        }
        gc += NCH;
      }
    }
  } else {
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    int gc = 0;
    for (int r = 0; r < NT; ++r) {
      int tmi, tni;
      tile_mn(r, tmi, tni);
      const int m0 = tmi * (2 * BMR) + (int)rank * BMR;
      const int n0 = tni * BN;
      const int row = m0 + 32 * quad + lane;
      const uint32_t lane_base = tm + ((uint32_t)(32 * quad) << 16) + (uint32_t)(half * HN);
      float a1[HN], a2[HN];
#pragma unroll
      for (int j = 0; j < HN; ++j) a1[j] = a2[j] = 0.f;
      for (int chunk = 0; chunk < NCH; ++chunk, ++gc) {
        const int b = gc & 1;
        mbar_wait(acc_full + b, (gc >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t base = lane_base + (uint32_t)b * 2 * BN;
#pragma unroll
        for (int c0 = 0; c0 < HN; c0 += 16) {
          uint32_t r1[16], r2[16];
          tc::ld16(base + c0, r1);
          tc::ld16(base + BN + c0, r2);
          asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            a1[c0 + j] += __uint_as_float(r1[j]);
            a2[c0 + j] += __uint_as_float(r2[j]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) tc2::arrive_cluster(tc2::mapa(smem_u32(acc_empty + b), 0));
      }
      c64_epilogue<FWD, HN>(p, row, n0 + half * HN, a1, a2);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  tc2::cluster_sync();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(TCOLS));
}

// Segment width of the persistent schedule: the divisor gw of tiles_n (gw <= npair) with the fewest
// panel reads per tile of a round, (gw + npair / gw) / ((npair / gw) gw).
inline int c64_segment_width(int tiles_n, int npair) {
  int best = 1;
  double bc = 1e30;
  for (int d = 1; d <= tiles_n && d <= npair; ++d) {
    if (tiles_n % d) continue;
    const int a = npair / d;
    const double c = (double)(d + a) / (double)(a * d);
    if (c < bc - 1e-12) { bc = c; best = d; }
  }
  return best;
}

}  // namespace chase

