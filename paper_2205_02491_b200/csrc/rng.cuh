// Counter-based start-vector generator (device side).  Philox4x32-10 (Salmon et al., SC'11):
// key = (seed lo, seed hi), counter = (global row lo, global row hi, column, stream).
// Entry = re + i im with re = ((u0 << 21) | (u1 >> 11)) * 2^-52 - 1 (exact), im likewise from
// (u2, u3).  Keyed by the GLOBAL row, so every process-grid shape draws the same block.
// (The CPU oracle implements the same definition independently; a GPU test checks bitwise
// agreement.)
#pragma once
#include <cstdint>

namespace chase {

struct Philox4 {
  uint32_t x[4];
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                 uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += W0; k1 += W1; }
    const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
    const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  Philox4 o;
  o.x[0] = c0; o.x[1] = c1; o.x[2] = c2; o.x[3] = c3;
  return o;
}

__device__ __forceinline__ double philox_unit(uint32_t a, uint32_t b) {
  const uint64_t v = ((uint64_t)a << 21) | ((uint64_t)b >> 11);
  return (double)v * 0x1p-52 - 1.0;
}

}  // namespace chase
