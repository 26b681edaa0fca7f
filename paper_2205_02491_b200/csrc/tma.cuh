// TMA (cp.async.bulk.tensor) + mbarrier primitives for sm_100a, written as inline PTX.
// Host side: tensor-map encoding through the driver entry point (no libcuda link needed).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include "common.cuh"

namespace chase {

// ---------------------------------------------------------------- device side
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// 2D tiled TMA load global -> shared, completion signalled on `bar` (complete_tx::bytes).
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* m, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* m, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- host side
// 2-D FP64 tensor map over a column-major complex matrix (rows x cols, leading dim ld in complex
// elements).  Dim 0 = 2*rows doubles (contiguous), dim 1 = cols.  Box = {16 doubles (8 complex,
// 128 B), box_cols}, SWIZZLE_128B: the 16-byte chunk index of every 128-B smem row is XORed with
// (row index mod 8).  Out-of-bounds elements are zero-filled.
void make_zmatrix_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                       int box_cols);
// 3-D view of the same matrix for "row-chunked" tiles (rows % 8 == 0): dim 0 = 16 doubles (8
// complex rows of a chunk), dim 1 = cols (stride ld), dim 2 = rows/8 chunks (stride 128 B).  One
// box {16, box_cols, box_chunks} lands as smem [chunk][col][8 rows] -- the forward-A layout -- in a
// single TMA instead of box_chunks 2-D loads.  Returns false if the driver rejects the map.
bool make_zmatrix_tmap_chunked(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                               int box_cols, int box_chunks);

}  // namespace chase
