// Host interface of the fused complex-double GEMM (see zgemm.cuh for the kernel).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace chase {

// f1: in-kernel all-reduce of a fused step's output over peer memory (CUDA IPC over NVLink).
// Every comm rank stages its partial tile, the last rank to arrive on a tile (system-scope atomic
// counter owned by comm rank 0) sums the n partials in comm-rank order -- identical bits on every
// rank -- and stores the sum into every rank's replica, then bumps every rank's `done` counter.
constexpr int kMaxPeers = 8;
struct PeerRed {
  int n = 0;                           // communicator size (<= 1: no fused reduction)
  int me = 0;                          // my rank in the communicator
  int64_t off = 0;                     // element offset of C inside the replica / staging buffers
  double2* stage[kMaxPeers] = {};      // staging buffer base of every comm rank (same layout as C)
  double2* out[kMaxPeers] = {};        // replica base of every comm rank (C = out[me] + off)
  unsigned* ctr = nullptr;             // tile arrival counters (comm rank 0's memory)
  unsigned* done[kMaxPeers] = {};      // completion counter of every comm rank
};

struct ZgemmDesc {
  int M = 0, N = 0, K = 0;
  bool conjA = false;            // op(A) = A^H with A stored K x M
  const void* A = nullptr; int64_t lda = 0;
  const void* B = nullptr; int64_t ldb = 0;
  void* C = nullptr; int64_t ldc = 0;
  double alpha = 1.0, beta = 0.0, gamma = 0.0;
  const void* S = nullptr; int64_t lds = 0;   // shift source (may be null)
  int shift_lo = 0, shift_hi = 0; int64_t shift_off = 0;
  bool use3m = false;            // 3M (Gauss) complex product: 3 real DMMAs per complex MAC
  bool upper_only = false;       // only tiles on/above the diagonal are computed (Hermitian C)
  bool b_upper = false;          // B upper triangular (zeros below the diagonal are skipped)
  const PeerRed* red = nullptr;  // f1: fused all-reduce of C over a communicator (3M kernel only)
};

// C = alpha*op(A)*B - alpha*gamma*S[shift rows] + beta*C   (all complex double, column-major)
void zgemm(const ZgemmDesc& d, cudaStream_t st);
// number of CTA tiles (= fused-reduction tiles) of the 3M kernel for an M x N output
int zgemm3m_tiles(int M, int N);
int dgemm_tiles(int M, int N);
// The same contract for real double (op(A) = A^T when conjA; use3m ignored).  Real-symmetric f2.
void dgemm(const ZgemmDesc& d, cudaStream_t st);

}  // namespace chase

namespace chase {
// Skinny product C[M x L] = alpha * A[M x K] * B[K x L] for L <= 8 (HBM-bound: streams A once;
// used by the Lanczos step).  `work` must hold skinny_work_bytes(M, K, L).
size_t skinny_work_bytes(int M, int K, int L);
// a_c64: A is complex single (c64 shard), read and accumulated in FP64
void zgemm_skinny(int M, int L, int K, double alpha, const void* A, int64_t lda, const void* B,
                  int64_t ldb, void* C, int64_t ldc, void* work, cudaStream_t st, bool a_c64 = false);
// real variant (f2); `work` as for the complex one (it needs half of it)
void dgemm_skinny(int M, int L, int K, double alpha, const void* A, int64_t lda, const void* B,
                  int64_t ldb, void* C, int64_t ldc, void* work, cudaStream_t st);
}  // namespace chase
