// Internal definition of chase_handle and the library's internal entry points.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <new>
#include <stdexcept>
#include "common.cuh"
#include <string>
#include <vector>
#include "../../include/chase.h"
#include "grid.h"
#include "zgemm.h"
#include "comm.h"
#include "linalg.h"

namespace chase {

struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// a fused-reduce peer stopped arriving: the communicators themselves are intact, so the status is
// still agreed on over the world before the handle is marked unusable
struct PeerTimeout : NcclError {
  using NcclError::NcclError;
};

#define CHASE_NCCL(call)                                                                        \
  do {                                                                                          \
    ncclResult_t _r = (call);                                                                   \
    if (_r != ncclSuccess)                                                                      \
      throw ::chase::NcclError(std::string(#call) + ": " + ncclGetErrorString(_r));             \
  } while (0)

// Device buffer owned by the handle.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void alloc(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    const cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaErrorMemoryAllocation) {          // surfaces as CHASE_E_NOMEM, handle stays usable
      cudaGetLastError();
      p = nullptr;
      throw std::bad_alloc();
    }
    CHASE_CUDA(e);
    bytes = b;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

struct Options {
  int deg_max = 36;
  int deg_extra = 2;            // degrees added to the optimal-degree estimate (reading 4b)
  int max_iter = 0;             // 0 = auto: iterate while converging (stall_iter rule), cap kAutoIterCap
  int stall_iter = 100;         // auto: stop after this many iterations without progress
  int lanczos_steps = 25;
  int lanczos_runs = 4;
  uint64_t seed_v = 2;
  uint64_t seed_lanczos = 3;
  bool largest = false;
  bool approx = false;
  bool gemm3m = true;         // 3M complex products in the filter / HQ GEMMs
  double mixed_filter = 0.0;  // f4: complex-single filter while all active residuals exceed this
  bool fused_reduce = true;   // f1: filter steps all-reduce inside the GEMM over peer memory
  bool fused_reduce_c64 = false;  // f1 for the complex-single filter (measured slower than NCCL + rebuild)
  double peer_timeout = 120.0;    // f1: seconds a rank waits for its peers' tiles before failing
  double comm_timeout = 0.0;      // host waits poll ncclCommGetAsyncError; > 0: also fail after this many s
  double oz_gemm_min = 4e9;       // plain iteration GEMMs with M N K >= this also run on the emulation
  double oz_gemm_kmin = 12288;    // ... if their contraction length K is at least this
  int fp64_emulation = 7;          // f4: > 0 = complex-double filter products on INT8 tensor cores (Ozaki)
  int oz_crt = 1;                  // 1: Ozaki scheme II (16 CRT moduli); 0 (or no room for the residues): S slices
};

}  // namespace chase

struct chase_handle {
  chase::Grid grid;
  int dtype = CHASE_C128;              // CHASE_C128 (complex Hermitian) or CHASE_R64 (real symmetric)
  bool real() const { return dtype == CHASE_R64; }
  bool c64() const { return dtype == CHASE_C64; }
  size_t es() const { return dtype == CHASE_C128 ? 16 : 8; }   // bytes per element
  int nd() const { return real() ? 1 : 2; }              // doubles per element
  int device = 0;
  int world_size = 1;
  cudaStream_t stream = nullptr;       // library stream (all kernels, NCCL)
  cudaStream_t user_stream = nullptr;  // caller stream to order against
  chase::Comm world, rowc, colc;       // NCCL or co-located transport (comm.h)
  bool colocated = false;              // ranks are threads of this process (comm.h)
  chase::Options opt;
  int n_e_max = 0;
  // workspace
  chase::DBuf V, W, HV, V2, G, G2, Z, scratch, red, lz;
  chase::DBuf Hlo;                     // c64: 3xTF32 lo part of the caller's H shard
  chase::DBuf c64v, c64w;              // c64: planar V-layout / W-layout operand formats (c64.cu)
  chase::DBuf H32;                     // f4: complex-single shadow of a complex-double shard
  chase::DBuf Hstage, Vstage;          // chase_solve with host buffers: device copies of H / vectors
  struct OzShard {                     // fp64_emulation: the shard's int8 slice set (ozaki.cu)
    const void* src = nullptr;
    int64_t ld = 0;
    int S = 0;
    chase::DBuf slices, exps, diag;
  } oz_fwd, oz_g;                     // the shard's set; the A operand of a general emulated GEMM
  bool oz_off = false;                 // fp64_emulation fell back to DMMA (slices did not fit)
  bool oz_gemm_off = false;            // plain GEMMs back on DMMA (their A slices did not fit)
  chase::DBuf oz_b, oz_t, oz_sync;     // fp64_emulation: slices of the block X, FP64 product accumulators
  chase::DBuf oz_i;                    // oz_crt: the products' residues (one byte per modulus and output)
  const void* h32_src = nullptr;
  int64_t h32_ld = 0;
  const void* hlo_src = nullptr;
  int64_t hlo_ld = 0;
  chase::JacobiWork* jacobi = nullptr;  // RR eigensolver workspace (linalg.h)
  std::vector<double> host_scratch;
  std::string err;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // filter pipelining (grid runs): GEMM chunks on `stream`, their all-reduces on `comm_stream`
  cudaStream_t comm_stream = nullptr;
  static constexpr int MAX_CHUNKS = 8;
  cudaEvent_t ev_gemm[MAX_CHUNKS] = {}, ev_comm[2][MAX_CHUNKS] = {}, ev_join = nullptr;
  bool broken = false;
  // f1: fused all-reduce over peer memory (peer.cu)
  struct Peer {
    bool ready = false, failed = false;
    chase::DBuf stage, ctr, flag, xbuf;
    unsigned* done_local = nullptr;
    unsigned* err = nullptr;              // device view of err_host (mapped pinned memory)
    volatile unsigned* err_host = nullptr;  // set by the wait kernel on timeout; read between steps
    unsigned expected = 0;
    chase::PeerRed row, col;
    bool c64_ready = false;
    float* c64w_row[chase::kMaxPeers] = {};   // row peers' c64 W-layout format buffers
    float* c64v_col[chase::kMaxPeers] = {};   // column peers' c64 V-layout format buffers
    std::vector<void*> opened;
  } peer;
};

namespace chase {

// complex (3M / 4M) or real GEMM by the handle's dtype, on the handle's stream
void gemm(chase_handle* h, const ZgemmDesc& d);
// one fused distributed recurrence step (a2/a3 or a4/a5); see chase.h chase_hemm_step
void hemm_step(chase_handle* h, int dir, const void* H, int64_t ldh, const void* X, int64_t ldx,
               void* Y, int64_t ldy, int ncols, double alpha, double beta, double gamma);
// V <- Filter(...) (a1-a5)
int64_t filter(chase_handle* h, const void* H, int64_t ldh, void* V, int64_t ldv, void* W,
               int64_t ldw, int ncols, const int* degrees, double b_sup, double mu_1, double mu_ne);
// in-place sum over a communicator of a column block (rows x ncols, ld)
void allreduce_block(chase_handle* h, const Comm& comm, void* Y, int64_t rows, int64_t ld, int ncols);
void allreduce_doubles(chase_handle* h, const Comm& comm, double* x, size_t n);

struct LanczosOut {
  double b_sup, mu_1, mu_ne, nu;
};
LanczosOut lanczos(chase_handle* h, const void* H, int64_t ldh, int n_e);

void random_block(chase_handle* h, void* V, int64_t ldv, int64_t rows, int64_t grow0, int col0,
                  int ncols, uint64_t seed, uint32_t stream_id, bool c64_out = false);

// complex-single (c64) path: tcgen05 3xTF32 fused step and filter (c64.cu)
void allreduce_c64(chase_handle* h, const Comm& comm, void* Y, int64_t rows, int64_t ld, int ncols);
void c64_hemm_step(chase_handle* h, int dir, const void* H, int64_t ldh, const void* X, int64_t ldx, void* Y,
                   int64_t ldy, int ncols, double alpha, double beta, double gamma);
int64_t c64_filter(chase_handle* h, const void* H, int64_t ldh, void* V, int64_t ldv, int ncols, const int* degrees,
                   double b_sup, double mu_1, double mu_ne);
// f4: complex64 shadow (ld p) of a complex128 shard, rebuilt when H / ldh change
const void* c64_shadow(chase_handle* h, const void* H, int64_t ldh);
// rank-local argument checks of a complex-single call (alignment, ld, width); throws UsageError
void c64_check_call(chase_handle* h, const void* H, int64_t ldh, int ncols);
// H_lo of the shard (validates the c64 layout; recomputed when H / ldh change)
const void* c64_hlo(chase_handle* h, const void* H, int64_t ldh);
// mixed solve (c64 shard, complex128 iteration): filter / HX on complex128 blocks, and conversions
int64_t c64_filter_mixed(chase_handle* h, const void* H, int64_t ldh, double2* V, int64_t ldv, int ncols,
                         const int* degrees, double b_sup, double mu_1, double mu_ne);
void c64_forward_mixed(chase_handle* h, const void* H, int64_t ldh, const double2* X, int64_t ldx, double2* Y,
                       int64_t ldy, int ncols);
void c64_convert(void* dst, int64_t ldd, bool dst_c128, const void* src, int64_t lds, int64_t rows, int cols,
                 cudaStream_t st);

// f1 (peer.cu): set up / use the fused peer all-reduce of the filter steps
bool peer_reduce_ready(chase_handle* h);
bool peer_c64_ready(chase_handle* h);
const PeerRed* peer_red_for(chase_handle* h, int dir, const void* Y);
void peer_wait(chase_handle* h, int tiles);
void peer_check(chase_handle* h);
void peer_release(chase_handle* h);
// f4 (ozaki.cu): one local fused step with the complex products emulated on INT8 tensor cores
void ozaki_step(chase_handle* h, const ZgemmDesc& d);
// a general C = alpha op(A) B + beta C on the emulation (no shift, no triangular B, no fused reduce)
void ozaki_gemm(chase_handle* h, const ZgemmDesc& d);
void ozaki_release(chase_handle* h);
// tile count of one fused step fits the arrival counters (else the step all-reduces with NCCL)
bool peer_tiles_fit(int tiles);
// barrier over the world before a fused filter (ranks enter within the peer timeout of each other)
void peer_enter(chase_handle* h);
// throws PeerTimeout if a wait kernel has timed out (host read of mapped memory, no sync)
void peer_poll(chase_handle* h);
// synchronise the library stream, polling the communicators' asynchronous errors (and the
// comm_timeout option) while waiting
void sync_stream(chase_handle* h, cudaStream_t st);

chase_status solve(chase_handle* h, const void* H, int64_t ldh, int nev, int nex, int deg,
                   double tol, double* ritz_values, void* ritz_vectors, int64_t ldv,
                   chase_report* rep);

}  // namespace chase
