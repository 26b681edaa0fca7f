// C ABI of the ChASE B200 library + the filter driver.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "dense.h"
#include "handle.h"
#include "linalg.h"
#include "rng.cuh"
#include "trace.h"

using namespace chase;

namespace chase {

unsigned long long g_kernel_launches = 0;

// ------------------------------------------------------------------------------ collectives
void allreduce_block(chase_handle* h, const Comm& comm, void* Y, int64_t rows, int64_t ld, int ncols) {
  if (!comm.active() || ncols <= 0 || rows <= 0) return;   // inactive: emulated grid
  const int nd = h->nd();
  comm_allreduce(comm, Y, nd * rows, nd * ld, ncols, DT::F64, Op::Sum, h->stream);
}

void allreduce_doubles(chase_handle* h, const Comm& comm, double* x, size_t n) {
  if (!comm.active() || n == 0) return;
  comm_allreduce(comm, x, (int64_t)n, (int64_t)n, 1, DT::F64, Op::Sum, h->stream);
}

// complex (3M / 4M) or real GEMM by the handle's dtype.  Large long-K plain products of the
// iteration (RR's Q^H (HQ), the CholQR Gram, the CGS projection Y^H V) run on the INT8 emulation as
// well when it is on; triangular products (V R^-1), short-K and small ones stay on DMMA.
void gemm(chase_handle* h, const ZgemmDesc& d) {
  if (!h->c64() && h->opt.fp64_emulation > 0 && !h->oz_off && !h->oz_gemm_off && !d.red && !d.S && !d.b_upper &&
      (double)d.M * d.N * d.K >= h->opt.oz_gemm_min && d.K >= h->opt.oz_gemm_kmin &&
      d.K <= (h->opt.oz_crt ? 131071 : 133143)) {
    // K >= oz_gemm_kmin (12288): each of the 7 slice-product launches per real product
    // read-modify-writes the M x N FP64 accumulator once, a cost the MMAs hide only for long K
    // (measured at 30000 x 3000: Q Z with K = 3000 57 ms emulated vs 25 ms DMMA; the Gram with
    // K = 30000 23 ms vs 37 ms)
    try {
      ozaki_gemm(h, d);
      return;
    } catch (const std::bad_alloc&) {
      // the A operand's slices did not fit: plain GEMMs go back to DMMA, the filter keeps its
      // emulation (ozaki_gemm allocates before it launches anything)
      h->oz_gemm_off = true;
      h->oz_g.slices.release();
      h->oz_g.exps.release();
      h->oz_g.diag.release();
      h->oz_g.src = nullptr;
    }
  }
  if (h->real()) dgemm(d, h->stream);
  else zgemm(d, h->stream);
}

// ------------------------------------------------------------------- fused recurrence step
// Local part of one distributed step (a2 / a4): the GEMM descriptor for this rank's shard.
static ZgemmDesc step_desc(chase_handle* h, int dir, const void* H, int64_t ldh, const void* X, int64_t ldx,
                           void* Y, int64_t ldy, int ncols, double alpha, double beta, double gamma) {
  const Grid& g = h->grid;
  const int64_t r0 = g.rows.start, p = g.rows.len, c0 = g.cols.start, q = g.cols.len;
  ZgemmDesc d;
  d.N = ncols;
  d.A = H; d.lda = ldh;
  d.B = X; d.ldb = ldx;
  d.C = Y; d.ldc = ldy;
  // `largest` solves on -H (ledger #17): alpha((sH) X - gamma X) = (s alpha)(H X - (s gamma) X)
  const double hs = h->opt.largest ? -1.0 : 1.0;
  d.alpha = alpha * hs;
  d.gamma = gamma * hs;
  d.S = X; d.lds = ldx;
  if (dir == 0) {                       // W_i = alpha (H_ij V_j - gamma E_ij V_j) + beta W_i   (Eq. w=av)
    d.M = (int)p; d.K = (int)q; d.conjA = false;
    d.shift_lo = (int)std::max<int64_t>(0, c0 - r0);
    d.shift_hi = (int)std::min<int64_t>(p, c0 + q - r0);
    d.shift_off = r0 - c0;
    d.beta = g.beta_owner_fwd() ? beta : 0.0;
  } else {                              // V_j = alpha (H_ij^H W_i - gamma E_ij^T W_i) + beta V_j (Eq. v=aw)
    d.M = (int)q; d.K = (int)p; d.conjA = true;
    d.shift_lo = (int)std::max<int64_t>(0, r0 - c0);
    d.shift_hi = (int)std::min<int64_t>(q, r0 + p - c0);
    d.shift_off = c0 - r0;
    d.beta = g.beta_owner_bwd() ? beta : 0.0;
  }
  if (gamma == 0.0 || d.shift_lo >= d.shift_hi) { d.S = nullptr; d.shift_lo = d.shift_hi = 0; }
  d.use3m = h->opt.gemm3m;
  return d;
}

// local product of a step: FP64 DMMA GEMM, or (f4, fp64_emulation > 0, complex double) the
// Ozaki-scheme emulation on the INT8 tensor cores (ozaki.cu)
// (default, S = 7).  Falls back to DMMA for good when the slices do not fit in device memory, and
// for K > 133143 (int32-exact accumulation bound; K chunking is not built).
static void step_gemm(chase_handle* h, const ZgemmDesc& d) {
  if (!h->c64() && h->opt.fp64_emulation > 0 && !d.red && !h->oz_off && d.K <= (h->opt.oz_crt ? 131071 : 133143)) {
    try {
      ozaki_step(h, d);
      return;
    } catch (const std::bad_alloc&) {
      // (every emulated product allocates before it launches, and only its own buffers are
      // written before the final combine, so a retry starts clean)
      ozaki_release(h);
      if (h->opt.oz_crt) {               // scheme II's residues (48 B per element) did not fit:
        h->opt.oz_crt = 0;               // the 7-slice scheme (21 B per element)
        try {
          ozaki_step(h, d);
          return;
        } catch (const std::bad_alloc&) {
          ozaki_release(h);
        }
      }
      h->oz_off = true;
    }
  }
  gemm(h, d);
}

void hemm_step(chase_handle* h, int dir, const void* H, int64_t ldh, const void* X, int64_t ldx,
               void* Y, int64_t ldy, int ncols, double alpha, double beta, double gamma) {
  if (ncols <= 0) return;
  const Grid& g = h->grid;
  step_gemm(h, step_desc(h, dir, H, ldh, X, ldx, Y, ldy, ncols, alpha, beta, gamma));
  if (dir == 0)
    allreduce_block(h, h->rowc, Y, g.rows.len, ldy, ncols);     // row communicator
  else
    allreduce_block(h, h->colc, Y, g.cols.len, ldy, ncols);     // column communicator
}

// ------------------------------------------------------------------------ Chebyshev filter
// Scalars (ledger #1): c = (b_sup+mu_ne)/2, e = (b_sup-mu_ne)/2, sigma_1 =
// e/(mu_1-c); k=1: alpha = sigma_1/e, beta = 0; k>=2: sigma_k = 1/(2/sigma_1 - sigma_{k-1}),
// alpha = 2 sigma_k/e, beta = -sigma_{k-1} sigma_k; gamma = c.  Odd steps run forward
// (V-layout -> W-layout), even steps backward (W -> V), so even degrees end in V.
// Step k runs on the active suffix {a : m_a >= k} of the degree-sorted columns.
int64_t filter(chase_handle* h, const void* H, int64_t ldh, void* V, int64_t ldv, void* W,
               int64_t ldw, int ncols, const int* degrees, double b_sup, double mu_1, double mu_ne) {
  if (ncols <= 0) return 0;
  int64_t matvecs = 0;
  for (int a = 0; a < ncols; ++a) {
    if (degrees[a] < 0 || (degrees[a] & 1)) throw UsageError("filter degrees must be even and >= 0");
    if (a > 0 && degrees[a] < degrees[a - 1]) throw UsageError("filter degrees must be sorted ascending");
    matvecs += degrees[a];
  }
  const int kmax = degrees[ncols - 1];
  if (kmax == 0) return 0;
  const double c = 0.5 * (b_sup + mu_ne), e = 0.5 * (b_sup - mu_ne);
  if (!(e > 0.0)) throw UsageError("filter interval is empty (b_sup <= mu_ne)");
  const double sigma1 = e / (mu_1 - c);
  double sigma_prev = sigma1;
  char* Vz = reinterpret_cast<char*>(V);
  char* Wz = reinterpret_cast<char*>(W);
  const int64_t es = (int64_t)h->es();
  const Grid& g = h->grid;
  // Overlap: on a real grid the columns are cut into chunks with fixed absolute
  // boundaries; each chunk's all-reduce runs on the comm stream while the next chunk's GEMM runs,
  // and step k's GEMM on chunk c waits only for step k-1's all-reduce of chunk c (columns are
  // independent through the whole recurrence).
  const bool comm = h->comm_stream && (g.r > 1 || g.c > 1) && h->world.active();
  // Chunking costs GEMM tile/wave efficiency (~1-2 % per extra chunk), so it is only worth it when
  // the all-reduce is a visible fraction of a step: t_comm / t_gemm ~ (16 B/elem / ~600 GB/s) /
  // (8 K flop/elem / ~40 TF/s) ~ 133 / K.  Measured on B200 (2x2 grid, K = 30000) it is 0.4 %, so
  // large shards run one GEMM + one all-reduce per step; small-K shards pipeline.
  const int64_t kmin = std::min(g.rows.len, g.cols.len);
  int nchunks = (comm && 133.0 / (double)kmin > 0.03)
                    ? std::max(1, std::min(chase_handle::MAX_CHUNKS, ncols / 384)) : 1;
  if (comm) {
    if (const char* env = std::getenv("CHASE_FILTER_CHUNKS"))      // testing / tuning override
      nchunks = std::max(1, std::min({chase_handle::MAX_CHUNKS, ncols, std::atoi(env)}));
  }
  // f1: all-reduce inside the GEMM over peer memory (internal V / W buffers only: the peers'
  // replicas are the handles' workspace at the same offsets)
  auto inside = [](const DBuf& b, const void* ptr) {
    const char* c = reinterpret_cast<const char*>(ptr);
    const char* s = reinterpret_cast<const char*>(b.p);
    return b.p && c >= s && c < s + b.bytes;
  };
  // The arrival counters hold kCtrPerComm tiles per communicator: a step with more tiles (the
  // largest is step 1, all columns, on the largest shard of the grid -- the same answer on every
  // rank) all-reduces with NCCL instead.
  const int64_t pmax = (g.N + g.r - 1) / g.r, qmax = (g.N + g.c - 1) / g.c;
  const int max_tiles = h->real() ? std::max(dgemm_tiles((int)pmax, ncols), dgemm_tiles((int)qmax, ncols))
                                  : std::max(zgemm3m_tiles((int)pmax, ncols), zgemm3m_tiles((int)qmax, ncols));
  const bool fused = comm && ldv == g.cols.len && ldw == g.rows.len && inside(h->V, V) && inside(h->W, W) &&
                     h->opt.fp64_emulation == 0 && peer_tiles_fit(max_tiles) && peer_reduce_ready(h);
  if (fused) {
    nchunks = 1;
    peer_enter(h);                // every rank has entered this filter call (peer-timeout skew guard)
  }
  std::vector<int> bnd(nchunks + 1);
  for (int c = 0; c <= nchunks; ++c) bnd[c] = (int)((int64_t)ncols * c / nchunks);
  bool rec[2][chase_handle::MAX_CHUNKS] = {};
  int first = 0;
  for (int k = 1; k <= kmax; ++k) {
    while (first < ncols && degrees[first] < k) ++first;
    double alpha, beta;
    if (k == 1) {
      alpha = sigma1 / e;
      beta = 0.0;
    } else {
      const double sigma = 1.0 / (2.0 / sigma1 - sigma_prev);
      alpha = 2.0 * sigma / e;
      beta = -sigma_prev * sigma;
      sigma_prev = sigma;
    }
    const int dir = (k & 1) ? 0 : 1;        // odd: forward V -> W; even: backward W -> V
    nvtx_push_step(k, dir, ncols - first);
    struct PopAtEnd { ~PopAtEnd() { nvtx_pop(); } } pop_at_end;
    char* X = dir == 0 ? Vz : Wz;
    char* Y = dir == 0 ? Wz : Vz;
    const int64_t ldx = dir == 0 ? ldv : ldw, ldy = dir == 0 ? ldw : ldv;
    if (!comm) {
      hemm_step(h, dir, H, ldh, X + (int64_t)first * ldx * es, ldx, Y + (int64_t)first * ldy * es, ldy,
                ncols - first, alpha, beta, c);
      continue;
    }
    if (fused) {
      char* Yk = Y + (int64_t)first * ldy * es;
      ZgemmDesc d = step_desc(h, dir, H, ldh, X + (int64_t)first * ldx * es, ldx, Yk, ldy, ncols - first, alpha,
                              beta, c);
      d.red = peer_red_for(h, dir, Yk);
      peer_poll(h);                               // a timed-out wait stops the launches here
      if (d.red) {
        gemm(h, d);
        peer_wait(h, h->real() ? dgemm_tiles(d.M, d.N) : zgemm3m_tiles(d.M, d.N));
      } else {                                   // this direction's communicator has one rank
        gemm(h, d);
      }
      continue;
    }
    const int64_t rows = dir == 0 ? g.rows.len : g.cols.len;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int lo = std::max(first, bnd[ch]), hi = bnd[ch + 1];
      if (lo >= hi) continue;
      if (rec[(k - 1) & 1][ch]) CHASE_CUDA(cudaStreamWaitEvent(h->stream, h->ev_comm[(k - 1) & 1][ch], 0));
      step_gemm(h, step_desc(h, dir, H, ldh, X + (int64_t)lo * ldx * es, ldx, Y + (int64_t)lo * ldy * es, ldy,
                             hi - lo, alpha, beta, c));
      CHASE_CUDA(cudaEventRecord(h->ev_gemm[ch], h->stream));
      CHASE_CUDA(cudaStreamWaitEvent(h->comm_stream, h->ev_gemm[ch], 0));
      cudaStream_t saved = h->stream;
      h->stream = h->comm_stream;               // allreduce_block enqueues on h->stream
      if (dir == 0)
        allreduce_block(h, h->rowc, Y + (int64_t)lo * ldy * es, rows, ldy, hi - lo);
      else
        allreduce_block(h, h->colc, Y + (int64_t)lo * ldy * es, rows, ldy, hi - lo);
      h->stream = saved;
      CHASE_CUDA(cudaEventRecord(h->ev_comm[k & 1][ch], h->comm_stream));
      rec[k & 1][ch] = true;
      rec[(k - 1) & 1][ch] = false;
    }
  }
  if (fused) {
    peer_check(h);
  } else if (comm) {
    CHASE_CUDA(cudaEventRecord(h->ev_join, h->comm_stream));
    CHASE_CUDA(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
  }
  return matvecs;
}

// -------------------------------------------------------------------- random start block
template <class TV>
__global__ void k_random_block(TV* V, int64_t ldv, int64_t rows, int64_t grow0, int col0,
                               int ncols, uint32_t k0, uint32_t k1, uint32_t stream_id) {
  const int64_t total = rows * ncols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rloc = idx % rows;
    const int cl = (int)(idx / rows);
    const uint64_t grow = (uint64_t)(grow0 + rloc);
    const Philox4 o = philox4x32_10((uint32_t)grow, (uint32_t)(grow >> 32), (uint32_t)(col0 + cl),
                                    stream_id, k0, k1);
    V[rloc + (int64_t)cl * ldv].x = philox_unit(o.x[0], o.x[1]);     // complex64: rounded to fp32
    V[rloc + (int64_t)cl * ldv].y = philox_unit(o.x[2], o.x[3]);
  }
}

// real variant: the real part of the same counter-based entry
__global__ void k_random_block_real(double* V, int64_t ldv, int64_t rows, int64_t grow0, int col0, int ncols,
                                    uint32_t k0, uint32_t k1, uint32_t stream_id) {
  const int64_t total = rows * ncols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rloc = idx % rows;
    const int cl = (int)(idx / rows);
    const uint64_t grow = (uint64_t)(grow0 + rloc);
    const Philox4 o = philox4x32_10((uint32_t)grow, (uint32_t)(grow >> 32), (uint32_t)(col0 + cl),
                                    stream_id, k0, k1);
    V[rloc + (int64_t)cl * ldv] = philox_unit(o.x[0], o.x[1]);
  }
}

void random_block(chase_handle* h, void* V, int64_t ldv, int64_t rows, int64_t grow0, int col0,
                  int ncols, uint64_t seed, uint32_t stream_id, bool c64_out) {
  if (rows <= 0 || ncols <= 0) return;
  const int64_t total = rows * ncols;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (h->real())
    k_random_block_real<<<blocks, 256, 0, h->stream>>>(reinterpret_cast<double*>(V), ldv, rows, grow0, col0, ncols,
                                                       (uint32_t)seed, (uint32_t)(seed >> 32), stream_id);
  else if (c64_out)
    k_random_block<<<blocks, 256, 0, h->stream>>>(reinterpret_cast<float2*>(V), ldv, rows, grow0, col0, ncols,
                                                  (uint32_t)seed, (uint32_t)(seed >> 32), stream_id);
  else
    k_random_block<<<blocks, 256, 0, h->stream>>>(reinterpret_cast<double2*>(V), ldv, rows, grow0,
                                                  col0, ncols, (uint32_t)seed, (uint32_t)(seed >> 32),
                                                  stream_id);
  CHASE_CHECK_LAUNCH();
}

}  // namespace chase

// ============================================================================== C ABI
namespace {

// Collective status agreement: every rank returns the same status (chase.h "Validation").  A
// broken handle cannot communicate (its communicators were aborted, see fail_hard).
chase_status agree(chase_handle* h, chase_status st) {
  if (!h || h->world_size <= 1 || !h->world.active() || h->broken) return st;
  try {
    h->peer.flag.alloc(sizeof(int));
    int v = (int)st;
    if (h->world.local) {
      v = comm_allreduce_int(h->world, v, Op::Max, h->peer.flag.p, h->stream);
    } else {                       // NCCL: wait with async-error polling (a dead peer -> error)
      CHASE_CUDA(cudaMemcpyAsync(h->peer.flag.p, &v, sizeof(int), cudaMemcpyHostToDevice, h->stream));
      CHASE_NCCL(ncclAllReduce(h->peer.flag.p, h->peer.flag.p, 1, ncclInt32, ncclMax, h->world.nccl, h->stream));
      CHASE_CUDA(cudaMemcpyAsync(&v, h->peer.flag.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
      sync_stream(h, h->stream);
    }
    if (v != (int)st && h->err.empty()) h->err = "another rank failed with status " + std::to_string(v);
    return (chase_status)v;
  } catch (...) {
    h->broken = true;
    return CHASE_E_NCCL;
  }
}

// A CUDA / NCCL failure leaves the handle unusable; its NCCL communicators are aborted so that
// peers blocked in a collective with this rank see an error (ncclCommGetAsyncError, polled by
// sync_stream) instead of waiting forever.
void fail_hard(chase_handle* h) {
  h->broken = true;
  comm_abort(h->world);
  comm_abort(h->rowc);
  comm_abort(h->colc);
}

// Run f() and map exceptions to statuses.  PeerTimeout keeps the communicators usable, so its
// status is still agreed on before the handle is marked unusable.
template <class F>
chase_status run_mapped(chase_handle* h, F&& f, bool& hard, bool& soft_broken) {
  chase_status st = CHASE_OK;
  try {
    CHASE_CUDA(cudaSetDevice(h->device));
    st = f();
  } catch (const UsageError& e) {
    h->err = e.what(); st = CHASE_E_USAGE;
  } catch (const NumericError& e) {
    h->err = e.what(); st = CHASE_E_NUMERIC;
  } catch (const PeerTimeout& e) {
    h->err = e.what(); st = CHASE_E_NCCL; soft_broken = true;
  } catch (const NcclError& e) {
    h->err = e.what(); st = CHASE_E_NCCL; hard = true;
  } catch (const CudaError& e) {
    h->err = e.what(); st = CHASE_E_CUDA; hard = true;
  } catch (const std::bad_alloc&) {
    h->err = "out of memory (device workspace or host)"; st = CHASE_E_NOMEM;
  } catch (const std::exception& e) {
    h->err = e.what(); st = CHASE_E_CUDA; hard = true;
  }
  return st;
}

// Collective calls: validate() runs first and touches no communicator; its status is agreed on
// over the world, so either every rank proceeds to work() (which issues the collectives) or
// every rank returns the same error -- a rank-local argument problem (uneven shards, ld, layout)
// can therefore never leave the other ranks blocked inside a collective.  work()'s status is
// agreed on as well.
template <class V, class F>
chase_status guarded2(chase_handle* h, V&& validate, F&& work) {
  if (!h) return CHASE_E_USAGE;
  if (h->broken) { h->err = "handle is unusable after an earlier CUDA/NCCL error"; return CHASE_E_CUDA; }
  bool hard = false, soft = false;
  chase_status st = run_mapped(h, validate, hard, soft);
  if (hard) { fail_hard(h); return st; }
  st = agree(h, st);
  if (st != CHASE_OK) return st;
  st = run_mapped(h, work, hard, soft);
  if (hard) { fail_hard(h); return st; }
  st = agree(h, st);
  if (soft) h->broken = true;
  return st;
}

// single-phase variant (local calls, and collectives with nothing rank-local to validate)
template <class F>
chase_status guarded(chase_handle* h, F&& f, bool collective = true) {
  if (!h) return CHASE_E_USAGE;
  if (h->broken) { h->err = "handle is unusable after an earlier CUDA/NCCL error"; return CHASE_E_CUDA; }
  bool hard = false, soft = false;
  chase_status st = run_mapped(h, f, hard, soft);
  if (hard) { fail_hard(h); return st; }
  if (collective) st = agree(h, st);
  if (soft) h->broken = true;
  return st;
}

// Derived copies of the caller's shard (Ozaki slices, the c64 lo part, the f4 shadow) are cached
// by pointer only within one API call: the caller may rewrite H, or free it and get the same
// address back for a different matrix, between calls.
void invalidate_shard_caches(chase_handle* h) {
  h->oz_fwd.src = nullptr;
  h->hlo_src = nullptr;
  h->h32_src = nullptr;
}

void order_after_user(chase_handle* h) {
  invalidate_shard_caches(h);
  if (h->user_stream && h->user_stream != h->stream) {
    CHASE_CUDA(cudaEventRecord(h->ev0, h->user_stream));
    CHASE_CUDA(cudaStreamWaitEvent(h->stream, h->ev0, 0));
  }
}

}  // namespace

extern "C" {

unsigned long long chase_kernel_launches(void) { return chase::g_kernel_launches; }

chase_status chase_nccl_unique_id(void* out128) {
  if (!out128) return CHASE_E_USAGE;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return CHASE_E_NCCL;
  std::memcpy(out128, &id, sizeof(id));
  return CHASE_OK;
}

const char* chase_version(void) {
  return "chase-b200 0.3 (sm_100a: FP64 via Ozaki INT8 tcgen05 emulation or DMMA, tcgen05 3xTF32 complex single, NCCL / fused NVLink all-reduce)";
}

const char* chase_last_error(const chase_handle* h) { return h ? h->err.c_str() : "null handle"; }

// true for host memory (pinned or pageable), false for device / managed memory
static bool host_ptr(const void* ptr) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}

// Auto grid (ledger #19): r x c = world, r <= c, |r - c| minimal.
static void auto_grid(int ws, int& r, int& c) {
  r = 1;
  for (int d = 1; (int64_t)d * d <= ws; ++d)
    if (ws % d == 0) r = d;
  c = ws / r;
}

// complex single: the TMA operand views need every shard of the grid to have q % 4 == 0 and even
// p; decided from the global N / r / c so that every rank reaches the same answer
static bool c64_grid_layout_ok(const Grid& g) {
  for (int i = 0; i < g.r; ++i)
    if (block_range(g.N, g.r, i).len % 2 != 0) return false;
  for (int j = 0; j < g.c; ++j)
    if (block_range(g.N, g.c, j).len % 4 != 0) return false;
  return true;
}

chase_status chase_init(chase_handle** out, const chase_init_args* a) {
  if (!out || !a) return CHASE_E_USAGE;
  *out = nullptr;
  chase_handle* h = new chase_handle();
  try {
    if (a->dtype != CHASE_C128 && a->dtype != CHASE_R64 && a->dtype != CHASE_C64)
      throw UsageError("dtype must be CHASE_C128, CHASE_C64 or CHASE_R64");
    h->dtype = a->dtype;
    if (a->N <= 0 || a->nev_max <= 0 || a->nex_max <= 0 || a->nev_max + (int64_t)a->nex_max > a->N)
      throw UsageError("invalid N / nev_max / nex_max");
    int ws = std::max(1, a->world_size);
    int r = a->grid_rows, c = a->grid_cols;
    if (r <= 0 || c <= 0) auto_grid(ws, r, c);
    // world_size == 1 with r*c > 1: emulated-grid mode (one shard of an r x c grid, no
    // communicators; collective sums are left to the caller).  Used by single-GPU grid tests.
    if (r * c != ws && ws != 1) throw UsageError("grid_rows * grid_cols must equal world_size");
    if (a->rank < 0 || a->rank >= r * c) throw UsageError("rank out of range");
    if (a->N < std::max(r, c)) throw UsageError("N must be >= max(r, c)");
    if (a->colocated && ws <= 1) throw UsageError("colocated needs world_size > 1");
    h->world_size = ws;
    h->device = a->cuda_device;
    h->colocated = a->colocated != 0;
    CHASE_CUDA(cudaSetDevice(h->device));
    int major = 0;
    CHASE_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, h->device));
    if (major < 10) throw UsageError("this library requires an sm_100a (B200) device");
    h->grid.setup(a->N, r, c, a->rank);
    if (h->c64() && !c64_grid_layout_ok(h->grid))
      throw UsageError("CHASE_C64 needs every shard of the grid to have q % 4 == 0 and even p");
    CHASE_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    // NULL means the caller's work is on the legacy default stream; the library stream is
    // non-blocking, so ordering against it must be explicit (an event on cudaStreamLegacy).
    h->user_stream = a->cuda_stream ? reinterpret_cast<cudaStream_t>(a->cuda_stream) : cudaStreamLegacy;
    CHASE_CUDA(cudaEventCreate(&h->ev0));
    CHASE_CUDA(cudaEventCreate(&h->ev1));
    if (ws > 1) {
      if (!a->nccl_unique_id) throw UsageError("nccl_unique_id required when world_size > 1");
      h->world.size = ws;
      h->world.rank = a->rank;
      h->rowc.size = c;                 // row comm i: colour i, key j
      h->rowc.rank = h->grid.j;
      h->colc.size = r;                 // column comm j: colour j, key i
      h->colc.rank = h->grid.i;
      if (h->colocated) {
        // in-process rendezvous keyed by the 128-byte id (comm.h)
        std::string key(reinterpret_cast<const char*>(a->nccl_unique_id), 128);
        const std::string kw = key + "/world", kr = key + "/row" + std::to_string(h->grid.i),
                          kc = key + "/col" + std::to_string(h->grid.j);
        h->world.local = local_join(kw.data(), kw.size(), ws, a->rank);
        h->rowc.local = local_join(kr.data(), kr.size(), c, h->grid.j);
        h->colc.local = local_join(kc.data(), kc.size(), r, h->grid.i);
      } else {
        ncclUniqueId id;
        std::memcpy(&id, a->nccl_unique_id, sizeof(id));
        CHASE_NCCL(ncclCommInitRank(&h->world.nccl, ws, id, a->rank));
        CHASE_NCCL(ncclCommSplit(h->world.nccl, h->grid.i, h->grid.j, &h->rowc.nccl, nullptr));   // row comm i
        CHASE_NCCL(ncclCommSplit(h->world.nccl, h->grid.j, h->grid.i, &h->colc.nccl, nullptr));   // column comm j
      }
      CHASE_CUDA(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
      for (int k = 0; k < chase_handle::MAX_CHUNKS; ++k) {
        CHASE_CUDA(cudaEventCreateWithFlags(&h->ev_gemm[k], cudaEventDisableTiming));
        CHASE_CUDA(cudaEventCreateWithFlags(&h->ev_comm[0][k], cudaEventDisableTiming));
        CHASE_CUDA(cudaEventCreateWithFlags(&h->ev_comm[1][k], cudaEventDisableTiming));
      }
      CHASE_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    }
    h->n_e_max = a->nev_max + a->nex_max;
    // Workspace: V, V2 (V-layout q x n_e), W, HV (W-layout p x n_e), n_e x n_e
    // matrices, allocated here; the memory check (P:507-531 analogue) also counts what is
    // allocated on first use: Lanczos Krylov basis (N x L x (m+1) + N x L), the RR eigensolver's
    // padded n_e x n_e pair, the fused-reduce staging buffer (grids), and for complex single the
    // shard's 3xTF32 lo part and the operand formats.
    const int64_t p = h->grid.rows.len, q = h->grid.cols.len, ne = h->n_e_max, N = a->N;
    const int64_t np = (ne + 63) / 64 * 64;
    size_t need = 16 * (size_t)(2 * q * ne + 2 * p * ne + 3 * ne * ne);
    need += 16 * (size_t)N * 4 * 27 + 2 * 16 * (size_t)np * np;
    if (ws > 1) need += 16 * (size_t)std::max(p, q) * ne;
    if (h->c64()) need += 8 * (size_t)p * q + 16 * (size_t)q * ne + 32 * (size_t)p * ne;
    size_t fre = 0, tot = 0;
    CHASE_CUDA(cudaMemGetInfo(&fre, &tot));
    if (need > fre) throw std::bad_alloc();
    h->V.alloc(16 * (size_t)q * ne);
    h->V2.alloc(16 * (size_t)q * ne);
    h->W.alloc(16 * (size_t)p * ne);
    h->HV.alloc(16 * (size_t)p * ne);
    h->G.alloc(16 * (size_t)ne * ne);
    h->G2.alloc(16 * (size_t)ne * ne);
    h->Z.alloc(16 * (size_t)ne * ne);
  } catch (const UsageError& e) {
    h->err = e.what();
    *out = h;
    return CHASE_E_USAGE;
  } catch (const std::bad_alloc&) {
    h->err = "workspace does not fit in device memory";
    *out = h;
    return CHASE_E_NOMEM;
  } catch (const NcclError& e) {
    h->err = e.what();
    *out = h;
    return CHASE_E_NCCL;
  } catch (const std::exception& e) {
    h->err = e.what();
    *out = h;
    return CHASE_E_CUDA;
  }
  *out = h;
  return CHASE_OK;
}

chase_status chase_get_option(chase_handle* h, const char* key, double* value) {
  return guarded(h, [&]() {
    if (!key || !value) throw UsageError("null option key or value pointer");
    std::string k(key);
    double v;
    if (k == "ozaki_scheme")             // the FP64 product path in effect (after any memory fallback)
      v = (h->c64() || h->opt.fp64_emulation <= 0 || h->oz_off) ? 0.0 : (h->opt.oz_crt ? 2.0 : 1.0);
    else if (k == "oz_crt") v = h->opt.oz_crt;
    else if (k == "fp64_emulation") v = h->opt.fp64_emulation;
    else if (k == "deg_max") v = h->opt.deg_max;
    else if (k == "deg_extra") v = h->opt.deg_extra;
    else if (k == "max_iter") v = h->opt.max_iter;
    else if (k == "mixed_filter") v = h->opt.mixed_filter;
    else throw UsageError("unknown option " + k);
    *value = v;
    return CHASE_OK;
  }, false);
}

chase_status chase_set_option(chase_handle* h, const char* key, double v) {
  return guarded(h, [&]() {
    if (!key) throw UsageError("null option key");
    std::string k(key);
    if (k == "deg_max") { if (v < 2) throw UsageError("deg_max >= 2"); h->opt.deg_max = (int)v; }
    else if (k == "oz_crt") { h->opt.oz_crt = v != 0.0 ? 1 : 0; invalidate_shard_caches(h); }
    else if (k == "oz_gemm_kmin") { if (v < 0) throw UsageError("oz_gemm_kmin >= 0"); h->opt.oz_gemm_kmin = v; }
    else if (k == "oz_gemm_min") { if (v < 0) throw UsageError("oz_gemm_min >= 0"); h->opt.oz_gemm_min = v; }
    else if (k == "deg_extra") { if (v < 0) throw UsageError("deg_extra >= 0"); h->opt.deg_extra = (int)v; }
    else if (k == "max_iter") { if (v < 0) throw UsageError("max_iter >= 0 (0 = auto)"); h->opt.max_iter = (int)v; }
    else if (k == "stall_iter") { if (v < 1) throw UsageError("stall_iter >= 1"); h->opt.stall_iter = (int)v; }
    else if (k == "lanczos_steps") { if (v < 2) throw UsageError("lanczos_steps >= 2"); h->opt.lanczos_steps = (int)v; }
    else if (k == "lanczos_runs") { if (v < 1) throw UsageError("lanczos_runs >= 1"); h->opt.lanczos_runs = (int)v; }
    else if (k == "seed_v") h->opt.seed_v = (uint64_t)v;
    else if (k == "seed_lanczos") h->opt.seed_lanczos = (uint64_t)v;
    else if (k == "largest") h->opt.largest = v != 0.0;
    else if (k == "approx") h->opt.approx = v != 0.0;
    else if (k == "gemm3m") h->opt.gemm3m = v != 0.0;
    else if (k == "mixed_filter") h->opt.mixed_filter = v;
    else if (k == "fused_reduce") h->opt.fused_reduce = v != 0.0;
    else if (k == "fused_reduce_c64") h->opt.fused_reduce_c64 = v != 0.0;
    else if (k == "peer_timeout") { if (!(v > 0)) throw UsageError("peer_timeout > 0"); h->opt.peer_timeout = v; }
    else if (k == "fp64_emulation") {
      if (v != 0 && (v < 3 || v > 8)) throw UsageError("fp64_emulation: 0 (off) or 3..8 slices");
      h->opt.fp64_emulation = (int)v;
    }
    else if (k == "comm_timeout") { if (v < 0) throw UsageError("comm_timeout >= 0"); h->opt.comm_timeout = v; }
    else throw UsageError("unknown option " + k);
    return CHASE_OK;
  }, false);
}

chase_status chase_local_layout(const chase_handle* h, int64_t* row0, int64_t* p, int64_t* col0,
                                int64_t* q) {
  if (!h) return CHASE_E_USAGE;
  if (row0) *row0 = h->grid.rows.start;
  if (p) *p = h->grid.rows.len;
  if (col0) *col0 = h->grid.cols.start;
  if (q) *q = h->grid.cols.len;
  return CHASE_OK;
}

chase_status chase_hemm_step(chase_handle* h, int32_t dir, const void* H, int64_t ldh,
                             const void* X, int64_t ldx, void* Y, int64_t ldy, int32_t ncols,
                             double alpha, double beta, double gamma) {
  return guarded2(h, [&]() {
    const int64_t p = h->grid.rows.len, q = h->grid.cols.len;
    if (dir != 0 && dir != 1) throw UsageError("dir must be 0 or 1");
    if (ncols == 0) return CHASE_OK;   // empty block: no-op, pointers may be NULL
    if (!H || !X || !Y || ncols < 0 || ldh < p) throw UsageError("bad pointers / sizes");
    if (ldx < (dir == 0 ? q : p) || ldy < (dir == 0 ? p : q)) throw UsageError("bad leading dimension");
    if (h->c64()) c64_check_call(h, H, ldh, ncols);
    return CHASE_OK;
  }, [&]() {
    if (ncols == 0) return CHASE_OK;
    order_after_user(h);
    if (h->c64())
      c64_hemm_step(h, dir, H, ldh, X, ldx, Y, ldy, ncols, alpha, beta, gamma);
    else
      hemm_step(h, dir, H, ldh, X, ldx, Y, ldy, ncols, alpha, beta, gamma);
    sync_stream(h, h->stream);
    return CHASE_OK;
  });
}

chase_status chase_filter(chase_handle* h, const void* H, int64_t ldh, void* V, int64_t ldv,
                          void* W, int64_t ldw, int32_t ncols, const int32_t* degrees,
                          double b_sup, double mu_1, double mu_ne, int64_t* matvecs) {
  if (matvecs) *matvecs = 0;
  return guarded2(h, [&]() {
    const int64_t p = h->grid.rows.len, q = h->grid.cols.len;
    if (ncols == 0) return CHASE_OK;   // empty block: no-op, pointers may be NULL
    if (!H || !V || !W || ncols < 0 || !degrees) throw UsageError("bad pointers");
    if (ldh < p || ldv < q || ldw < p) throw UsageError("bad leading dimension");
    for (int a = 0; a < ncols; ++a) {
      if (degrees[a] < 0 || (degrees[a] & 1)) throw UsageError("filter degrees must be even and >= 0");
      if (a > 0 && degrees[a] < degrees[a - 1]) throw UsageError("filter degrees must be sorted ascending");
    }
    if (degrees[ncols - 1] > 0 && !(b_sup > mu_ne)) throw UsageError("filter interval is empty (b_sup <= mu_ne)");
    if (h->c64()) c64_check_call(h, H, ldh, ncols);
    return CHASE_OK;
  }, [&]() {
    if (ncols == 0) return CHASE_OK;
    const int64_t p = h->grid.rows.len, q = h->grid.cols.len;
    order_after_user(h);
    const Grid& g = h->grid;
    // f1 runs on the library's V / W workspace (the peers' replicas): stage the caller's block
    const bool staged = !h->c64() && h->opt.fused_reduce && (h->real() || h->opt.gemm3m) && h->world_size > 1 &&
                        (g.r > 1 || g.c > 1) && ncols > 0 && ncols <= h->n_e_max;
    int64_t mv;
    if (h->c64()) {
      mv = c64_filter(h, H, ldh, V, ldv, ncols, degrees, b_sup, mu_1, mu_ne);
    } else if (staged && h->real()) {
      copy2d<double>(h->V.p, q, V, ldv, q, ncols, h->stream);
      mv = filter(h, H, ldh, h->V.p, q, h->W.p, p, ncols, degrees, b_sup, mu_1, mu_ne);
      copy2d<double>(V, ldv, h->V.p, q, q, ncols, h->stream);
    } else if (staged) {
      copy2d<double2>(h->V.p, q, V, ldv, q, ncols, h->stream);
      mv = filter(h, H, ldh, h->V.p, q, h->W.p, p, ncols, degrees, b_sup, mu_1, mu_ne);
      copy2d<double2>(V, ldv, h->V.p, q, q, ncols, h->stream);
    } else {
      mv = filter(h, H, ldh, V, ldv, W, ldw, ncols, degrees, b_sup, mu_1, mu_ne);
    }
    sync_stream(h, h->stream);
    if (matvecs) *matvecs = mv;
    return CHASE_OK;
  });
}

chase_status chase_lanczos(chase_handle* h, const void* H, int64_t ldh, int32_t n_e, double* b_sup,
                           double* mu_1, double* mu_ne, double* nu) {
  return guarded2(h, [&]() {
    if (!H || ldh < h->grid.rows.len || n_e <= 0 || n_e > h->grid.N) throw UsageError("bad arguments");
    return CHASE_OK;
  }, [&]() {
    order_after_user(h);
    LanczosOut o = lanczos(h, H, ldh, n_e);
    if (b_sup) *b_sup = o.b_sup;
    if (mu_1) *mu_1 = o.mu_1;
    if (mu_ne) *mu_ne = o.mu_ne;
    if (nu) *nu = o.nu;
    return CHASE_OK;
  });
}

chase_status chase_random_block(chase_handle* h, void* V, int64_t ldv, int32_t col0, int32_t ncols,
                                uint64_t seed, uint32_t stream) {
  return guarded(h, [&]() {
    if (ncols == 0) return CHASE_OK;   // empty block: no-op, V may be NULL
    if (!V || ldv < h->grid.cols.len || ncols < 0) throw UsageError("bad arguments");
    order_after_user(h);
    random_block(h, V, ldv, h->grid.cols.len, h->grid.cols.start, col0, ncols, seed, stream, h->c64());
    sync_stream(h, h->stream);
    return CHASE_OK;
  }, false);
}

chase_status chase_solve(chase_handle* h, const void* H, int64_t ldh, int64_t N, int32_t nev,
                         int32_t nex, int32_t deg, double tol, double* ritz_values,
                         void* ritz_vectors, int64_t ldv, chase_report* report) {
  return guarded2(h, [&]() {
    if (N != h->grid.N) throw UsageError("N differs from chase_init");
    if (!(nev > 0 && nex > 0 && (int64_t)nev + nex <= N && tol > 0 && deg >= 1))
      throw UsageError("invalid nev / nex / tol / deg (S:407)");
    if (nev + nex > h->n_e_max) throw UsageError("nev + nex exceeds nev_max + nex_max of chase_init");
    if (!H || ldh < h->grid.rows.len || !ritz_values || !ritz_vectors || ldv < h->grid.cols.len)
      throw UsageError("bad pointers / leading dimensions");
    if (h->c64()) c64_check_call(h, host_ptr(H) ? nullptr : H, host_ptr(H) ? 0 : ldh, nev + nex);
    if (h->dtype == CHASE_C128 && h->opt.mixed_filter > 0.0) {
      if (!c64_grid_layout_ok(h->grid))
        throw UsageError("mixed_filter needs every shard of the grid to have q % 4 == 0 and even p");
    }
    return CHASE_OK;
  }, [&]() {
    order_after_user(h);
    // Host buffers (pinned or pageable) are accepted for the shard and the vectors: the shard is
    // copied into a library-owned device buffer (ld p) and the vectors staged through one, inside
    // this call -- the end-to-end path of a caller whose H lives in host memory.
    const int64_t p = h->grid.rows.len, q = h->grid.cols.len;
    const size_t es = h->es();
    const void* Hd = H;
    int64_t ldhd = ldh;
    if (host_ptr(H)) {
      h->Hstage.alloc(es * (size_t)p * q);
      CHASE_CUDA(cudaMemcpy2DAsync(h->Hstage.p, es * p, H, es * ldh, es * p, q, cudaMemcpyHostToDevice, h->stream));
      Hd = h->Hstage.p;
      ldhd = p;
      h->hlo_src = nullptr;            // derived copies of the shard are keyed by pointer: rebuild
      h->h32_src = nullptr;
    }
    void* Vd = ritz_vectors;
    int64_t ldvd = ldv;
    const bool vhost = host_ptr(ritz_vectors);
    if (vhost) {
      h->Vstage.alloc(es * (size_t)q * (nev + nex));
      Vd = h->Vstage.p;
      ldvd = q;
      if (h->opt.approx)
        CHASE_CUDA(cudaMemcpy2DAsync(Vd, es * q, ritz_vectors, es * ldv, es * q, nev + nex, cudaMemcpyHostToDevice,
                                     h->stream));
    }
    const chase_status st = solve(h, Hd, ldhd, nev, nex, deg, tol, ritz_values, Vd, ldvd, report);
    if (vhost) {
      CHASE_CUDA(cudaMemcpy2DAsync(ritz_vectors, es * ldv, Vd, es * q, es * q, nev, cudaMemcpyDeviceToHost, h->stream));
      sync_stream(h, h->stream);
    }
    return st;
  });
}

chase_status chase_heev(chase_handle* h, void* G, int64_t ld, int32_t n, double* theta, void* Z, int64_t ldz,
                        int32_t* sweeps) {
  return guarded(h, [&]() {
    if (!G || !theta || !Z || n <= 0 || ld < n || ldz < n) throw UsageError("bad arguments");
    order_after_user(h);
    const int sw = heev_jacobi(G, ld, n, theta, Z, ldz, h->stream, &h->jacobi);
    sync_stream(h, h->stream);
    if (sweeps) *sweeps = sw;
    return CHASE_OK;
  }, false);
}

chase_status chase_finalize(chase_handle* h) {
  if (!h) return CHASE_E_USAGE;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  chase::peer_release(h);
  chase::ozaki_release(h);
  for (chase::DBuf* b : {&h->V, &h->W, &h->HV, &h->V2, &h->G, &h->G2, &h->Z, &h->scratch, &h->red, &h->lz, &h->Hlo,
                         &h->c64v, &h->c64w, &h->H32, &h->Hstage, &h->Vstage})
    b->release();
  heev_work_release(h->jacobi);
  h->jacobi = nullptr;
  comm_destroy(h->rowc);
  comm_destroy(h->colc);
  comm_destroy(h->world);
  if (h->comm_stream) cudaStreamSynchronize(h->comm_stream);
  for (int c = 0; c < chase_handle::MAX_CHUNKS; ++c) {
    if (h->ev_gemm[c]) cudaEventDestroy(h->ev_gemm[c]);
    if (h->ev_comm[0][c]) cudaEventDestroy(h->ev_comm[0][c]);
    if (h->ev_comm[1][c]) cudaEventDestroy(h->ev_comm[1][c]);
  }
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return CHASE_OK;
}

}  // extern "C"
