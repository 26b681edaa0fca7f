// f1: the fused steps' all-reduce over peer memory instead of NCCL.
//
// Setup (once per handle, collective over the row and column communicators): a staging buffer
// (16 B x max(p, q) x n_e), tile-arrival counters and a completion counter are allocated; their
// CUDA IPC handles, and those of the V / W workspace replicas, are all-gathered over each
// communicator (ncclAllGather of the 64-byte handles) and opened, so every rank holds device
// pointers to its row peers' W and staging buffers and its column peers' V and staging buffers.
// NVLink5 / NVSwitch carries the peer loads and stores issued by the GEMM epilogue
// (zgemm3m.cuh).  After each fused step a one-thread kernel waits on the local completion
// counter, which the reducers bump once per tile, so the next step reads a complete replica.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <vector>
#include "handle.h"

namespace chase {

namespace {
constexpr int kCtrPerComm = 1 << 17;          // tile counters per communicator (> max tiles per step)

__global__ void k_wait_done(const unsigned* done, unsigned target, unsigned* err, unsigned long long timeout_ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
    if ((int)(v - target) >= 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      *reinterpret_cast<volatile unsigned*>(err) = 1u;
      __threadfence_system();
      return;
    }
    __nanosleep(200);
  }
}

struct Handles {
  cudaIpcMemHandle_t stage, vec, ctr;
  void *raw_stage, *raw_vec, *raw_ctr;     // co-located ranks: the device pointers themselves
};

// all-gather `mine` over `comm` -> out[comm.size]
template <class T>
void gather(chase_handle* h, const Comm& comm, const T& mine, std::vector<T>& out) {
  out.assign(comm.size, T{});
  h->peer.xbuf.alloc(sizeof(T) * (comm.size + 1));
  comm_allgather_host(comm, &mine, sizeof(T), out.data(), h->peer.xbuf.p, h->stream);
}

void* open_peer(chase_handle* h, const cudaIpcMemHandle_t& hd, void* raw) {
  if (h->colocated) return raw;            // same process (and device): no IPC mapping needed
  void* p = nullptr;
  CHASE_CUDA(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
  h->peer.opened.push_back(p);
  return p;
}
}  // namespace

// every rank's local success flag, min over the world (collective); false if any rank failed
static bool all_ok(chase_handle* h, bool ok) {
  h->peer.flag.alloc(sizeof(int));
  return comm_allreduce_int(h->world, ok ? 1 : 0, Op::Min, h->peer.flag.p, h->stream) != 0;
}

static void give_up(chase_handle* h, const char* why) {
  for (void* p : h->peer.opened) cudaIpcCloseMemHandle(p);
  h->peer.opened.clear();
  h->peer.failed = true;
  if (std::getenv("CHASE_DEBUG_PEER"))
    std::fprintf(stderr, "[chase] rank %d: fused peer all-reduce unavailable (%s); using NCCL\n", h->grid.rank, why);
}

static bool peer_base_ready(chase_handle* h) {
  const Grid& g = h->grid;
  if (h->peer.failed || !h->opt.fused_reduce) return false;
  if (h->world_size <= 1 || !h->world.active() || (g.r <= 1 && g.c <= 1)) return false;
  if (g.r > kMaxPeers || g.c > kMaxPeers) return false;
  if (h->peer.ready) return true;
  // ---- collective setup (every rank of the grid reaches this point with the same options).  Local
  // failures (no IPC / peer access in this environment, allocation) are agreed on over the world,
  // so either every rank uses the fused path or none does.
  const int64_t p = g.rows.len, q = g.cols.len, ne = h->n_e_max;
  bool ok = true;
  Handles row_mine{}, col_mine{};
  unsigned* base = nullptr;
  try {
    h->peer.stage.alloc(16 * (size_t)std::max(p, q) * ne);
    h->peer.ctr.alloc(sizeof(unsigned) * (2 * (size_t)kCtrPerComm + 64));
    CHASE_CUDA(cudaMemsetAsync(h->peer.ctr.p, 0, h->peer.ctr.bytes, h->stream));
    base = h->peer.ctr.as<unsigned>();
    h->peer.done_local = base + 2 * kCtrPerComm;
    if (!h->peer.err_host) {
      unsigned* hp = nullptr;
      CHASE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hp), 64, cudaHostAllocMapped));
      *hp = 0;
      h->peer.err_host = hp;
      CHASE_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->peer.err), hp, 0));
    }
    if (!h->colocated) {
      CHASE_CUDA(cudaIpcGetMemHandle(&row_mine.stage, h->peer.stage.p));
      CHASE_CUDA(cudaIpcGetMemHandle(&row_mine.ctr, h->peer.ctr.p));
    }
    row_mine.raw_stage = h->peer.stage.p;
    row_mine.raw_ctr = h->peer.ctr.p;
    col_mine = row_mine;
    row_mine.raw_vec = h->W.p;                                   // row comm sums W-layout blocks
    col_mine.raw_vec = h->V.p;                                   // column comm sums V-layout blocks
    if (!h->colocated) {
      CHASE_CUDA(cudaIpcGetMemHandle(&row_mine.vec, h->W.p));
      CHASE_CUDA(cudaIpcGetMemHandle(&col_mine.vec, h->V.p));
    }
  } catch (const std::exception&) {
    cudaGetLastError();
    ok = false;
  }
  std::vector<Handles> rows_h, cols_h;
  if (g.c > 1) gather(h, h->rowc, row_mine, rows_h);
  if (g.r > 1) gather(h, h->colc, col_mine, cols_h);
  if (!all_ok(h, ok)) {
    give_up(h, "setup");
    return false;
  }
  auto fill = [&](PeerRed& pr, int n, int me, const std::vector<Handles>& hs, void* own_vec, int ctr_slot) {
    pr.n = n;
    pr.me = me;
    std::vector<unsigned*> ctrs(n);
    for (int r = 0; r < n; ++r) {
      if (r == me) {
        pr.stage[r] = h->peer.stage.as<double2>();
        pr.out[r] = reinterpret_cast<double2*>(own_vec);
        ctrs[r] = base;
      } else {
        pr.stage[r] = reinterpret_cast<double2*>(open_peer(h, hs[r].stage, hs[r].raw_stage));
        pr.out[r] = reinterpret_cast<double2*>(open_peer(h, hs[r].vec, hs[r].raw_vec));
        ctrs[r] = reinterpret_cast<unsigned*>(open_peer(h, hs[r].ctr, hs[r].raw_ctr));
      }
      pr.done[r] = ctrs[r] + 2 * kCtrPerComm;
    }
    pr.ctr = ctrs[0] + (size_t)ctr_slot * kCtrPerComm;        // owned by comm rank 0
  };
  // rank within the row comm = j (split key j), within the column comm = i (key i)
  try {
    if (g.c > 1) fill(h->peer.row, g.c, g.j, rows_h, h->W.p, 0);
    if (g.r > 1) fill(h->peer.col, g.r, g.i, cols_h, h->V.p, 1);
    CHASE_CUDA(cudaStreamSynchronize(h->stream));
  } catch (const std::exception&) {
    cudaGetLastError();
    ok = false;
  }
  if (!all_ok(h, ok)) {                  // also the barrier: every rank's counters are zeroed
    h->peer.row = PeerRed{};
    h->peer.col = PeerRed{};
    give_up(h, "opening peer memory");
    return false;
  }
  h->peer.expected = 0;
  h->peer.ready = true;
  if (std::getenv("CHASE_DEBUG_PEER"))
    std::fprintf(stderr, "[chase] rank %d: fused peer all-reduce ready (row comm %d, column comm %d)\n", g.rank,
                 h->peer.row.n, h->peer.col.n);
  return true;
}

bool peer_reduce_ready(chase_handle* h) {
  if (h->dtype == CHASE_C128 && !h->opt.gemm3m) return false;     // the 4M kernel has no fused epilogue
  return peer_base_ready(h);
}

// complex single: the replicas are the operand-format buffers c64w (row comm) / c64v (column
// comm); their handles are exchanged once they exist (c64.cu allocates them on first use)
bool peer_c64_ready(chase_handle* h) {
  if (h->real() || !peer_base_ready(h)) return false;
  if (h->peer.c64_ready) return true;
  const Grid& g = h->grid;
  if (!h->c64v.p || !h->c64w.p) throw std::logic_error("peer_c64_ready before the c64 formats exist");
  struct H2 { cudaIpcMemHandle_t buf; void* raw; } mine_r{}, mine_c{};
  if (!h->colocated) {
    CHASE_CUDA(cudaIpcGetMemHandle(&mine_r.buf, h->c64w.p));
    CHASE_CUDA(cudaIpcGetMemHandle(&mine_c.buf, h->c64v.p));
  }
  mine_r.raw = h->c64w.p;
  mine_c.raw = h->c64v.p;
  bool ok = true;
  auto xchg = [&](const Comm& comm, int n, int me, const H2& mine, float** out, void* own) {
    std::vector<H2> all;
    gather(h, comm, mine, all);
    try {
      for (int r = 0; r < n; ++r)
        out[r] = r == me ? reinterpret_cast<float*>(own) : reinterpret_cast<float*>(open_peer(h, all[r].buf, all[r].raw));
    } catch (const std::exception&) {
      cudaGetLastError();
      ok = false;
    }
  };
  if (g.c > 1) xchg(h->rowc, g.c, g.j, mine_r, h->peer.c64w_row, h->c64w.p);
  if (g.r > 1) xchg(h->colc, g.r, g.i, mine_c, h->peer.c64v_col, h->c64v.p);
  if (!all_ok(h, ok)) {
    give_up(h, "opening complex-single peer buffers");
    return false;
  }
  h->peer.c64_ready = true;
  if (std::getenv("CHASE_DEBUG_PEER"))
    std::fprintf(stderr, "[chase] rank %d: fused peer all-reduce ready for complex single\n", g.rank);
  return true;
}

// launch-side helpers for one fused step on the internal buffers: `Y` lies in h->W (dir 0) or h->V
const PeerRed* peer_red_for(chase_handle* h, int dir, const void* Y) {
  PeerRed& pr = dir == 0 ? h->peer.row : h->peer.col;
  if (pr.n <= 1) return nullptr;
  const char* base = reinterpret_cast<const char*>(dir == 0 ? h->W.p : h->V.p);
  pr.off = (reinterpret_cast<const char*>(Y) - base) / (h->real() ? 8 : 16);
  return &pr;
}

bool peer_tiles_fit(int tiles) { return tiles >= 0 && tiles <= kCtrPerComm; }

void peer_enter(chase_handle* h) {
  h->peer.flag.alloc(sizeof(int));
  comm_allreduce_int(h->world, 1, Op::Min, h->peer.flag.p, h->stream);
}

void peer_poll(chase_handle* h) {
  if (h->peer.err_host && *h->peer.err_host) {
    h->peer.failed = true;
    throw PeerTimeout("fused peer all-reduce timed out (a peer stopped arriving)");
  }
}

void peer_wait(chase_handle* h, int tiles) {
  h->peer.expected += (unsigned)tiles;
  if (h->colocated) {
    // co-located ranks share this process (and usually the device): no kernel may spin on a peer
    // whose launch depends on a host thread, so completion is ordered by events -- every rank's
    // fused GEMM of this step (hence every last-arriver reduction) precedes the next step.  The
    // wait kernel below then only checks the counter protocol (it returns at once when it holds).
    comm_event_barrier(h->world, h->stream);
  }
  const double tmo = std::max(0.001, h->opt.peer_timeout);
  k_wait_done<<<1, 1, 0, h->stream>>>(h->peer.done_local, h->peer.expected, h->peer.err,
                                      (unsigned long long)(tmo * 1e9));
  CHASE_CHECK_LAUNCH();
}

void peer_check(chase_handle* h) {
  if (!h->peer.ready) return;
  sync_stream(h, h->stream);
  peer_poll(h);
}

void peer_release(chase_handle* h) {
  for (void* p : h->peer.opened) cudaIpcCloseMemHandle(p);
  h->peer.opened.clear();
  h->peer.stage.release();
  h->peer.ctr.release();
  h->peer.flag.release();
  h->peer.xbuf.release();
  if (h->peer.err_host) cudaFreeHost(const_cast<unsigned*>(h->peer.err_host));
  h->peer.err_host = nullptr;
  h->peer.err = nullptr;
  h->peer.ready = false;
  h->peer.c64_ready = false;
}

void sync_stream(chase_handle* h, cudaStream_t st) {
  const bool poll = h->world.nccl || h->rowc.nccl || h->colc.nccl;
  if (!poll && h->opt.comm_timeout <= 0.0) {
    CHASE_CUDA(cudaStreamSynchronize(st));
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  unsigned spins = 0;
  while (true) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) CHASE_CUDA(e);
    comm_check_async(h->world);
    comm_check_async(h->rowc);
    comm_check_async(h->colc);
    if (h->opt.comm_timeout > 0.0 &&
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > h->opt.comm_timeout)
      throw NcclError("library stream did not complete within comm_timeout (a peer may have failed)");
    if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

}  // namespace chase
