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
#include <cstdio>
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
      atomicExch(err, 1u);
      return;
    }
    __nanosleep(200);
  }
}

struct Handles {
  cudaIpcMemHandle_t stage, vec, ctr;
};

// all-gather `mine` over `comm` (size n) -> out[n]
void gather_handles(chase_handle* h, ncclComm_t comm, int n, const Handles& mine, std::vector<Handles>& out) {
  out.assign(n, Handles{});
  void* d = nullptr;
  CHASE_CUDA(cudaMalloc(&d, sizeof(Handles) * (n + 1)));
  CHASE_CUDA(cudaMemcpyAsync(d, &mine, sizeof(Handles), cudaMemcpyHostToDevice, h->stream));
  CHASE_NCCL(ncclAllGather(d, reinterpret_cast<char*>(d) + sizeof(Handles), sizeof(Handles), ncclUint8, comm,
                           h->stream));
  CHASE_CUDA(cudaMemcpyAsync(out.data(), reinterpret_cast<char*>(d) + sizeof(Handles), sizeof(Handles) * n,
                             cudaMemcpyDeviceToHost, h->stream));
  CHASE_CUDA(cudaStreamSynchronize(h->stream));
  cudaFree(d);
}

void* open_peer(chase_handle* h, const cudaIpcMemHandle_t& hd) {
  void* p = nullptr;
  CHASE_CUDA(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
  h->peer.opened.push_back(p);
  return p;
}
}  // namespace

// every rank's local success flag, min over the world (collective); false if any rank failed
static bool all_ok(chase_handle* h, bool ok) {
  h->peer.flag.alloc(sizeof(int));
  int v = ok ? 1 : 0;
  CHASE_CUDA(cudaMemcpyAsync(h->peer.flag.p, &v, sizeof(int), cudaMemcpyHostToDevice, h->stream));
  CHASE_NCCL(ncclAllReduce(h->peer.flag.p, h->peer.flag.p, 1, ncclInt32, ncclMin, h->world, h->stream));
  CHASE_CUDA(cudaMemcpyAsync(&v, h->peer.flag.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CHASE_CUDA(cudaStreamSynchronize(h->stream));
  return v != 0;
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
  if (h->world_size <= 1 || !h->world || (g.r <= 1 && g.c <= 1)) return false;
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
    h->peer.err = base + 2 * kCtrPerComm + 32;
    CHASE_CUDA(cudaIpcGetMemHandle(&row_mine.stage, h->peer.stage.p));
    CHASE_CUDA(cudaIpcGetMemHandle(&row_mine.ctr, h->peer.ctr.p));
    col_mine = row_mine;
    CHASE_CUDA(cudaIpcGetMemHandle(&row_mine.vec, h->W.p));      // row comm sums W-layout blocks
    CHASE_CUDA(cudaIpcGetMemHandle(&col_mine.vec, h->V.p));      // column comm sums V-layout blocks
  } catch (const std::exception&) {
    cudaGetLastError();
    ok = false;
  }
  std::vector<Handles> rows_h, cols_h;
  if (g.c > 1) gather_handles(h, h->rowc, g.c, row_mine, rows_h);
  if (g.r > 1) gather_handles(h, h->colc, g.r, col_mine, cols_h);
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
        pr.stage[r] = reinterpret_cast<double2*>(open_peer(h, hs[r].stage));
        pr.out[r] = reinterpret_cast<double2*>(open_peer(h, hs[r].vec));
        ctrs[r] = reinterpret_cast<unsigned*>(open_peer(h, hs[r].ctr));
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
  struct H2 { cudaIpcMemHandle_t buf; } mine_r{}, mine_c{};
  CHASE_CUDA(cudaIpcGetMemHandle(&mine_r.buf, h->c64w.p));
  CHASE_CUDA(cudaIpcGetMemHandle(&mine_c.buf, h->c64v.p));
  bool ok = true;
  auto xchg = [&](ncclComm_t comm, int n, int me, const H2& mine, float** out, void* own) {
    std::vector<H2> all(n);
    void* d = nullptr;
    CHASE_CUDA(cudaMalloc(&d, sizeof(H2) * (n + 1)));
    CHASE_CUDA(cudaMemcpyAsync(d, &mine, sizeof(H2), cudaMemcpyHostToDevice, h->stream));
    CHASE_NCCL(ncclAllGather(d, reinterpret_cast<char*>(d) + sizeof(H2), sizeof(H2), ncclUint8, comm, h->stream));
    CHASE_CUDA(cudaMemcpyAsync(all.data(), reinterpret_cast<char*>(d) + sizeof(H2), sizeof(H2) * n,
                               cudaMemcpyDeviceToHost, h->stream));
    CHASE_CUDA(cudaStreamSynchronize(h->stream));
    cudaFree(d);
    try {
      for (int r = 0; r < n; ++r)
        out[r] = r == me ? reinterpret_cast<float*>(own) : reinterpret_cast<float*>(open_peer(h, all[r].buf));
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

void peer_wait(chase_handle* h, int tiles) {
  h->peer.expected += (unsigned)tiles;
  k_wait_done<<<1, 1, 0, h->stream>>>(h->peer.done_local, h->peer.expected, h->peer.err, 20ull * 1000000000ull);
  CHASE_CHECK_LAUNCH();
}

void peer_check(chase_handle* h) {
  if (!h->peer.ready) return;
  unsigned e = 0;
  CHASE_CUDA(cudaMemcpyAsync(&e, h->peer.err, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream));
  CHASE_CUDA(cudaStreamSynchronize(h->stream));
  if (e) {
    h->peer.failed = true;
    throw NcclError("fused peer all-reduce timed out (a peer stopped arriving)");
  }
}

void peer_release(chase_handle* h) {
  for (void* p : h->peer.opened) cudaIpcCloseMemHandle(p);
  h->peer.opened.clear();
  h->peer.stage.release();
  h->peer.ctr.release();
  h->peer.flag.release();
  h->peer.ready = false;
  h->peer.c64_ready = false;
}

}  // namespace chase
