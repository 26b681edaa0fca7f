// Communicator transports (see comm.h): NCCL, or an in-process group of co-located ranks.
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include "handle.h"

namespace chase {

namespace {
constexpr int kMaxLocal = 64;
constexpr double kLocalTimeoutS = 600.0;   // a co-located rank that never arrives -> NcclError

ncclDataType_t nccl_type(DT t) { return t == DT::F64 ? ncclDouble : (t == DT::F32 ? ncclFloat : ncclInt32); }
ncclRedOp_t nccl_op(Op o) { return o == Op::Sum ? ncclSum : (o == Op::Max ? ncclMax : ncclMin); }
size_t dt_bytes(DT t) { return t == DT::F64 ? 8 : 4; }
}  // namespace

struct LocalGroup {
  std::string key;
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  int refs = 0;
  std::vector<void*> ptr;
  std::vector<cudaEvent_t> ev_ready, ev_done;
  std::vector<int> ival;
  std::vector<std::vector<char>> bytes;

  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::duration<double>(kLocalTimeoutS), [&] { return gen != g; }))
      throw NcclError("co-located communicator: a rank did not arrive within " +
                      std::to_string((int)kLocalTimeoutS) + " s");
  }
};

namespace {
std::mutex g_reg_m;
std::map<std::string, LocalGroup*> g_reg;

template <class T>
struct PtrTable {
  T* p[kMaxLocal];
};

template <class T, int OP>
__device__ inline T red_op(T a, T b) {
  if constexpr (OP == 0) return a + b;
  else if constexpr (OP == 1) return a > b ? a : b;
  else return a < b ? a : b;
}

// rank-ordered reduction of elements [lo, hi) of a (rows x ncols, ld) block over n replicas; the
// result is stored into every replica
template <class T, int OP>
__global__ void k_local_allreduce(PtrTable<T> t, int n, int64_t rows, int64_t ld, int64_t lo, int64_t hi) {
  for (int64_t idx = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < hi;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t off = (idx % rows) + (idx / rows) * ld;
    T s = t.p[0][off];
    for (int k = 1; k < n; ++k) s = red_op<T, OP>(s, t.p[k][off]);
    for (int k = 0; k < n; ++k) t.p[k][off] = s;
  }
}

template <class T>
void launch_local(LocalGroup* g, int me, int64_t rows, int64_t ld, int64_t ncols, Op op, cudaStream_t st) {
  PtrTable<T> t{};
  for (int k = 0; k < g->n; ++k) t.p[k] = reinterpret_cast<T*>(g->ptr[k]);
  const int64_t total = rows * ncols;
  const int64_t lo = total * me / g->n, hi = total * (me + 1) / g->n;
  if (hi <= lo) return;
  const int blocks = (int)std::min<int64_t>((hi - lo + 255) / 256, 148 * 8);
  if (op == Op::Sum) k_local_allreduce<T, 0><<<blocks, 256, 0, st>>>(t, g->n, rows, ld, lo, hi);
  else if (op == Op::Max) k_local_allreduce<T, 1><<<blocks, 256, 0, st>>>(t, g->n, rows, ld, lo, hi);
  else k_local_allreduce<T, 2><<<blocks, 256, 0, st>>>(t, g->n, rows, ld, lo, hi);
  CHASE_CHECK_LAUNCH();
}

void local_allreduce(const Comm& c, void* buf, int64_t rows, int64_t ld, int64_t ncols, DT dt, Op op,
                     cudaStream_t st) {
  LocalGroup* g = c.local;
  const int me = c.rank;
  CHASE_CUDA(cudaEventRecord(g->ev_ready[me], st));
  g->ptr[me] = buf;
  g->barrier();                                         // every rank's (pointer, ready event) published
  for (int k = 0; k < g->n; ++k)
    if (k != me) CHASE_CUDA(cudaStreamWaitEvent(st, g->ev_ready[k], 0));
  if (dt == DT::F64) launch_local<double>(g, me, rows, ld, ncols, op, st);
  else if (dt == DT::F32) launch_local<float>(g, me, rows, ld, ncols, op, st);
  else launch_local<int>(g, me, rows, ld, ncols, op, st);
  CHASE_CUDA(cudaEventRecord(g->ev_done[me], st));
  g->barrier();                                         // every slice enqueued; pointers consumed
  for (int k = 0; k < g->n; ++k)
    if (k != me) CHASE_CUDA(cudaStreamWaitEvent(st, g->ev_done[k], 0));
}
}  // namespace

void comm_allreduce(const Comm& c, void* buf, int64_t rows, int64_t ld, int64_t ncols, DT dt, Op op,
                    cudaStream_t st) {
  if (!c.active() || rows <= 0 || ncols <= 0) return;
  if (c.local) {
    local_allreduce(c, buf, rows, ld, ncols, dt, op, st);
    return;
  }
  if (ld == rows || ncols == 1) {
    CHASE_NCCL(ncclAllReduce(buf, buf, (size_t)(rows * ncols), nccl_type(dt), nccl_op(op), c.nccl, st));
    return;
  }
  CHASE_NCCL(ncclGroupStart());
  for (int64_t j = 0; j < ncols; ++j) {
    char* col = reinterpret_cast<char*>(buf) + (size_t)j * ld * dt_bytes(dt);
    CHASE_NCCL(ncclAllReduce(col, col, (size_t)rows, nccl_type(dt), nccl_op(op), c.nccl, st));
  }
  CHASE_NCCL(ncclGroupEnd());
}

void comm_allgather_host(const Comm& c, const void* mine, size_t bytes, void* out, void* dscratch, cudaStream_t st) {
  if (c.size <= 1 || (!c.nccl && !c.local)) {
    std::memcpy(out, mine, bytes);
    return;
  }
  if (c.local) {
    LocalGroup* g = c.local;
    g->bytes[c.rank].assign(reinterpret_cast<const char*>(mine), reinterpret_cast<const char*>(mine) + bytes);
    g->barrier();
    for (int k = 0; k < g->n; ++k) std::memcpy(reinterpret_cast<char*>(out) + k * bytes, g->bytes[k].data(), bytes);
    g->barrier();
    return;
  }
  char* d = reinterpret_cast<char*>(dscratch);
  CHASE_CUDA(cudaMemcpyAsync(d, mine, bytes, cudaMemcpyHostToDevice, st));
  CHASE_NCCL(ncclAllGather(d, d + bytes, bytes, ncclUint8, c.nccl, st));
  CHASE_CUDA(cudaMemcpyAsync(out, d + bytes, bytes * c.size, cudaMemcpyDeviceToHost, st));
  CHASE_CUDA(cudaStreamSynchronize(st));
}

int comm_allreduce_int(const Comm& c, int v, Op op, void* dscratch, cudaStream_t st) {
  if (c.size <= 1 || (!c.nccl && !c.local)) return v;
  if (c.local) {
    LocalGroup* g = c.local;
    g->ival[c.rank] = v;
    g->barrier();
    int r = g->ival[0];
    for (int k = 1; k < g->n; ++k)
      r = op == Op::Sum ? r + g->ival[k] : (op == Op::Max ? std::max(r, g->ival[k]) : std::min(r, g->ival[k]));
    g->barrier();
    return r;
  }
  CHASE_CUDA(cudaMemcpyAsync(dscratch, &v, sizeof(int), cudaMemcpyHostToDevice, st));
  CHASE_NCCL(ncclAllReduce(dscratch, dscratch, 1, ncclInt32, nccl_op(op), c.nccl, st));
  CHASE_CUDA(cudaMemcpyAsync(&v, dscratch, sizeof(int), cudaMemcpyDeviceToHost, st));
  CHASE_CUDA(cudaStreamSynchronize(st));
  return v;
}

void comm_barrier(const Comm& c) {
  if (c.local && c.size > 1) c.local->barrier();
}

void comm_event_barrier(const Comm& c, cudaStream_t st) {
  if (!c.local || c.size <= 1) return;
  LocalGroup* g = c.local;
  CHASE_CUDA(cudaEventRecord(g->ev_ready[c.rank], st));
  g->barrier();
  for (int k = 0; k < g->n; ++k)
    if (k != c.rank) CHASE_CUDA(cudaStreamWaitEvent(st, g->ev_ready[k], 0));
  g->barrier();                        // every wait issued before any rank re-records its event
}

LocalGroup* local_join(const char* key, size_t keylen, int n, int rank) {
  if (n < 1 || n > kMaxLocal) throw UsageError("co-located group size must be 1.." + std::to_string(kMaxLocal));
  LocalGroup* g = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_reg_m);
    std::string k(key, keylen);
    auto it = g_reg.find(k);
    if (it == g_reg.end()) {
      g = new LocalGroup();
      g->key = k;
      g->n = n;
      g->ptr.assign(n, nullptr);
      g->ev_ready.assign(n, nullptr);
      g->ev_done.assign(n, nullptr);
      g->ival.assign(n, 0);
      g->bytes.assign(n, {});
      g_reg[k] = g;
    } else {
      g = it->second;
      if (g->n != n) throw UsageError("co-located group joined with a different size");
    }
    ++g->refs;
  }
  CHASE_CUDA(cudaEventCreateWithFlags(&g->ev_ready[rank], cudaEventDisableTiming));
  CHASE_CUDA(cudaEventCreateWithFlags(&g->ev_done[rank], cudaEventDisableTiming));
  g->barrier();                        // all n ranks joined
  return g;
}

void local_leave(LocalGroup* g, int rank) {
  if (!g) return;
  if (g->ev_ready[rank]) cudaEventDestroy(g->ev_ready[rank]);
  if (g->ev_done[rank]) cudaEventDestroy(g->ev_done[rank]);
  g->ev_ready[rank] = g->ev_done[rank] = nullptr;
  std::lock_guard<std::mutex> lk(g_reg_m);
  if (--g->refs == 0) {
    g_reg.erase(g->key);
    delete g;
  }
}

void comm_check_async(const Comm& c) {
  if (!c.nccl) return;
  ncclResult_t r = ncclSuccess;
  if (ncclCommGetAsyncError(c.nccl, &r) != ncclSuccess) return;
  if (r != ncclSuccess && r != ncclInProgress)
    throw NcclError(std::string("NCCL asynchronous error: ") + ncclGetErrorString(r));
}

void comm_abort(Comm& c) {
  if (c.nccl) ncclCommAbort(c.nccl);
  c.nccl = nullptr;
}

void comm_destroy(Comm& c) {
  if (c.nccl) ncclCommDestroy(c.nccl);
  c.nccl = nullptr;
  if (c.local) local_leave(c.local, c.rank);
  c.local = nullptr;
  c.size = 1;
}

}  // namespace chase
