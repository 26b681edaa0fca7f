// Communicators of one rank: the world, its row communicator (colour i, key j) and
// its column communicator (colour j, key i).  Two transports behind one interface:
//
//  * NCCL (one process per GPU, the production path): ncclAllReduce / ncclAllGather on the
//    caller's stream over NVLink5 / NVSwitch.
//  * Co-located group (several ranks of one grid driven by threads of ONE process, possibly on ONE
//    device -- NCCL refuses two ranks on one GPU): an in-process rendezvous keyed by the 128-byte id.
//    All-reduce is stream-ordered without any device-side waiting: each rank records an event when
//    its buffer is ready, a host barrier publishes (pointer, event), every rank's stream waits on the
//    peers' events, and rank k then sums slice k of the block over all ranks in rank order and
//    stores it into every replica (disjoint slices, so no rank reads what another writes), and a
//    second event round orders the ranks' next writes after every slice is done.  Sums are taken
//    in communicator-rank order, so replicas are bitwise identical (ledger #20), as with NCCL.
//    Used to run the multi-rank data plane (a3/a5 all-reduces and the fused f1 epilogue, whose peer
//    tables then hold the co-located handles' own device pointers) on a single GPU.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <cstddef>
#include <cstdint>

struct chase_handle;

namespace chase {

struct LocalGroup;   // comm.cu

enum class DT { F64, F32, I32 };
enum class Op { Sum, Max, Min };

struct Comm {
  ncclComm_t nccl = nullptr;
  LocalGroup* local = nullptr;
  int size = 1, rank = 0;
  bool active() const { return size > 1 && (nccl != nullptr || local != nullptr); }
};

// In-place all-reduce of a strided block on `st`: `ncols` columns of `rows` scalars with leading
// dimension `ld` (scalars).  No-op when the communicator is inactive.
void comm_allreduce(const Comm& c, void* buf, int64_t rows, int64_t ld, int64_t ncols, DT dt, Op op,
                    cudaStream_t st);
// All-gather of `bytes` host bytes per rank into out[size * bytes] (synchronous; `st` and the
// device scratch `dscratch` (>= (size + 1) * bytes) are used by the NCCL transport).
void comm_allgather_host(const Comm& c, const void* mine, size_t bytes, void* out, void* dscratch, cudaStream_t st);
// Host-side integer all-reduce (synchronous); `dscratch` >= 4 bytes of device memory (NCCL transport).
int comm_allreduce_int(const Comm& c, int v, Op op, void* dscratch, cudaStream_t st);
// Host barrier of a co-located group (no-op for NCCL).
void comm_barrier(const Comm& c);
// Co-located group: `st` waits for the work every rank has enqueued so far (event all-to-all;
// no-op for NCCL).
void comm_event_barrier(const Comm& c, cudaStream_t st);
// Co-located rendezvous: join (create if absent) the group `key` of `n` ranks as `rank`.
// Blocks until all n ranks have joined (timeout -> NcclError).
LocalGroup* local_join(const char* key, size_t keylen, int n, int rank);
void local_leave(LocalGroup* g, int rank);
// Cross-rank error check for NCCL communicators (ncclCommGetAsyncError); throws NcclError.
void comm_check_async(const Comm& c);
void comm_abort(Comm& c);
void comm_destroy(Comm& c);

}  // namespace chase
