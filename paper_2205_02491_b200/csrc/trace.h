// NVTX ranges (SURVEY §5 tracing): one per Alg. 1 phase of chase_solve (Lanczos, Filter, QR, RR,
// Resid -- the Table 2 columns) and one per filter step ("filter k=.. fwd/bwd n_k=..").
// Header-only NVTX3: a no-op unless a tool (nsys / ncu --nvtx) is attached.
#pragma once
#include <nvtx3/nvToolsExt.h>
#include <cstdio>

namespace chase {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
inline void nvtx_push_step(int k, int dir, int ncols) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "filter k=%d %s n_k=%d", k, dir == 0 ? "fwd" : "bwd", ncols);
  nvtxRangePushA(buf);
}
inline void nvtx_pop() { nvtxRangePop(); }
}  // namespace chase
