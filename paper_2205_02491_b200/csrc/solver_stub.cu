// Temporary: Lanczos / solve land in lanczos.cu / solver.cu.
#include "handle.h"
namespace chase {
LanczosOut lanczos(chase_handle*, const void*, int64_t, int) { throw UsageError("chase_lanczos: not implemented yet"); }
chase_status solve(chase_handle*, const void*, int64_t, int, int, int, double, double*, void*, int64_t, chase_report*) {
  throw UsageError("chase_solve: not implemented yet");
}
}
