// Common helpers for the ChASE B200 library (sm_100a only).
#pragma once
#include <unordered_map>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "this library targets sm_100a (B200) only"
#endif

namespace chase {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CHASE_CUDA(call)                                                                      \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      throw ::chase::CudaError(std::string(#call) + ": " + cudaGetErrorString(_e) + " @" +    \
                               __FILE__ + ":" + std::to_string(__LINE__));                    \
  } while (0)

// Every kernel launch of the library is followed by CHASE_CHECK_LAUNCH(), which also counts it
// (exported as chase_kernel_launches() for the benchmark's gpu_launches claim).
extern unsigned long long g_kernel_launches;
#define CHASE_CHECK_LAUNCH()            \
  do {                                  \
    ++::chase::g_kernel_launches;       \
    CHASE_CUDA(cudaGetLastError());     \
  } while (0)

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// complex double stored interleaved (re, im) == double2 == torch.complex128
using z_t = double2;

__host__ __device__ inline double2 zmk(double r, double i) { return make_double2(r, i); }

}  // namespace chase

// Per-device latch for one-time kernel attribute setup (cudaFuncSetAttribute is per device, and one
// process may drive several GPUs): true the first time it is called on the current device.
// Per calling THREAD and device: co-located ranks are threads of one process, and a shared flag
// would let a second thread launch before the first one's cudaFuncSetAttribute (shared-memory
// opt-in) completed -- a failed launch on that rank and a hang on its peers.  Setting the same
// attribute once per thread is idempotent and cheap.  `mask` only identifies the call site.
inline bool first_on_device(unsigned long long& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  thread_local std::unordered_map<const void*, unsigned long long> seen;
  unsigned long long& m = seen[&mask];
  const unsigned long long bit = 1ull << (dev & 63);
  if (m & bit) return false;
  m |= bit;
  return true;
}
