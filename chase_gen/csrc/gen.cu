// Device twin of the G2 test-matrix generator (chase_gen/dense.py, G2Matrix.block).
// SEEDED INPUT GENERATION ONLY -- none of ChASE's arithmetic.  Evaluates
//   H[r, c] = phi_r conj(phi_c) circ[(r - c) mod n] + sum_t U[r, t] conj(V[c, t])
// with the same separate real multiplies/adds, in the same order, as the host evaluation
// (__dmul_rn/__dadd_rn/__dsub_rn: no FMA contraction), so host and device bytes agree.
#include <cuda_runtime.h>
#include <cstdint>

__global__ void k_gen_g2(double2* __restrict__ out, int64_t ld, int64_t r0, int64_t nr, int64_t c0,
                         int64_t nc, int64_t n, int rank, const double2* __restrict__ circ,
                         const double2* __restrict__ phi, const double2* __restrict__ U,
                         const double2* __restrict__ V) {
  const int64_t total = nr * nc;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rl = idx % nr, cl = idx / nr;
    const int64_t r = r0 + rl, c = c0 + cl;
    int64_t d = (r - c) % n;
    if (d < 0) d += n;
    const double2 cv = circ[d];
    const double2 pr = phi[r], pc = phi[c];
    const double pcr = pc.x, pci = -pc.y;
    const double sr = __dsub_rn(__dmul_rn(pr.x, pcr), __dmul_rn(pr.y, pci));
    const double si = __dadd_rn(__dmul_rn(pr.x, pci), __dmul_rn(pr.y, pcr));
    double hr = __dsub_rn(__dmul_rn(sr, cv.x), __dmul_rn(si, cv.y));
    double hi = __dadd_rn(__dmul_rn(sr, cv.y), __dmul_rn(si, cv.x));
    for (int t = 0; t < rank; ++t) {
      const double2 a = U[r * rank + t];
      const double2 b = V[c * rank + t];
      const double br = b.x, bi = -b.y;
      hr = __dadd_rn(hr, __dsub_rn(__dmul_rn(a.x, br), __dmul_rn(a.y, bi)));
      hi = __dadd_rn(hi, __dadd_rn(__dmul_rn(a.x, bi), __dmul_rn(a.y, br)));
    }
    out[rl + cl * ld] = make_double2(hr, hi);
  }
}

extern "C" int chase_gen_g2_block(void* out, int64_t ld, int64_t r0, int64_t nr, int64_t c0, int64_t nc,
                                  int64_t n, int rank, const void* circ, const void* phi, const void* U,
                                  const void* V, void* stream) {
  if (nr <= 0 || nc <= 0) return 0;
  const int64_t total = nr * nc;
  const int blocks = (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
  k_gen_g2<<<blocks, 256, 0, (cudaStream_t)stream>>>((double2*)out, ld, r0, nr, c0, nc, n, rank,
                                                     (const double2*)circ, (const double2*)phi,
                                                     (const double2*)U, (const double2*)V);
  return (int)cudaGetLastError();
}

// Real-symmetric twin (chase_gen/dense.py, R2Matrix.block):
//   H[r, c] = (s_r s_c) (u[(r - c) mod n] + w[(r + c) mod n]) + sum_t U[r, t] V[c, t]
__global__ void k_gen_r2(double* __restrict__ out, int64_t ld, int64_t r0, int64_t nr, int64_t c0, int64_t nc,
                         int64_t n, int rank, const double* __restrict__ u, const double* __restrict__ w,
                         const double* __restrict__ sgn, const double* __restrict__ U,
                         const double* __restrict__ V) {
  const int64_t total = nr * nc;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rl = idx % nr, cl = idx / nr;
    const int64_t r = r0 + rl, c = c0 + cl;
    int64_t dm = (r - c) % n;
    if (dm < 0) dm += n;
    const int64_t dp = (r + c) % n;
    double h = __dmul_rn(__dmul_rn(sgn[r], sgn[c]), __dadd_rn(u[dm], w[dp]));
    for (int t = 0; t < rank; ++t) h = __dadd_rn(h, __dmul_rn(U[r * rank + t], V[c * rank + t]));
    out[rl + cl * ld] = h;
  }
}

extern "C" int chase_gen_r2_block(void* out, int64_t ld, int64_t r0, int64_t nr, int64_t c0, int64_t nc,
                                  int64_t n, int rank, const void* u, const void* w, const void* sgn,
                                  const void* U, const void* V, void* stream) {
  if (nr <= 0 || nc <= 0) return 0;
  const int64_t total = nr * nc;
  const int blocks = (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
  k_gen_r2<<<blocks, 256, 0, (cudaStream_t)stream>>>((double*)out, ld, r0, nr, c0, nc, n, rank, (const double*)u,
                                                     (const double*)w, (const double*)sgn, (const double*)U,
                                                     (const double*)V);
  return (int)cudaGetLastError();
}
