// Complex-single (CHASE_C64) filter path: host side of the tcgen05 3xTF32 fused step
// (cgemm_tc.cuh), format conversions and the c64 filter driver (SURVEY §8 a1-a5 in complex single).
//
// Internal operand formats (chosen so that every MMA operand arrives by TMA in the layout the next
// step needs):
//   V-layout (input of forward steps, output of backward steps): planar Re/Im fp32 planes plus their
//     3xTF32 lo planes -- 4 planes of q x n (ld q);
//   W-layout (output of forward steps, input of backward steps): W interleaved complex64, the
//     rotated copy -iW, and both lo copies -- 4 arrays of p x n complex64 (ld p);
//   H_lo: lo part of the caller's H shard, computed once per shard pointer.
#include <algorithm>
#include <vector>
#include "cgemm_tc.cuh"
#include "handle.h"
#include "trace.h"

namespace chase {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {   // thread-safe one-time init
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CHASE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

CUtensorMapL2promotion promo() {
  static const int v = getenv("CHASE_C64_PROMO") ? atoi(getenv("CHASE_C64_PROMO")) : 3;
  return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
       : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// fp32 matrix, dim 0 = rows (contiguous), dim 1 = cols (stride ld floats); box {32, box_cols}
void f32_tmap(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_cols,
              CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_cols};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, promo(),
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (fp32) failed: " + std::to_string((int)r));
}

__global__ void k_lo(float* dst, const float* src, int64_t rows, int cols, int64_t ldd, int64_t lds) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows, c = i / rows;
    dst[r + c * ldd] = tc::tf32_lo(src[r + c * lds]);
  }
}

// interleaved complex (complex64, or complex128 rounded to fp32 in the mixed solve) (rows x cols,
// ld complex) -> planar Re, Im, Re_lo, Im_lo (ld rows)
template <class TX>
__global__ void k_to_planar(const TX* X, int64_t ldx, int64_t rows, int cols, float* Pr, float* Pi, float* Prl,
                            float* Pil, int64_t ldp) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows, c = i / rows;
    const TX x = X[r + c * ldx];
    const float2 v = make_float2((float)x.x, (float)x.y);
    const int64_t o = r + c * ldp;
    Pr[o] = v.x;
    Pi[o] = v.y;
    if (Prl) Prl[o] = tc::tf32_lo(v.x);
    if (Pil) Pil[o] = tc::tf32_lo(v.y);
  }
}

template <class TX>
__global__ void k_from_planar(TX* X, int64_t ldx, int64_t rows, int cols, const float* Pr, const float* Pi,
                              int64_t ldp) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows, c = i / rows;
    X[r + c * ldx].x = Pr[r + c * ldp];
    X[r + c * ldx].y = Pi[r + c * ldp];
  }
}

// complex64 <-> complex128 block copies (mixed solve: the c128 iteration around the c64 shard)
template <class TD, class TS>
__global__ void k_convert(TD* D, int64_t ldd, const TS* S, int64_t lds, int64_t rows, int cols) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows, c = i / rows;
    const TS v = S[r + c * lds];
    D[r + c * ldd].x = v.x;
    D[r + c * ldd].y = v.y;
  }
}

// interleaved X -> W (copy, ld rows), -iX, and lo copies of both
__global__ void k_to_wfmt(const float2* X, int64_t ldx, int64_t rows, int cols, float2* W, float2* Wr, float2* Wl,
                          float2* Wrl, int64_t ldw) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % rows, c = i / rows;
    const float2 v = X[r + c * ldx];
    const int64_t o = r + c * ldw;
    const float2 rot = make_float2(v.y, -v.x);
    if (W) W[o] = v;
    Wr[o] = rot;
    Wl[o] = make_float2(tc::tf32_lo(v.x), tc::tf32_lo(v.y));
    Wrl[o] = make_float2(tc::tf32_lo(rot.x), tc::tf32_lo(rot.y));
  }
}

inline int grid_for(int64_t total) { return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 32)); }

struct VFmt {        // planar V-layout block: 4 planes, ld = q
  float *r, *i, *rl, *il;
  int64_t ld;
};
struct WFmt {        // W-layout block: 4 complex64 arrays, ld = p
  float2 *w, *wr, *wl, *wrl;
  int64_t ld;
};

// one local fused step (no communication); `first` columns offset already applied by the caller
template <int BN>
void c64_step_bn(chase_handle* h, int dir, const void* H, int64_t ldh, const void* Hlo, const VFmt& v,
                 const WFmt& w, int ncols, double alpha, double beta, double gamma, bool beta_on, const C64Red* red) {
  using namespace tc;
  constexpr size_t SMEM = Cfg<BN>::SMEM;
  const Grid& g = h->grid;
  const int64_t r0 = g.rows.start, p = g.rows.len, c0 = g.cols.start, q = g.cols.len;
  CUtensorMap ta, tal, tb1, tb1l, tb2, tb2l;
  C64Params P{};
  P.N = ncols;
  P.alpha = (float)alpha; P.beta = (float)beta; P.gamma = (float)gamma;
  P.beta_on = beta_on ? 1 : 0;
  static const int kcs = getenv("CHASE_C64_KC") ? atoi(getenv("CHASE_C64_KC")) : 0;
  P.kc_stages = kcs;
  static const int rg = getenv("CHASE_C64_RASTER") ? atoi(getenv("CHASE_C64_RASTER")) : 0;
  P.raster_group = rg;
  if (dir == 0) {       // forward: W = alpha (H V - gamma E V) + beta W
    f32_tmap(&ta, H, 2 * p, q, 2 * ldh, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    f32_tmap(&tal, Hlo, 2 * p, q, 2 * p, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    f32_tmap(&tb1, v.r, q, ncols, v.ld, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    f32_tmap(&tb1l, v.rl, q, ncols, v.ld, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    f32_tmap(&tb2, v.i, q, ncols, v.ld, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    f32_tmap(&tb2l, v.il, q, ncols, v.ld, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    P.M = (int)(2 * p);
    P.K = (int)q;
    P.S0 = v.r; P.S1 = v.i; P.lds = v.ld;
    P.shift_lo = (int)std::max<int64_t>(0, c0 - r0);
    P.shift_hi = (int)std::min<int64_t>(p, c0 + q - r0);
    P.shift_off = r0 - c0;
    P.Y0 = reinterpret_cast<float*>(w.w); P.Y1 = reinterpret_cast<float*>(w.wr);
    P.Y0lo = reinterpret_cast<float*>(w.wl); P.Y1lo = reinterpret_cast<float*>(w.wrl);
    P.ldy = 2 * w.ld;
  } else {              // backward: V = alpha (H^H W - gamma E^T W) + beta V
    f32_tmap(&ta, H, 2 * p, q, 2 * ldh, BMR, CU_TENSOR_MAP_SWIZZLE_128B);
    f32_tmap(&tal, Hlo, 2 * p, q, 2 * p, BMR, CU_TENSOR_MAP_SWIZZLE_128B);
    f32_tmap(&tb1, w.w, 2 * p, ncols, 2 * w.ld, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    f32_tmap(&tb1l, w.wl, 2 * p, ncols, 2 * w.ld, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    f32_tmap(&tb2, w.wr, 2 * p, ncols, 2 * w.ld, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    f32_tmap(&tb2l, w.wrl, 2 * p, ncols, 2 * w.ld, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    P.M = (int)q;
    P.K = (int)(2 * p);
    P.S0 = reinterpret_cast<const float*>(w.w); P.S1 = nullptr; P.lds = w.ld;
    P.shift_lo = (int)std::max<int64_t>(0, r0 - c0);
    P.shift_hi = (int)std::min<int64_t>(q, r0 + p - c0);
    P.shift_off = c0 - r0;
    P.Y0 = v.r; P.Y1 = v.i; P.Y0lo = v.rl; P.Y1lo = v.il;
    P.ldy = v.ld;
  }
  if (gamma == 0.0 || P.shift_lo >= P.shift_hi) P.shift_lo = P.shift_hi = 0;
  static unsigned long long attr[2] = {0, 0};
  // CTA pairs (default; CHASE_C64_PAIR=0 selects the single-CTA kernel)
  static const bool pair = !getenv("CHASE_C64_PAIR") || atoi(getenv("CHASE_C64_PAIR")) != 0;
  if (red && !pair) throw UsageError("fused c64 all-reduce needs the CTA-pair kernel");
  if (red) P.red = *red;
  if (pair) {
    // CTA pairs: one cluster of 2 per 256-row x BN tile
    constexpr size_t SMEM2 = Cfg2<BN>::SMEM;
    static unsigned long long attr2[4] = {0, 0, 0, 0};
    const int grid2 = 2 * ceil_div(P.M, 2 * BMR) * ceil_div(P.N, BN);
    auto go = [&](auto kern, int slot) {
      if (first_on_device(attr2[slot]))
        CHASE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM2));
      kern<<<grid2, C64_THREADS, SMEM2, h->stream>>>(ta, tal, tb1, tb1l, tb2, tb2l, P);
    };
    static const bool persistent = !getenv("CHASE_C64_PERSIST") || atoi(getenv("CHASE_C64_PERSIST")) != 0;
    if (!red && persistent) {
      // persistent grouped schedule with the L2 round barrier (cgemm_tc.cuh c64_step_kernel_p)
      static unsigned long long attrp[2] = {0, 0};
      int sms = 148, dev = 0;
      CHASE_CUDA(cudaGetDevice(&dev));
      CHASE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      const int ptiles = ceil_div(P.M, 2 * BMR) * ceil_div(P.N, BN);
      const int gridp = 2 * std::min(ptiles, sms / 2);
      static const int gw_env = getenv("CHASE_C64_GW") ? atoi(getenv("CHASE_C64_GW")) : 0;
      const int tiles_n = ceil_div(P.N, BN);
      int gw = c64_segment_width(tiles_n, gridp / 2);
      if (gw_env > 0 && tiles_n % gw_env == 0 && gw_env <= gridp / 2) gw = gw_env;   // tuning knob
      h->oz_sync.alloc(256);
      CHASE_CUDA(cudaMemsetAsync(h->oz_sync.p, 0, 64, h->stream));
      unsigned* sy = h->colocated ? nullptr : h->oz_sync.as<unsigned>();   // co-located ranks share the SMs
      auto gp = [&](auto kern, int slot) {
        if (first_on_device(attrp[slot]))
          CHASE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM2));
        kern<<<gridp, C64_THREADS, SMEM2, h->stream>>>(ta, tal, tb1, tb1l, tb2, tb2l, P, sy, gw);
      };
      if (dir == 0) gp(c64_step_kernel_p<true, BN>, 0); else gp(c64_step_kernel_p<false, BN>, 1);
      CHASE_CHECK_LAUNCH();
      return;
    }
    if (dir == 0) {
      if (red) go(c64_step_kernel2<true, BN, true>, 0); else go(c64_step_kernel2<true, BN, false>, 1);
    } else {
      if (red) go(c64_step_kernel2<false, BN, true>, 2); else go(c64_step_kernel2<false, BN, false>, 3);
    }
    CHASE_CHECK_LAUNCH();
    return;
  }
  const int grid = ceil_div(P.M, BMR) * ceil_div(P.N, BN);
  if (dir == 0) {
    if (first_on_device(attr[0])) CHASE_CUDA(cudaFuncSetAttribute(c64_step_kernel<true, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    c64_step_kernel<true, BN><<<grid, C64_THREADS, SMEM, h->stream>>>(ta, tal, tb1, tb1l, tb2, tb2l, P);
  } else {
    if (first_on_device(attr[1])) CHASE_CUDA(cudaFuncSetAttribute(c64_step_kernel<false, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    c64_step_kernel<false, BN><<<grid, C64_THREADS, SMEM, h->stream>>>(ta, tal, tb1, tb1l, tb2, tb2l, P);
  }
  CHASE_CHECK_LAUNCH();
}

// column tile: 128 (MMA N = 256) unless CHASE_C64_BN=64 (N = 128)
void c64_step_local(chase_handle* h, int dir, const void* H, int64_t ldh, const void* Hlo, const VFmt& v,
                    const WFmt& w, int ncols, double alpha, double beta, double gamma, bool beta_on,
                    const C64Red* red = nullptr) {
  static const int bn = [] { const char* e = getenv("CHASE_C64_BN"); return e ? atoi(e) : 128; }();
  if (bn == 64)
    c64_step_bn<64>(h, dir, H, ldh, Hlo, v, w, ncols, alpha, beta, gamma, beta_on, red);
  else
    c64_step_bn<128>(h, dir, H, ldh, Hlo, v, w, ncols, alpha, beta, gamma, beta_on, red);
}

// number of CTAs (= reduction tiles) the step launches
int c64_step_tiles(int M, int N) {
  static const int bn = [] { const char* e = getenv("CHASE_C64_BN"); return e ? atoi(e) : 128; }();
  return 2 * ceil_div(M, 2 * tc::BMR) * ceil_div(N, bn == 64 ? 64 : 128);
}

static bool c64_pair_kernel() {
  static const bool pair = !getenv("CHASE_C64_PAIR") || atoi(getenv("CHASE_C64_PAIR")) != 0;
  return pair;
}

}  // namespace

// in-place float sum of a complex64 column block (rows x ncols, ld) over a communicator
void allreduce_c64(chase_handle* h, const Comm& comm, void* Y, int64_t rows, int64_t ld, int ncols) {
  if (!comm.active() || ncols <= 0 || rows <= 0) return;
  comm_allreduce(comm, Y, 2 * rows, 2 * ld, ncols, DT::F32, Op::Sum, h->stream);
}

// f4: complex64 shadow of a complex128 shard (rounded to nearest), ld p
const void* c64_shadow(chase_handle* h, const void* H, int64_t ldh) {
  const int64_t p = h->grid.rows.len, q = h->grid.cols.len;
  if (h->h32_src != H || h->h32_ld != ldh || !h->H32.p) {
    h->H32.alloc(8 * (size_t)p * q);
    k_convert<<<grid_for(p * q), 256, 0, h->stream>>>(h->H32.as<float2>(), p, reinterpret_cast<const double2*>(H), ldh,
                                                      p, (int)q);
    CHASE_CHECK_LAUNCH();
    h->h32_src = H;
    h->h32_ld = ldh;
    h->hlo_src = nullptr;                   // the shadow's lo part must be rebuilt
  }
  return h->H32.p;
}

// H_lo for the shard (recomputed when the caller's H pointer or ld changes)
void c64_check_call(chase_handle* h, const void* H, int64_t ldh, int ncols) {
  if (H && (ldh % 2 != 0 || (reinterpret_cast<uintptr_t>(H) % 16) != 0))
    throw UsageError("CHASE_C64 needs an even ldh and a 16-byte aligned H shard");
  if (ncols > h->n_e_max) throw UsageError("c64: ncols exceeds nev_max + nex_max");
}

const void* c64_hlo(chase_handle* h, const void* H, int64_t ldh) {
  const int64_t p = h->grid.rows.len, q = h->grid.cols.len;
  // TMA: 16-byte aligned bases / strides for the fp32 planes (ld q), the interleaved W (ld 2p
  // floats) and H (ld 2*ldh floats)
  if (q % 4 != 0 || p % 2 != 0 || ldh % 2 != 0 || (reinterpret_cast<uintptr_t>(H) % 16) != 0)
    throw UsageError("CHASE_C64 (round 1) needs shard columns q % 4 == 0, rows p even, even ldh, 16-B aligned H");
  if (h->hlo_src != H || h->hlo_ld != ldh || !h->Hlo.p) {
    h->Hlo.alloc(8 * (size_t)p * q);
    k_lo<<<grid_for(2 * p * q), 256, 0, h->stream>>>(h->Hlo.as<float>(), reinterpret_cast<const float*>(H), 2 * p,
                                                    (int)q, 2 * p, 2 * ldh);
    CHASE_CHECK_LAUNCH();
    h->hlo_src = H;
    h->hlo_ld = ldh;
  }
  return h->Hlo.p;
}

// internal-format views of the handle's workspace for `ncols` columns starting at column `c`
static VFmt vfmt(chase_handle* h, int ncap, int c) {
  const int64_t q = h->grid.cols.len;
  h->c64v.alloc(16 * (size_t)q * ncap);
  float* base = h->c64v.as<float>();       // 16 B per element = 4 planes of q x ncap
  VFmt v;
  v.ld = q;
  v.r = base + (int64_t)c * q;
  v.i = base + (int64_t)ncap * q + (int64_t)c * q;
  v.rl = base + 2 * (int64_t)ncap * q + (int64_t)c * q;
  v.il = base + 3 * (int64_t)ncap * q + (int64_t)c * q;
  return v;
}
static WFmt wfmt(chase_handle* h, int ncap, int c) {
  const int64_t p = h->grid.rows.len;
  h->c64w.alloc(32 * (size_t)p * ncap);
  float2* a = h->c64w.as<float2>();                         // W, -iW
  float2* b = a + 2 * (int64_t)ncap * p;                    // lo copies
  WFmt w;
  w.ld = p;
  w.w = a + (int64_t)c * p;
  w.wr = a + (int64_t)ncap * p + (int64_t)c * p;
  w.wl = b + (int64_t)c * p;
  w.wrl = b + (int64_t)ncap * p + (int64_t)c * p;
  return w;
}

// public single step (interleaved complex64 X / Y), see chase_hemm_step
void c64_hemm_step(chase_handle* h, int dir, const void* H, int64_t ldh, const void* X, int64_t ldx, void* Y,
                   int64_t ldy, int ncols, double alpha, double beta, double gamma) {
  if (ncols <= 0) return;
  if (ncols > h->n_e_max) throw UsageError("c64 step: ncols exceeds nev_max + nex_max");
  const Grid& g = h->grid;
  const int64_t p = g.rows.len, q = g.cols.len;
  const void* Hlo = c64_hlo(h, H, ldh);
  const double hs = h->opt.largest ? -1.0 : 1.0;
  const int ncap = h->n_e_max;
  VFmt v = vfmt(h, ncap, 0);
  WFmt w = wfmt(h, ncap, 0);
  const bool beta_owner = dir == 0 ? g.beta_owner_fwd() : g.beta_owner_bwd();
  if (dir == 0) {
    k_to_planar<<<grid_for(q * ncols), 256, 0, h->stream>>>(reinterpret_cast<const float2*>(X), ldx, q, ncols, v.r, v.i,
                                                            v.rl, v.il, v.ld);
    CHASE_CHECK_LAUNCH();
    WFmt out{reinterpret_cast<float2*>(Y), nullptr, nullptr, nullptr, ldy};
    c64_step_local(h, 0, H, ldh, Hlo, v, out, ncols, alpha * hs, beta, gamma * hs, beta_owner && beta != 0.0);
    allreduce_c64(h, h->rowc, Y, p, ldy, ncols);
  } else {
    k_to_wfmt<<<grid_for(p * ncols), 256, 0, h->stream>>>(reinterpret_cast<const float2*>(X), ldx, p, ncols, w.w, w.wr,
                                                          w.wl, w.wrl, w.ld);
    CHASE_CHECK_LAUNCH();
    const bool bo = beta_owner && beta != 0.0;
    if (bo) {
      k_to_planar<<<grid_for(q * ncols), 256, 0, h->stream>>>(reinterpret_cast<const float2*>(Y), ldy, q, ncols, v.r,
                                                              v.i, nullptr, nullptr, v.ld);
      CHASE_CHECK_LAUNCH();
    }
    c64_step_local(h, 1, H, ldh, Hlo, v, w, ncols, alpha * hs, beta, gamma * hs, bo);
    k_from_planar<<<grid_for(q * ncols), 256, 0, h->stream>>>(reinterpret_cast<float2*>(Y), ldy, q, ncols, v.r, v.i,
                                                              v.ld);
    CHASE_CHECK_LAUNCH();
    allreduce_c64(h, h->colc, Y, q, ldy, ncols);
  }
}

// mixed solve: (HX) in complex128 from a complex128 X (q x ncols, V-layout) through the c64 forward
// step (RR's HQ, a8 step 1); the product itself is the tcgen05 3xTF32 step (FP32-class accuracy)
void c64_forward_mixed(chase_handle* h, const void* H, int64_t ldh, const double2* X, int64_t ldx, double2* Y,
                       int64_t ldy, int ncols) {
  if (ncols <= 0) return;
  const Grid& g = h->grid;
  const int64_t p = g.rows.len, q = g.cols.len;
  const void* Hlo = c64_hlo(h, H, ldh);
  const double hs = h->opt.largest ? -1.0 : 1.0;
  VFmt v = vfmt(h, h->n_e_max, 0);
  WFmt w = wfmt(h, h->n_e_max, 0);
  k_to_planar<<<grid_for(q * ncols), 256, 0, h->stream>>>(X, ldx, q, ncols, v.r, v.i, v.rl, v.il, v.ld);
  CHASE_CHECK_LAUNCH();
  WFmt out{w.w, nullptr, nullptr, nullptr, w.ld};
  c64_step_local(h, 0, H, ldh, Hlo, v, out, ncols, hs, 0.0, 0.0, false);
  allreduce_c64(h, h->rowc, w.w, p, w.ld, ncols);
  k_convert<<<grid_for(p * ncols), 256, 0, h->stream>>>(Y, ldy, w.w, w.ld, p, ncols);
  CHASE_CHECK_LAUNCH();
}

void c64_convert(void* dst, int64_t ldd, bool dst_c128, const void* src, int64_t lds, int64_t rows, int cols,
                 cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  if (dst_c128)
    k_convert<<<grid_for(rows * cols), 256, 0, st>>>(reinterpret_cast<double2*>(dst), ldd,
                                                     reinterpret_cast<const float2*>(src), lds, rows, cols);
  else
    k_convert<<<grid_for(rows * cols), 256, 0, st>>>(reinterpret_cast<float2*>(dst), ldd,
                                                     reinterpret_cast<const double2*>(src), lds, rows, cols);
  CHASE_CHECK_LAUNCH();
}

// c64 filter (a1-a5): same schedule / scalars as the c128 filter; V interleaved in/out (complex64,
// or complex128 in the mixed solve, rounded to fp32 on entry), internal planar / rotated formats
// in between.  The all-reduce of each step runs on the interleaved W (forward) or the planar V
// (backward) -- both are plain sums.
template <class TV>
static int64_t c64_filter_t(chase_handle* h, const void* H, int64_t ldh, TV* V, int64_t ldv, int ncols,
                            const int* degrees, double b_sup, double mu_1, double mu_ne) {
  if (ncols <= 0) return 0;
  if (ncols > h->n_e_max) throw UsageError("c64 filter: ncols exceeds nev_max + nex_max");
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
  const Grid& g = h->grid;
  const int64_t p = g.rows.len, q = g.cols.len;
  const void* Hlo = c64_hlo(h, H, ldh);
  const double hs = h->opt.largest ? -1.0 : 1.0;
  const int ncap = h->n_e_max;
  VFmt v0 = vfmt(h, ncap, 0);
  k_to_planar<<<grid_for(q * ncols), 256, 0, h->stream>>>(V, ldv, q, ncols, v0.r, v0.i, v0.rl, v0.il, v0.ld);
  CHASE_CHECK_LAUNCH();
  const double sigma1 = e / (mu_1 - c);
  double sigma_prev = sigma1;
  int first = 0;
  // f1: all-reduce inside the step kernel over peer memory (CTA-pair kernel only)
  wfmt(h, ncap, 0);
  const int64_t pmax = (g.N + g.r - 1) / g.r, qmax = (g.N + g.c - 1) / g.c;   // same on every rank
  const bool fused = (g.r > 1 || g.c > 1) && h->opt.fused_reduce_c64 && c64_pair_kernel() &&
                     peer_tiles_fit(std::max(c64_step_tiles((int)(2 * pmax), ncols), c64_step_tiles((int)qmax, ncols))) &&
                     peer_c64_ready(h);
  if (fused) peer_enter(h);
  const int64_t plane = 2 * std::max(p, q) * (int64_t)ncap;
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
    const int nk = ncols - first;
    nvtx_push_step(k, (k & 1) ? 0 : 1, nk);
    struct PopAtEnd { ~PopAtEnd() { nvtx_pop(); } } pop_at_end;
    VFmt v = vfmt(h, ncap, first);
    WFmt w = wfmt(h, ncap, first);
    const int cn = (k & 1) ? g.c : g.r;
    if (fused && cn > 1) {
      peer_poll(h);
      const PeerRed& pr = (k & 1) ? h->peer.row : h->peer.col;
      C64Red R;
      R.n = pr.n;
      R.me = pr.me;
      R.ctr = pr.ctr;
      float* own = (k & 1) ? h->c64w.as<float>() : h->c64v.as<float>();
      for (int r = 0; r < pr.n; ++r) {
        R.stage[r] = reinterpret_cast<float*>(pr.stage[r]);
        R.base[r] = (k & 1) ? h->peer.c64w_row[r] : h->peer.c64v_col[r];
        R.done[r] = pr.done[r];
      }
      if (k & 1) {
        R.o0 = reinterpret_cast<float*>(w.w) - own;
        R.o1 = reinterpret_cast<float*>(w.wr) - own;
        R.o0lo = reinterpret_cast<float*>(w.wl) - own;
        R.o1lo = reinterpret_cast<float*>(w.wrl) - own;
      } else {
        R.o0 = v.r - own;
        R.o1 = v.i - own;
        R.o0lo = v.rl - own;
        R.o1lo = v.il - own;
      }
      R.plane = plane;
      if (k & 1)
        c64_step_local(h, 0, H, ldh, Hlo, v, w, nk, alpha * hs, beta, c * hs, g.beta_owner_fwd() && beta != 0.0, &R);
      else
        c64_step_local(h, 1, H, ldh, Hlo, v, w, nk, alpha * hs, beta, c * hs, g.beta_owner_bwd() && beta != 0.0, &R);
      peer_wait(h, c64_step_tiles((k & 1) ? (int)(2 * p) : (int)q, nk));
      if (k & 1) {
        k_to_wfmt<<<grid_for(p * nk), 256, 0, h->stream>>>(w.w, w.ld, p, nk, nullptr, w.wr, w.wl, w.wrl, w.ld);
        CHASE_CHECK_LAUNCH();
      } else {
        k_lo<<<grid_for(q * nk), 256, 0, h->stream>>>(v.rl, v.r, q, nk, v.ld, v.ld);
        CHASE_CHECK_LAUNCH();
        k_lo<<<grid_for(q * nk), 256, 0, h->stream>>>(v.il, v.i, q, nk, v.ld, v.ld);
        CHASE_CHECK_LAUNCH();
      }
      continue;
    }
    if (k & 1) {
      c64_step_local(h, 0, H, ldh, Hlo, v, w, nk, alpha * hs, beta, c * hs, g.beta_owner_fwd() && beta != 0.0);
      if (g.c > 1 && h->rowc.active()) {
        // the sum must also reach the rotated / lo copies: all-reduce W, then rebuild them
        allreduce_c64(h, h->rowc, w.w, p, w.ld, nk);
        k_to_wfmt<<<grid_for(p * nk), 256, 0, h->stream>>>(w.w, w.ld, p, nk, nullptr, w.wr, w.wl, w.wrl, w.ld);
        CHASE_CHECK_LAUNCH();
      }
    } else {
      c64_step_local(h, 1, H, ldh, Hlo, v, w, nk, alpha * hs, beta, c * hs, g.beta_owner_bwd() && beta != 0.0);
      if (g.r > 1 && h->colc.active()) {
        // planar Re / Im planes (ld q): sum both, then rebuild the lo planes
        comm_allreduce(h->colc, v.r, q, v.ld, nk, DT::F32, Op::Sum, h->stream);
        comm_allreduce(h->colc, v.i, q, v.ld, nk, DT::F32, Op::Sum, h->stream);
        k_lo<<<grid_for(q * nk), 256, 0, h->stream>>>(v.rl, v.r, q, nk, v.ld, v.ld);
        CHASE_CHECK_LAUNCH();
        k_lo<<<grid_for(q * nk), 256, 0, h->stream>>>(v.il, v.i, q, nk, v.ld, v.ld);
        CHASE_CHECK_LAUNCH();
      }
    }
  }
  if (fused) peer_check(h);
  // columns of degree 0 were never touched: write back only the filtered suffix
  int f0 = 0;
  while (f0 < ncols && degrees[f0] == 0) ++f0;
  VFmt vout = vfmt(h, ncap, f0);
  k_from_planar<<<grid_for(q * (ncols - f0)), 256, 0, h->stream>>>(V + (int64_t)f0 * ldv, ldv, q, ncols - f0, vout.r,
                                                                   vout.i, vout.ld);
  CHASE_CHECK_LAUNCH();
  return matvecs;
}

int64_t c64_filter(chase_handle* h, const void* H, int64_t ldh, void* V, int64_t ldv, int ncols, const int* degrees,
                   double b_sup, double mu_1, double mu_ne) {
  return c64_filter_t(h, H, ldh, reinterpret_cast<float2*>(V), ldv, ncols, degrees, b_sup, mu_1, mu_ne);
}

int64_t c64_filter_mixed(chase_handle* h, const void* H, int64_t ldh, double2* V, int64_t ldv, int ncols,
                         const int* degrees, double b_sup, double mu_1, double mu_ne) {
  return c64_filter_t(h, H, ldh, V, ldv, ncols, degrees, b_sup, mu_1, mu_ne);
}

}  // namespace chase
