// ChASE driver (Alg. 1) on the device: Lanczos -> loop { Filter -> QR -> Rayleigh-Ritz
// -> residuals -> deflation & locking -> bounds -> degrees -> sort }.
//
// Everything that touches N-length data runs in the library's kernels on the caller's H shard;
// the host only makes the per-iteration scalar decisions (locking prefix, bounds, degrees, sort
// order) from n_act Ritz values and residuals copied back once per iteration -- identical on
// every rank because their inputs were all-reduced.  Distributed semantics:
//  * QR: 2x classical Gram-Schmidt against the locked block + CholQR2 (ledger #13; north_star);
//    Gram matrices V_j^H V_j are summed over the row communicator (it spans every column block).
//  * RR: HQ by the forward HEMM (W-layout), G = sum_ij Q_j[I_ij]^H (HQ)_i[I_ij] over the
//    intersection rows I_ij (each global row lies in exactly one), summed over the world;
//    G = Z diag(theta) Z^H by the device block Jacobi (redundant, deterministic); V <- Q Z and
//    HV <- (HQ) Z (reused by the residuals: no second HEMM).
//  * Residuals: ||HV_a - theta_a V_a||^2 over I_ij, summed over the world, normalised
//    by nu = max |Lanczos Ritz| (ledger #5).
// The paper's redundant QR/RR with a post-filter V-hat broadcast is replaced
// by these distributed forms (its future-work item).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>
#include "dense.h"
#include "handle.h"
#include "linalg.h"
#include "scalar.cuh"
#include "trace.h"

namespace chase {

namespace {

// m_a <- Degrees(tol, Res_a, lambda_a, c, e)  (Alg. 1 line 12; ledger #4 / S:366)
// deg_extra (reading 4b): degrees added to the estimate before the cap -- it aims at
// exactly tol, so a column just above tol would get m -> 1 and creep (measured on config 3:
// 100+ iterations at res = 1.01 tol).
int optimal_degree(double tol, double res, double theta, double c, double e, int deg_max, int deg_extra) {
  const double t = (c - theta) / e;
  int m;
  if (std::fabs(t) <= 1.0) {
    m = deg_max;
  } else {
    const double s = std::sqrt(t * t - 1.0);
    const double rho = std::max(std::fabs(t + s), std::fabs(t - s));
    const double ratio = res / tol;
    m = ratio > 0.0 ? (int)std::ceil(std::log(ratio) / std::log(rho)) : 1;
    m = std::min(std::max(m, 1) + deg_extra, deg_max);
  }
  m += (m & 1);
  const int cap_even = deg_max - (deg_max & 1);
  return std::min(m, cap_even);
}

struct PhaseTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  double total_ms = 0.0;
  PhaseTimer() { CHASE_CUDA(cudaEventCreate(&a)); CHASE_CUDA(cudaEventCreate(&b)); }
  ~PhaseTimer() { if (a) cudaEventDestroy(a); if (b) cudaEventDestroy(b); }
  void start(cudaStream_t st) { CHASE_CUDA(cudaEventRecord(a, st)); }
  void stop(cudaStream_t st) { CHASE_CUDA(cudaEventRecord(b, st)); }
  void collect() {   // call after the stream has been synchronised
    float ms = 0.f;
    CHASE_CUDA(cudaEventElapsedTime(&ms, a, b));
    total_ms += ms;
  }
};

// Small n x n factorizations: the complex path runs them directly; the real-symmetric path (f2)
// runs the same complex kernels on a complexified copy (the matrices stay real through them).
// G: Gram (upper triangle) on entry; on exit `Rinv` holds R^{-1} in the element type.
template <class T>
bool chol_and_inverse(void* G, void* G2, void* Z, int n, int* d_info, cudaStream_t st, void** Rinv);

template <>
bool chol_and_inverse<double2>(void* G, void* G2, void* Z, int n, int* d_info, cudaStream_t st, void** Rinv) {
  if (!cholesky_upper(G, n, n, d_info, st)) return false;
  trinv_upper(G, n, G2, n, Z, n, st);
  *Rinv = G2;
  return true;
}

template <>
bool chol_and_inverse<double>(void* G, void* G2, void* Z, int n, int* d_info, cudaStream_t st, void** Rinv) {
  double2* Gc = reinterpret_cast<double2*>(G2);
  real_to_complex(Gc, n, reinterpret_cast<const double*>(G), n, n, n, st);
  if (!cholesky_upper(Gc, n, n, d_info, st)) return false;
  trinv_upper(Gc, n, Z, n, G, n, st);                          // G reused as scratch (n^2/2 complex)
  complex_to_real(reinterpret_cast<double*>(G), n, reinterpret_cast<const double2*>(Z), n, n, n, st);
  *Rinv = G;
  return true;
}

// Rayleigh-Ritz eigensolver: G (n x n Hermitian / symmetric, destroyed) -> theta, eigenvectors in *Zout
template <class T>
void rr_eig(chase_handle* h, void* G, void* G2, void* Z, int n, double* theta, cudaStream_t st, void** Zout);

template <>
void rr_eig<double2>(chase_handle* h, void* G, void*, void* Z, int n, double* theta, cudaStream_t st, void** Zout) {
  heev_jacobi(G, n, n, theta, Z, n, st, &h->jacobi);
  *Zout = Z;
}

template <>
void rr_eig<double>(chase_handle* h, void* G, void* G2, void* Z, int n, double* theta, cudaStream_t st, void** Zout) {
  double2* Gc = reinterpret_cast<double2*>(G2);
  real_to_complex(Gc, n, reinterpret_cast<const double*>(G), n, n, n, st);
  heev_jacobi(Gc, n, n, theta, Z, n, st, &h->jacobi);           // real rotations: Z stays real
  complex_to_real(reinterpret_cast<double*>(G), n, reinterpret_cast<const double2*>(Z), n, n, n, st);
  *Zout = G;
}

}  // namespace

template <class T>
static chase_status solve_t(chase_handle* h, const void* Hv, int64_t ldh, int nev, int nex, int deg, double tol,
                            double* ritz_values, void* ritz_vectors, int64_t ldv_out, chase_report* rep) {
  constexpr int ND = SC<T>::ND;
  const Grid& g = h->grid;
  const int64_t p = g.rows.len, q = g.cols.len, r0 = g.rows.start, c0 = g.cols.start;
  const Range I = g.diag();
  const int n_e = nev + nex;
  cudaStream_t st = h->stream;
  const bool largest = h->opt.largest;
  const int deg_max = h->opt.deg_max;

  T* V = h->V.as<T>();
  T* V2 = h->V2.as<T>();
  T* W = h->W.as<T>();
  T* HV = h->HV.as<T>();
  T* G = h->G.as<T>();
  T* G2 = h->G2.as<T>();
  T* Z = h->Z.as<T>();
  // scratch: reduction partials | theta | res2 | perm | info
  const size_t red_doubles = colreduce_scratch(n_e);
  h->red.alloc(sizeof(double) * (red_doubles + 2 * (size_t)n_e) + sizeof(int) * ((size_t)n_e + 8));
  double* part = h->red.as<double>();
  double* d_theta = part + red_doubles;
  double* d_res2 = d_theta + n_e;
  int* d_perm = reinterpret_cast<int*>(d_res2 + n_e);
  int* d_info = d_perm + n_e;

  PhaseTimer t_all, t_lz, t_f, t_qr, t_rr, t_res;
  const bool trace = std::getenv("CHASE_TRACE") != nullptr;   // per-iteration phase trace to stderr
  t_all.start(st);

  // ---- Alg. 1 line 2: Lanczos bounds
  nvtxRangePushA("Lanczos");
  t_lz.start(st);
  LanczosOut lz = lanczos(h, Hv, ldh, n_e);
  t_lz.stop(st);
  nvtxRangePop();
  double b_sup = lz.b_sup, mu_1 = lz.mu_1, mu_ne = lz.mu_ne;
  const double nu = lz.nu > 0.0 ? lz.nu : 1.0;

  // CHASE_C64 (mixed solve): the shard is complex single; every product with it runs on the c64
  // kernels (tcgen05 3xTF32 filter / HQ, FP64-accumulated skinny Lanczos product), the iteration
  // around it (QR, RR, residuals) in complex double on the handle's workspace.
  const bool mixed = h->c64();
  // f4: complex-double solve whose early filters run on a complex-single shadow
  bool f4 = false;
  const void* H32 = nullptr;
  if constexpr (SC<T>::is_complex) {
    if (!mixed && h->opt.mixed_filter > 0.0) {
      H32 = c64_shadow(h, Hv, ldh);
      c64_hlo(h, H32, p);                       // validates the layout up front
      f4 = true;
    }
  }
  constexpr double kC64Floor = 1e-5;            // residual level the c64 filter can reach
  bool f4_next = f4;                             // iteration 1 starts from random vectors
  // ---- initial V-hat (Require of Alg. 1)
  if (h->opt.approx && mixed)
    c64_convert(V, q, true, ritz_vectors, ldv_out, q, n_e, st);
  else if (h->opt.approx)
    copy2d<T>(V, q, ritz_vectors, ldv_out, q, n_e, st);
  else
    random_block(h, V, q, q, c0, 0, n_e, h->opt.seed_v, 0);

  std::vector<int> m(n_e, deg + (deg & 1));                  // line 1 (even)
  std::vector<double> ritz(n_e, 0.0), res(n_e, 0.0), th_h(n_e), r2_h(n_e);
  int locked = 0, it = 0;
  int64_t matvecs = 0;
  double max_resid = 0.0;

  // max_iter = 0 (default, ledger #21 reading revised): iterate while the solve makes progress --
  // a new locked pair, or the smallest active residual below 0.99 x its best so far -- and stop
  // with CHASE_E_MAXITER after stall_iter (100) iterations without progress or kAutoIterCap in
  // total.  (The 1-2-1 family at N = 115000 needs 103 iterations, past a fixed cap of 100, and
  // locks nothing for its first 55: a 30-iteration / 10 % rule stopped it there.)
  constexpr int kAutoIterCap = 5000;
  const bool auto_iter = h->opt.max_iter <= 0;
  const int max_it = auto_iter ? kAutoIterCap : h->opt.max_iter;
  int last_progress = 0;
  double best_res = 1e300;
  while (locked < nev && it < max_it) {                          // line 3
    ++it;
    const int n_act = n_e - locked;
    T* Va = V + (int64_t)locked * q;
    T* Wa = W + (int64_t)locked * p;
    T* HVa = HV + (int64_t)locked * p;

    // ---- line 4: Filter
    nvtxRangePushA("Filter");
    t_f.start(st);
    const bool f4_now = f4 && f4_next;
    if constexpr (SC<T>::is_complex) {
      if (mixed)
        matvecs += c64_filter_mixed(h, Hv, ldh, Va, q, n_act, m.data() + locked, b_sup, mu_1, mu_ne);
      else if (f4_now)
        matvecs += c64_filter_mixed(h, H32, p, Va, q, n_act, m.data() + locked, b_sup, mu_1, mu_ne);
      else
        matvecs += filter(h, Hv, ldh, Va, q, Wa, p, n_act, m.data() + locked, b_sup, mu_1, mu_ne);
    } else {
      matvecs += filter(h, Hv, ldh, Va, q, Wa, p, n_act, m.data() + locked, b_sup, mu_1, mu_ne);
    }
    t_f.stop(st);
    nvtxRangePop();

    // ---- line 5: QR([Y V]) -- CGS2 against the locked Y, then CholQR2 (shifted fallback)
    nvtxRangePushA("QR");
    t_qr.start(st);
    for (int pass = 0; pass < 2 && locked > 0; ++pass) {
      ZgemmDesc d;                                  // T = Y^H Va   (locked x n_act)
      d.use3m = h->opt.gemm3m;
      d.M = locked; d.N = n_act; d.K = (int)q; d.conjA = true;
      d.A = V; d.lda = q; d.B = Va; d.ldb = q; d.C = G2; d.ldc = locked;
      gemm(h, d);
      allreduce_doubles(h, h->rowc, reinterpret_cast<double*>(G2), ND * (size_t)locked * n_act);
      ZgemmDesc e;                                  // Va -= Y T
      e.use3m = h->opt.gemm3m;
      e.M = (int)q; e.N = n_act; e.K = locked;
      e.A = V; e.lda = q; e.B = G2; e.ldb = locked; e.C = Va; e.ldc = q;
      e.alpha = -1.0; e.beta = 1.0;
      gemm(h, e);
    }
    int cholqr_passes = 2;
    for (int pass = 0; pass < cholqr_passes; ++pass) {
      auto gram = [&]() {
        ZgemmDesc d;                                // G = Va^H Va
        d.use3m = h->opt.gemm3m;
        d.M = n_act; d.N = n_act; d.K = (int)q; d.conjA = true;
        d.upper_only = true;                        // Cholesky reads the upper triangle only
        d.A = Va; d.lda = q; d.B = Va; d.ldb = q; d.C = G; d.ldc = n_act;
        gemm(h, d);
        allreduce_doubles(h, h->rowc, reinterpret_cast<double*>(G), ND * (size_t)n_act * n_act);
      };
      gram();
      void* Rinv = nullptr;
      if (!chol_and_inverse<T>(G, G2, Z, n_act, d_info, st, &Rinv)) {
        // shifted CholQR (Fukaya et al.): G + s I with s = 11 (N n + n(n+1)) u ||G||, then two
        // more unshifted passes (CholQR3)
        gram();
        std::vector<T> dg(n_act);
        CHASE_CUDA(cudaMemcpy2DAsync(dg.data(), sizeof(T), G, sizeof(T) * (n_act + 1), sizeof(T), n_act,
                                     cudaMemcpyDeviceToHost, st));
        sync_stream(h, st);
        double trace = 0.0;
        for (auto& v : dg) trace += SC<T>::re(v);
        const double s = 11.0 * ((double)g.N * n_act + (double)n_act * (n_act + 1)) * 1.1102230246251565e-16 * trace;
        add_diag<T>(G, n_act, n_act, s, st);
        if (!chol_and_inverse<T>(G, G2, Z, n_act, d_info, st, &Rinv))
          throw NumericError("CholQR failed even with the shifted fallback");
        cholqr_passes = 3;
      }
      ZgemmDesc d;                                  // V2 = Va R^{-1}
      d.use3m = h->opt.gemm3m;
      d.M = (int)q; d.N = n_act; d.K = n_act;
      d.b_upper = true;                             // R^{-1} is upper triangular
      d.A = Va; d.lda = q; d.B = Rinv; d.ldb = n_act; d.C = V2; d.ldc = q;
      gemm(h, d);
      copy2d<T>(Va, q, V2, q, q, n_act, st);
    }
    t_qr.stop(st);
    nvtxRangePop();

    // ---- line 6: Rayleigh-Ritz
    nvtxRangePushA("RR");
    t_rr.start(st);
    if constexpr (SC<T>::is_complex) {
      if (mixed)
        c64_forward_mixed(h, Hv, ldh, Va, q, HVa, p, n_act);              // HQ (W-layout)
      else
        hemm_step(h, 0, Hv, ldh, Va, q, HVa, p, n_act, 1.0, 0.0, 0.0);
    } else {
      hemm_step(h, 0, Hv, ldh, Va, q, HVa, p, n_act, 1.0, 0.0, 0.0);    // HQ (W-layout)
    }
    if (I.len > 0) {
      ZgemmDesc d;                                  // G = Q[I]^H HQ[I]
      d.use3m = h->opt.gemm3m;
      d.M = n_act; d.N = n_act; d.K = (int)I.len; d.conjA = true;
      d.A = Va + (I.start - c0); d.lda = q;
      d.B = HVa + (I.start - r0); d.ldb = p;
      d.C = G; d.ldc = n_act;
      gemm(h, d);
    } else {
      zero2d<T>(G, n_act, n_act, n_act, st);
    }
    allreduce_doubles(h, h->world, reinterpret_cast<double*>(G), ND * (size_t)n_act * n_act);
    hermitize<T>(G, n_act, n_act, st);
    void* Zr = nullptr;
    rr_eig<T>(h, G, G2, Z, n_act, d_theta, st, &Zr);
    {
      ZgemmDesc d;                                  // V <- Q Z
      d.use3m = h->opt.gemm3m;
      d.M = (int)q; d.N = n_act; d.K = n_act;
      d.A = Va; d.lda = q; d.B = Zr; d.ldb = n_act; d.C = V2; d.ldc = q;
      gemm(h, d);
      copy2d<T>(Va, q, V2, q, q, n_act, st);
      ZgemmDesc e;                                  // HV <- (HQ) Z   (into W, then swap roles)
      e.use3m = h->opt.gemm3m;
      e.M = (int)p; e.N = n_act; e.K = n_act;
      e.A = HVa; e.lda = p; e.B = Zr; e.ldb = n_act; e.C = Wa; e.ldc = p;
      gemm(h, e);
    }
    t_rr.stop(st);
    nvtxRangePop();

    // ---- line 7: residuals  ||H v - theta v|| over I_ij, summed over the world
    nvtxRangePushA("Resid");
    t_res.start(st);
    if (I.len > 0)
      resid_norms2<T>(Wa + (I.start - r0), p, Va + (I.start - c0), q, d_theta, I.len, n_act, d_res2, part, st);
    else
      CHASE_CUDA(cudaMemsetAsync(d_res2, 0, sizeof(double) * n_act, st));
    allreduce_doubles(h, h->world, d_res2, n_act);
    t_res.stop(st);
    nvtxRangePop();
    CHASE_CUDA(cudaMemcpyAsync(th_h.data(), d_theta, sizeof(double) * n_act, cudaMemcpyDeviceToHost, st));
    CHASE_CUDA(cudaMemcpyAsync(r2_h.data(), d_res2, sizeof(double) * n_act, cudaMemcpyDeviceToHost, st));
    sync_stream(h, st);
    const double f0 = t_f.total_ms, q0 = t_qr.total_ms, r0_ = t_rr.total_ms, s0 = t_res.total_ms;
    t_f.collect(); t_qr.collect(); t_rr.collect(); t_res.collect();
    for (int a = 0; a < n_act; ++a) {
      ritz[locked + a] = th_h[a];
      res[locked + a] = std::sqrt(std::max(0.0, r2_h[a])) / nu;
    }
    if (trace && g.rank == 0 && f4) std::fprintf(stderr, "[chase] it=%d filter=%s\n", it, f4_now ? "c64" : "c128");
    if (trace && g.rank == 0) {
      double rmin = 1e300, rmax = 0.0;
      for (int a = 0; a < n_act; ++a) { rmin = std::min(rmin, res[locked + a]); rmax = std::max(rmax, res[locked + a]); }
      std::fprintf(stderr, "[chase] it=%d n_act=%d locked_before=%d matvecs=%lld filter=%.3fs qr=%.3fs rr=%.3fs resid=%.4fs "
                   "res[0]=%.2e res_min=%.2e res_max=%.2e\n",
                   it, n_act, locked, (long long)matvecs, (t_f.total_ms - f0) * 1e-3, (t_qr.total_ms - q0) * 1e-3,
                   (t_rr.total_ms - r0_) * 1e-3, (t_res.total_ms - s0) * 1e-3, res[locked], rmin, rmax);
    }
    // ---- line 8: deflation & locking (prefix-contiguous in Ritz order, ledger #15)
    int nl = 0;
    while (nl < n_act && res[locked + nl] <= tol) ++nl;
    locked += nl;
    {
      double rmin = 1e300;
      for (int a = locked; a < n_e; ++a) rmin = std::min(rmin, res[a]);
      if (nl > 0 || rmin < 0.99 * best_res) last_progress = it;
      best_res = std::min(best_res, rmin);
    }
    if (auto_iter && locked < nev && it - last_progress >= h->opt.stall_iter) break;
    // ---- line 9-10: bounds and interval
    mu_1 = *std::min_element(ritz.begin(), ritz.end());
    mu_ne = *std::max_element(ritz.begin(), ritz.end());
    const double c = 0.5 * (b_sup + mu_ne), e = 0.5 * (b_sup - mu_ne);
    if (locked >= nev) break;
    // f4: next filter in complex single while every active residual is above the threshold;
    // its degrees then aim at what complex single can reach
    double tol_deg = tol;
    if (f4) {
      double rmin = 1e300;
      for (int a = locked; a < n_e; ++a) rmin = std::min(rmin, res[a]);
      f4_next = rmin > h->opt.mixed_filter;
      if (f4_next) tol_deg = std::max(tol, kC64Floor);
    }
    // ---- lines 11-14: degrees, stable sort by degree
    const int na = n_e - locked;
    std::vector<int> mm(na), perm(na);
    for (int a = 0; a < na; ++a) mm[a] = optimal_degree(tol_deg, res[locked + a], ritz[locked + a], c, e, deg_max, h->opt.deg_extra);
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return mm[x] < mm[y]; });
    std::vector<double> rz(na), rs(na);
    for (int a = 0; a < na; ++a) {
      m[locked + a] = mm[perm[a]];
      rz[a] = ritz[locked + perm[a]];
      rs[a] = res[locked + perm[a]];
    }
    for (int a = 0; a < na; ++a) { ritz[locked + a] = rz[a]; res[locked + a] = rs[a]; }
    CHASE_CUDA(cudaMemcpyAsync(d_perm, perm.data(), sizeof(int) * na, cudaMemcpyHostToDevice, st));
    permute_cols<T>(V2, q, V + (int64_t)locked * q, q, q, d_perm, na, st);
    copy2d<T>(V + (int64_t)locked * q, q, V2, q, q, na, st);
    sync_stream(h, st);   // perm (host) goes out of scope
  }

  // ---- results: nev smallest locked Ritz pairs, ascending
  const int k = locked >= nev ? locked : n_e;
  std::vector<int> order(k);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return ritz[x] < ritz[y]; });
  order.resize(nev);
  std::vector<int> out_cols(nev);
  for (int i = 0; i < nev; ++i) {
    const int src = largest ? order[nev - 1 - i] : order[i];
    ritz_values[i] = largest ? -ritz[src] : ritz[src];
    out_cols[i] = src;
    max_resid = std::max(max_resid, res[src]);
  }
  CHASE_CUDA(cudaMemcpyAsync(d_perm, out_cols.data(), sizeof(int) * nev, cudaMemcpyHostToDevice, st));
  if (mixed) {
    permute_cols<T>(V2, q, V, q, q, d_perm, nev, st);
    c64_convert(ritz_vectors, ldv_out, false, V2, q, q, nev, st);
  } else {
    permute_cols<T>(ritz_vectors, ldv_out, V, q, q, d_perm, nev, st);
  }
  t_all.stop(st);
  sync_stream(h, st);
  t_all.collect();
  t_lz.collect();
  if (rep) {
    rep->iterations = it;
    rep->locked = locked;
    rep->matvecs = matvecs;
    rep->filter_flops = (SC<T>::is_complex ? 8.0 : 2.0) * (double)g.N * (double)g.N * (double)matvecs;
    rep->t_all = t_all.total_ms * 1e-3;
    rep->t_lanczos = t_lz.total_ms * 1e-3;
    rep->t_filter = t_f.total_ms * 1e-3;
    rep->t_qr = t_qr.total_ms * 1e-3;
    rep->t_rr = t_rr.total_ms * 1e-3;
    rep->t_resid = t_res.total_ms * 1e-3;
    rep->b_sup = largest ? -b_sup : b_sup;
    rep->mu_1 = mu_1;
    rep->mu_ne = mu_ne;
    rep->nu = nu;
    rep->max_resid = max_resid;
  }
  if (locked < nev) {
    const std::string why = auto_iter && it < max_it
                                ? "no progress in stall_iter iterations: stopped after " + std::to_string(it) + " iterations with "
                                : std::string("max_iter reached with ");
    h->err = why + std::to_string(locked) + " of " + std::to_string(nev) + " pairs locked";
    return CHASE_E_MAXITER;
  }
  return CHASE_OK;
}

chase_status solve(chase_handle* h, const void* Hv, int64_t ldh, int nev, int nex, int deg, double tol,
                   double* ritz_values, void* ritz_vectors, int64_t ldv_out, chase_report* rep) {
  if (h->real())
    return solve_t<double>(h, Hv, ldh, nev, nex, deg, tol, ritz_values, ritz_vectors, ldv_out, rep);
  return solve_t<double2>(h, Hv, ldh, nev, nex, deg, tol, ritz_values, ritz_vectors, ldv_out, rep);
}

}  // namespace chase
