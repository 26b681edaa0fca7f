// Spectral bounds by repeated Lanczos + DoS (Alg. 1 line 2; ledger #14).
//
// L runs (default 4) of m steps (default 25) advance together as one N x L block.  Lanczos
// vectors are kept full length and replicated on every rank (N x L x (m+1) complex, tiny next to
// H): the product with H is this rank's shard GEMM H_ij X[cols j] written into rows i of a zeroed
// N x L buffer, followed by one world all-reduce -- so each step streams the H shard once.  All
// vector work (projections for full reorthogonalisation, norms) runs on the device with fixed-order
// reductions; the host only diagonalises the m x m tridiagonal T_m per run and applies the DoS
// rule: b_sup = max_r(theta_max + |beta_m|), mu_1 = min theta, mu_ne = smallest pooled theta whose
// cumulative weight (|z_1k|^2 / L) reaches n_e/N, nu = max |theta|; guard of S:478.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>
#include "dense.h"
#include "handle.h"
#include "scalar.cuh"

namespace chase {

namespace {
// h[k*L + r] = Q_k[:, r]^H F[:, r] for k <= j (2 doubles each: re, im); pass 1 of 2
template <class T>
__global__ void k_proj_p1(const T* Q, int64_t N, int L, int nk, const T* F, int chunks, double* part) {
  __shared__ double sh[2][256];
  const int col = blockIdx.x;          // col = k*L + r
  const int r = col % L, chunk = blockIdx.y;
  const int64_t len = (N + chunks - 1) / chunks;
  const int64_t i0 = chunk * len, i1 = min(N, i0 + len);
  const T* q = Q + (int64_t)col * N;
  const T* f = F + (int64_t)r * N;
  double re = 0.0, im = 0.0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += 256) {
    const T d = SC<T>::mulc(q[i], f[i]);
    re += SC<T>::re(d);
    im += SC<T>::im(d);
  }
  sh[0][threadIdx.x] = re;
  sh[1][threadIdx.x] = im;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) { sh[0][threadIdx.x] += sh[0][threadIdx.x + s]; sh[1][threadIdx.x] += sh[1][threadIdx.x + s]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[((int64_t)col * chunks + chunk) * 2] = sh[0][0];
    part[((int64_t)col * chunks + chunk) * 2 + 1] = sh[1][0];
  }
}

__global__ void k_proj_p2(const double* part, int chunks, int ncols, double* h) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ncols) return;
  double re = 0.0, im = 0.0;
  for (int c = 0; c < chunks; ++c) { re += part[((int64_t)col * chunks + c) * 2]; im += part[((int64_t)col * chunks + c) * 2 + 1]; }
  h[2 * col] = re;
  h[2 * col + 1] = im;
}

// F[:, r] -= sum_k Q_k[:, r] h[k*L + r]
template <class T>
__global__ void k_proj_sub(const T* Q, int64_t N, int L, int nk, const double* h, T* F) {
  const int64_t total = N * L;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % N;
    const int r = (int)(idx / N);
    T f = F[i + (int64_t)r * N];
    for (int k = 0; k < nk; ++k) {
      const T q = Q[i + (int64_t)(k * L + r) * N];
      f = SC<T>::sub(f, SC<T>::mul(q, SC<T>::make(h[2 * (k * L + r)], h[2 * (k * L + r) + 1])));
    }
    F[i + (int64_t)r * N] = f;
  }
}

// Q_next[:, r] = F[:, r] / beta_r  (0 if beta_r is 0); dots = squared norms (real parts)
template <class T>
__global__ void k_normalize(const T* F, int64_t N, int L, const double* dots, T* Qn) {
  const int64_t total = N * L;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / N);
    const double b2 = dots[2 * r];
    const double sc = b2 > 0.0 ? 1.0 / sqrt(b2) : 0.0;
    Qn[idx] = SC<T>::scale(F[idx], sc);
  }
}

// Jacobi eigen-decomposition of a small real symmetric matrix (host; m <= a few dozen).
void host_syev(int m, std::vector<double>& A, std::vector<double>& Z) {
  Z.assign((size_t)m * m, 0.0);
  for (int i = 0; i < m; ++i) Z[i * m + i] = 1.0;
  auto a = [&](int i, int j) -> double& { return A[(size_t)i * m + j]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) { tot += a(i, j) * a(i, j); if (i != j) off += a(i, j) * a(i, j); }
    if (off <= 1e-32 * tot) break;
    for (int p = 0; p < m - 1; ++p)
      for (int q = p + 1; q < m; ++q) {
        const double apq = a(p, q);
        if (std::fabs(apq) < 1e-300) continue;
        const double tau = (a(q, q) - a(p, p)) / (2.0 * apq);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (std::fabs(tau) + std::hypot(1.0, tau));
        const double c = 1.0 / std::hypot(1.0, t), s = t * c;
        for (int k = 0; k < m; ++k) {   // columns
          const double xp = a(k, p), xq = a(k, q);
          a(k, p) = c * xp - s * xq;
          a(k, q) = s * xp + c * xq;
        }
        for (int k = 0; k < m; ++k) {   // rows
          const double yp = a(p, k), yq = a(q, k);
          a(p, k) = c * yp - s * yq;
          a(q, k) = s * yp + c * yq;
        }
        for (int k = 0; k < m; ++k) {
          const double zp = Z[(size_t)k * m + p], zq = Z[(size_t)k * m + q];
          Z[(size_t)k * m + p] = c * zp - s * zq;
          Z[(size_t)k * m + q] = s * zp + c * zq;
        }
      }
  }
}
}  // namespace

template <class T>
static LanczosOut lanczos_t(chase_handle* h, const void* H, int64_t ldh, int n_e) {
  const Grid& g = h->grid;
  const int64_t N = g.N;
  const int L = h->opt.lanczos_runs;
  const int m = (int)std::min<int64_t>(h->opt.lanczos_steps, N);
  cudaStream_t st = h->stream;
  const double hsign = h->opt.largest ? -1.0 : 1.0;
  // buffers: Q (N x L x (m+1)), F (N x L), part, h coefficients, per-step dots
  const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(32, (N + 8191) / 8192));
  const size_t qbytes = sizeof(T) * (size_t)N * L * (m + 1), fbytes = sizeof(T) * (size_t)N * L;
  const size_t pbytes = sizeof(double) * 2 * (size_t)chunks * L * (m + 1);
  const size_t hbytes = sizeof(double) * 2 * (size_t)L * (m + 1);
  h->lz.alloc(qbytes + fbytes + pbytes + hbytes * (2 * (m + 1) + 2) + 256);
  char* base = h->lz.as<char>();
  T* Q = reinterpret_cast<T*>(base);
  T* F = reinterpret_cast<T*>(base + qbytes);
  double* part = reinterpret_cast<double*>(base + qbytes + fbytes);
  double* hc = reinterpret_cast<double*>(base + qbytes + fbytes + pbytes);         // per pass
  double* alpha_hist = hc + 2 * L * (m + 1);                                        // (m+1) x L x 2
  double* beta_hist = alpha_hist + 2 * (size_t)L * (m + 1);                         // (m+1) x L x 2

  h->scratch.alloc(skinny_work_bytes((int)g.rows.len, (int)g.cols.len, std::min(L, 8)) + 256);
  auto dots_into = [&](const T* X, int nk, const T* Y, double* out) {
    const int ncols = nk * L;
    k_proj_p1<T><<<dim3(ncols, chunks), 256, 0, st>>>(X, N, L, nk, Y, chunks, part);
    CHASE_CHECK_LAUNCH();
    k_proj_p2<<<(ncols + 127) / 128, 128, 0, st>>>(part, chunks, ncols, out);
    CHASE_CHECK_LAUNCH();
  };
  const int eblocks = (int)std::min<int64_t>((N * L + 255) / 256, 148 * 16);

  // start block: counter-based generator, stream 1, normalised
  random_block(h, Q, N, N, 0, 0, L, h->opt.seed_lanczos, 1);
  dots_into(Q, 1, Q, hc);
  k_normalize<T><<<eblocks, 256, 0, st>>>(Q, N, L, hc, Q);
  CHASE_CHECK_LAUNCH();

  for (int j = 0; j < m; ++j) {
    T* Qj = Q + (size_t)j * N * L;
    // F = H Q_j  (rows of block i from this shard; world sum assembles the full vectors)
    CHASE_CUDA(cudaMemsetAsync(F, 0, fbytes, st));
    if (h->c64() && !(L == 1 || L == 2 || L == 3 || L == 4 || L == 8))
      throw UsageError("CHASE_C64: lanczos_runs must be 1, 2, 3, 4 or 8");
    if (L == 1 || L == 2 || L == 3 || L == 4 || L == 8) {
      // HBM-bound skinny product: streams the shard once per step
      if (SC<T>::is_complex)
        zgemm_skinny((int)g.rows.len, L, (int)g.cols.len, hsign, H, ldh, Qj + g.cols.start, N,
                     F + g.rows.start, N, h->scratch.p, st, h->c64());
      else
        dgemm_skinny((int)g.rows.len, L, (int)g.cols.len, hsign, H, ldh, Qj + g.cols.start, N,
                     F + g.rows.start, N, h->scratch.p, st);
    } else {
      ZgemmDesc d;
      d.M = (int)g.rows.len; d.N = L; d.K = (int)g.cols.len;
      d.A = H; d.lda = ldh;
      d.B = Qj + g.cols.start; d.ldb = N;
      d.C = F + g.rows.start; d.ldc = N;
      d.alpha = hsign; d.beta = 0.0;
      gemm(h, d);
    }
    allreduce_doubles(h, h->world, reinterpret_cast<double*>(F), SC<T>::ND * (size_t)N * L);
    // two classical Gram-Schmidt passes against Q_0..Q_j (full reorthogonalisation); the first
    // pass's coefficient on Q_j is alpha_j = Re(q_j^H H q_j)
    dots_into(Q, j + 1, F, hc);
    CHASE_CUDA(cudaMemcpyAsync(alpha_hist + 2 * (size_t)j * L, hc + 2 * (size_t)j * L, sizeof(double) * 2 * L,
                               cudaMemcpyDeviceToDevice, st));
    k_proj_sub<T><<<eblocks, 256, 0, st>>>(Q, N, L, j + 1, hc, F);
    CHASE_CHECK_LAUNCH();
    dots_into(Q, j + 1, F, hc);
    k_proj_sub<T><<<eblocks, 256, 0, st>>>(Q, N, L, j + 1, hc, F);
    CHASE_CHECK_LAUNCH();
    double* dn = beta_hist + 2 * (size_t)j * L;
    dots_into(F, 1, F, dn);
    k_normalize<T><<<eblocks, 256, 0, st>>>(F, N, L, dn, Q + (size_t)(j + 1) * N * L);
    CHASE_CHECK_LAUNCH();
  }
  std::vector<double> ah(2 * (size_t)L * m), bh(2 * (size_t)L * m);
  CHASE_CUDA(cudaMemcpyAsync(ah.data(), alpha_hist, sizeof(double) * ah.size(), cudaMemcpyDeviceToHost, st));
  CHASE_CUDA(cudaMemcpyAsync(bh.data(), beta_hist, sizeof(double) * bh.size(), cudaMemcpyDeviceToHost, st));
  CHASE_CUDA(cudaStreamSynchronize(st));

  std::vector<double> ritz, wts;
  double b_sup = -INFINITY;
  for (int r = 0; r < L; ++r) {
    std::vector<double> al, be;
    for (int j = 0; j < m; ++j) {
      const double a = ah[2 * ((size_t)j * L + r)];
      const double b = std::sqrt(std::max(0.0, bh[2 * ((size_t)j * L + r)]));
      al.push_back(a);
      be.push_back(b);
      if (j + 1 < m && b <= 1e-14 * std::max(1.0, std::fabs(a))) break;   // invariant subspace
    }
    const int k = (int)al.size();
    std::vector<double> Tm((size_t)k * k, 0.0), Z;
    for (int i = 0; i < k; ++i) {
      Tm[(size_t)i * k + i] = al[i];
      if (i + 1 < k) Tm[(size_t)i * k + i + 1] = Tm[(size_t)(i + 1) * k + i] = be[i];
    }
    host_syev(k, Tm, Z);
    double thmax = -INFINITY;
    for (int i = 0; i < k; ++i) {
      const double th = Tm[(size_t)i * k + i];
      thmax = std::max(thmax, th);
      ritz.push_back(th);
      wts.push_back(Z[i] * Z[i] / L);          // |z_1i|^2 / L (first row of Z)
    }
    b_sup = std::max(b_sup, thmax + std::fabs(be[k - 1]));
  }
  std::vector<int> order(ritz.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ritz[a] < ritz[b]; });
  LanczosOut o;
  o.mu_1 = ritz[order[0]];
  const double q = (double)n_e / (double)N - 1e-15;
  double cdf = 0.0;
  size_t idx = order.size() - 1;
  for (size_t t = 0; t < order.size(); ++t) {
    cdf += wts[order[t]];
    if (cdf >= q) { idx = t; break; }
  }
  o.mu_ne = ritz[order[idx]];
  if (o.mu_ne >= b_sup - 1e-12 * std::max(1.0, std::fabs(b_sup))) b_sup += std::max(1.0, std::fabs(b_sup)) * 1e-8;
  o.b_sup = b_sup;
  double nu = 0.0;
  for (double t : ritz) nu = std::max(nu, std::fabs(t));
  o.nu = nu;
  return o;
}

LanczosOut lanczos(chase_handle* h, const void* H, int64_t ldh, int n_e) {
  return h->real() ? lanczos_t<double>(h, H, ldh, n_e) : lanczos_t<double2>(h, H, ldh, n_e);
}

}  // namespace chase
