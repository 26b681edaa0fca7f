// Hermitian eigensolver for the Rayleigh-Ritz quotient G = Q^H A Q (Alg. 1 line 6)
// on the device: block-cyclic two-sided Jacobi.
//
// The paper diagonalises G on the CPU with LAPACK divide & conquer.  Here it stays on
// the GPU: the index set is split into 2b blocks of 32; each round pairs the blocks (circle
// method) and, for every pair (P, Q), one CTA diagonalises the 64 x 64 subproblem
// G[P u Q, P u Q] by cyclic Jacobi in shared memory (32 disjoint rotations per parallel step).
// The resulting 64 x 64 unitaries U_k are then applied as G <- U^H G U with one 64 x 64 tile
// product per (l <= k) block pair (Hermitian symmetry halves the work) and Z <- Z U.  Converged
// when off(G)_F <= 1e-15 ||G||_F.  Deterministic (no atomics), so every rank that runs it
// redundantly on identical inputs gets identical bits (ledger #20).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>
#include "common.cuh"
#include "dense.h"
#include "tma.cuh"
#include "handle.h"
#include "linalg.h"

namespace chase {

namespace {
constexpr int W = 32;            // block width
constexpr int S = 2 * W;         // subproblem size
constexpr int LD = S + 1;        // padded smem row stride (complex)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {   // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

__device__ __forceinline__ int64_t gidx(const int* pairs, int k, int t) {
  // global index of local index t (0..63) of pair k: blocks P = pairs[2k], Q = pairs[2k+1]
  return (int64_t)(t < W ? pairs[2 * k] * W + t : pairs[2 * k + 1] * W + (t - W));
}

// A = pad(G): A[0:n,0:n] = G, padded diagonal = distinct values above the spectrum; Z = I.
__global__ void k_pad_init(const double2* G, int64_t ldg, int n, double2* A, double2* Z, int np, double padbase) {
  const int64_t total = (int64_t)np * np;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % np), j = (int)(idx / np);
    double2 v = make_double2(0.0, 0.0);
    if (i < n && j < n) v = G[i + (int64_t)j * ldg];
    else if (i == j) v = make_double2(padbase * (1.0 + (double)(i - n) / np), 0.0);
    A[idx] = v;
    Z[idx] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
}

// pair i of parallel step r of the circle method over S players (player S-1 fixed), p < q
__device__ __forceinline__ void pair_of(int r, int i, int& p, int& q) {
  if (i == 0) { p = r; q = S - 1; }
  else { p = (r + i) % (S - 1); q = (r - i + (S - 1)) % (S - 1); }
  if (p > q) { const int tmp = p; p = q; q = tmp; }
}

// U <- U J for one parallel step: items (row i, pair cb), 64 x 32 of them, item0, item0 + stride,
// ... (at most 3 per thread: all loads first, so the items' latencies overlap)
__device__ __forceinline__ void jacobi_u_update(double2* Um, const double* rc, const double* rs, const double2* rph,
                                                const int* rp, const int* rq, int item0, int stride) {
  constexpr int LD_ = 2 * 32 + 1;
  double2 xp[3], xq[3];
  int at[3][2];
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int idx = item0 + u * stride;
    if (idx < 64 * 32) {
      const int i = idx >> 5, cb = idx & 31;
      at[u][0] = i * LD_ + rp[cb];
      at[u][1] = i * LD_ + rq[cb];
      xp[u] = Um[at[u][0]];
      xq[u] = Um[at[u][1]];
    }
  }
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int idx = item0 + u * stride;
    if (idx < 64 * 32) {
      const int cb = idx & 31;
      const double cc = rc[cb], sc = rs[cb];
      const double2 q = cmul(rph[cb], xq[u]);
      Um[at[u][0]] = make_double2(cc * xp[u].x - sc * q.x, cc * xp[u].y - sc * q.y);
      Um[at[u][1]] = make_double2(sc * xp[u].x + cc * q.x, sc * xp[u].y + cc * q.y);
    }
  }
}

// One CTA per pair: diagonalise the 64 x 64 Hermitian subproblem by cyclic Jacobi; write U_k.
constexpr int SUB_T = 1024;
constexpr int NTRI = W * (W + 1) / 2;   // pair blocks (ra <= cb) of one parallel step
__global__ void __launch_bounds__(SUB_T) k_sub_eig(const double2* A, int np, const int* pairs, double2* U, int max_inner) {
  extern __shared__ double2 sm[];
  double2* Sm = sm;              // S x LD
  double2* Um = sm + S * LD;     // S x LD
  __shared__ double rcb[2][W], rsb[2][W];     // rotations of steps r (buffer r & 1) and r - 1
  __shared__ double2 rphb[2][W];
  __shared__ int rpb[2][W], rqb[2][W];
  __shared__ double red[SUB_T];
  const int k = blockIdx.x, t = threadIdx.x;
  for (int idx = t; idx < S * S; idx += SUB_T) {
    const int i = idx % S, j = idx / S;
    Sm[i * LD + j] = A[gidx(pairs, k, i) + gidx(pairs, k, j) * np];
    Um[i * LD + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  const int pr = t >> 5, sub = t & 31;    // warp, lane
  // thread t < NTRI owns the pair block (tri_r, tri_c), tri_r <= tri_c (row-major upper triangle)
  int tri_r = 0, tri_c = 0;
  if (t < NTRI) {
    int rem = t;
    while (rem >= W - tri_r) { rem -= W - tri_r; ++tri_r; }
    tri_c = tri_r + rem;
  }
  __shared__ int nrot;
  if (t == 0) nrot = 0;
  __syncthreads();
  for (int sweep = 0; sweep < max_inner; ++sweep) {
    // convergence test: off-diagonal Frobenius norm vs total
    double off = 0.0, tot = 0.0;
    for (int idx = t; idx < S * S; idx += SUB_T) {
      const int i = idx % S, j = idx / S;
      const double2 v = Sm[i * LD + j];
      const double m2 = v.x * v.x + v.y * v.y;
      tot += m2;
      if (i != j) off += m2;
    }
    // fixed-order (deterministic) reduction: xor-shuffle within warps, then warp 0 over the 32
    // warp sums
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if ((t & 31) == 0) { red[t >> 5] = off; red[32 + (t >> 5)] = tot; }
    __syncthreads();
    if (t < 32) {
      double a = red[t], b = red[32 + t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      if (t == 0) { red[64] = a; red[65] = b; }
    }
    __syncthreads();
    const double offs = red[64], tots = red[65];
    __syncthreads();
    if (offs <= 1e-32 * tots || offs == 0.0) break;
    if (sweep > 0 && nrot == 0) break;          // previous sweep found nothing above threshold
    __syncthreads();
    if (t == 0) nrot = 0;
    __syncthreads();
    // Per parallel step r: (A) warp 0 computes the 32 rotations of step r from S while warps
    // 1..31 apply the rotations of step r - 1 to U (U's update only feeds the output, so it runs
    // one step behind, under the rotation math); (B) S <- J_r^H S J_r.
    for (int r = 0; r < S - 1; ++r) {
      if (pr == 0) {
        // circle method: player S-1 fixed; pair 0 = (r, S-1); pair i = ((r+i) % 63, (r-i+63) % 63);
        // lane i: pair i
        int p, q;
        pair_of(r, sub, p, q);
        const double a = Sm[p * LD + p].x, d = Sm[q * LD + q].x;
        const double2 b = Sm[p * LD + q];
        const double ab2 = b.x * b.x + b.y * b.y;          // |a_pq|^2 <= ||G||_F^2: no overflow
        double c = 1.0, s = 0.0;
        double2 ph = make_double2(1.0, 0.0);               // e^{-i phi}
        // rotate only if |a_pq| is significant relative to the diagonal (Demmel-Veselic):
        // |a_pq| > 2e-16 sqrt(|a_pp a_qq|)
        const bool rot = ab2 >= 2.2250738585072014e-308 && ab2 > 4e-32 * fabs(a) * fabs(d);   // ab2 normal
        if (rot) {
          const double inv = rsqrt(ab2);                   // 1 / |a_pq|
          const double tau = 0.5 * (d - a) * inv;
          const double at = fabs(tau);
          // t = sign(tau) / (|tau| + sqrt(1 + tau^2)) (the smaller root; 1 / (2 tau) once tau^2 overflows)
          const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (at > 1e150 ? 2.0 * at : at + sqrt(1.0 + tau * tau));
          c = rsqrt(1.0 + tt * tt);
          s = tt * c;
          ph = make_double2(b.x * inv, -b.y * inv);
        }
        const unsigned nr = __popc(__ballot_sync(0xffffffffu, rot));
        if (sub == 0) nrot += (int)nr;
        const int o = r & 1;
        rcb[o][sub] = c; rsb[o][sub] = s; rphb[o][sub] = ph; rpb[o][sub] = p; rqb[o][sub] = q;
      } else if (r > 0) {
        jacobi_u_update(Um, rcb[(r - 1) & 1], rsb[(r - 1) & 1], rphb[(r - 1) & 1], rpb[(r - 1) & 1],
                        rqb[(r - 1) & 1], t - 32, SUB_T - 32);
      }
      __syncthreads();
      // The 32 rotations are disjoint, so S' = J^H S J splits into 2 x 2 blocks (rows of pair ra,
      // columns of pair cb; J = [[c, s], [-s e^{-i phi}, c e^{-i phi}]] on (p, q)).  S stays
      // Hermitian: threads 0..527 take the blocks ra <= cb (columns first, then rows -- the order of
      // the two-pass form) and store the mirror block as its conjugate transpose.
      if (t < NTRI) {
        const int o = r & 1;
        const int ra = tri_r, cb = tri_c;
        const int pa = rpb[o][ra], qa = rqb[o][ra], pb = rpb[o][cb], qb = rqb[o][cb];
        const double ca = rcb[o][ra], sa = rsb[o][ra], cc = rcb[o][cb], sc = rsb[o][cb];
        const double2 pha = make_double2(rphb[o][ra].x, -rphb[o][ra].y), phb = rphb[o][cb];
        double2 e[2][2] = {{Sm[pa * LD + pb], Sm[pa * LD + qb]}, {Sm[qa * LD + pb], Sm[qa * LD + qb]}};
#pragma unroll
        for (int x = 0; x < 2; ++x) {          // columns:  x_p' = c x_p - s e^{-i phi} x_q ; x_q' = s x_p + c e^{-i phi} x_q
          const double2 xp = e[x][0], xq = cmul(phb, e[x][1]);
          e[x][0] = make_double2(cc * xp.x - sc * xq.x, cc * xp.y - sc * xq.y);
          e[x][1] = make_double2(sc * xp.x + cc * xq.x, sc * xp.y + cc * xq.y);
        }
#pragma unroll
        for (int y = 0; y < 2; ++y) {          // rows:  y_p' = c y_p - s e^{+i phi} y_q ; y_q' = s y_p + c e^{+i phi} y_q
          const double2 yp = e[0][y], yq = cmul(pha, e[1][y]);
          e[0][y] = make_double2(ca * yp.x - sa * yq.x, ca * yp.y - sa * yq.y);
          e[1][y] = make_double2(sa * yp.x + ca * yq.x, sa * yp.y + ca * yq.y);
        }
        if (ra == cb) {                         // diagonal block: Hermitian by construction
          e[1][0] = make_double2(e[0][1].x, -e[0][1].y);
        } else {
          Sm[pb * LD + pa] = make_double2(e[0][0].x, -e[0][0].y);
          Sm[qb * LD + pa] = make_double2(e[0][1].x, -e[0][1].y);
          Sm[pb * LD + qa] = make_double2(e[1][0].x, -e[1][0].y);
          Sm[qb * LD + qa] = make_double2(e[1][1].x, -e[1][1].y);
        }
        Sm[pa * LD + pb] = e[0][0]; Sm[pa * LD + qb] = e[0][1];
        Sm[qa * LD + pb] = e[1][0]; Sm[qa * LD + qb] = e[1][1];
      }
      __syncthreads();
    }
    // the last step's rotations on U
    jacobi_u_update(Um, rcb[(S - 2) & 1], rsb[(S - 2) & 1], rphb[(S - 2) & 1], rpb[(S - 2) & 1], rqb[(S - 2) & 1],
                    t, SUB_T);
    __syncthreads();
  }
  double2* Uk = U + (int64_t)k * S * S;
  for (int idx = t; idx < S * S; idx += SUB_T) {
    const int i = idx % S, j = idx / S;
    Uk[idx] = Um[i * LD + j];          // column-major 64 x 64
  }
}

// ---- 64x64x64 complex tile products on the FP64 tensor cores (DMMA.8x8x4, complex 3M) ------
// Tiles live in shared memory in the same swizzled "[k-chunk][row][8 k]" layout the filter GEMM
// uses (16-byte complex elements, chunk index XOR row%8), so every fragment load of the 8 warps is
// bank-conflict free.  off(r, k): byte offset of element (row r, contraction index k).
__device__ __forceinline__ uint32_t toff(int r, int k) {
  return (uint32_t)((((k >> 3) * S + r) << 7) + ((((k & 7) ^ (r & 7))) << 4));
}
__device__ __forceinline__ void tst(unsigned char* base, int r, int k, double2 v) {
  *reinterpret_cast<double2*>(base + toff(r, k)) = v;
}

__device__ __forceinline__ void dmma_j(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 lds_j(uint32_t addr) {
  double2 v;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}

// acc = op(X) * Y with X (rows x k) and Y (k x cols) tiles; warp w owns rows 32*(w/4) + [0,32),
// cols 16*(w%4) + [0,16): acc[mt][nt][{re,im}][j] = C[32 wm + 8 mt + g][16 wn + 8 nt + 2 t + j].
// 3M complex product (3 real DMMAs per complex multiply-add, as the filter's zgemm3m):
// T1 = Xr Yr, T2 = Xi Yi, T3 = (Xr + Xi)(Yr + Yi); Re = T1 - T2, Im = T3 - T1 - T2.
template <bool CONJX>
__device__ __forceinline__ void tile_dmma(uint32_t xs, uint32_t ys, double (&acc)[4][2][2][2]) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = w >> 2, wn = w & 3, g = lane >> 2, t = lane & 3;
  double t3[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      acc[i][j][0][0] = acc[i][j][0][1] = acc[i][j][1][0] = acc[i][j][1][1] = 0.0;
      t3[i][j][0] = t3[i][j][1] = 0.0;
    }
#pragma unroll 4
  for (int ks = 0; ks < S / 4; ++ks) {
    const int k = (ks >> 1) * 8 + 2 * t + (ks & 1);
    double2 a[4], b[2];
    double as[4], bs[2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      a[mt] = lds_j(xs + toff(wm * 32 + mt * 8 + g, k));
      if (CONJX) a[mt].y = -a[mt].y;
      as[mt] = a[mt].x + a[mt].y;
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      b[nt] = lds_j(ys + toff(wn * 16 + nt * 8 + g, k));
      bs[nt] = b[nt].x + b[nt].y;
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        dmma_j(acc[mt][nt][0][0], acc[mt][nt][0][1], a[mt].x, b[nt].x);      // T1
        dmma_j(acc[mt][nt][1][0], acc[mt][nt][1][1], a[mt].y, b[nt].y);      // T2
        dmma_j(t3[mt][nt][0], t3[mt][nt][1], as[mt], bs[nt]);                // T3
      }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double t1 = acc[i][j][0][e], t2 = acc[i][j][1][e];
        acc[i][j][0][e] = t1 - t2;
        acc[i][j][1][e] = t3[i][j][e] - t1 - t2;
      }
}

__device__ void apply_z_block(double2* Z, int np, const int* pairs, const double2* U, int rt, int k,
                              unsigned char* sm);

// One launch per round: blocks [0, b(b+1)/2) do A[I_l, I_k] <- U_l^H A[I_l, I_k] U_k for l <= k
// (and the mirror block for l < k); the remaining (np/64) x b blocks do Z[rows, I_k] <- Z U_k.
__global__ void __launch_bounds__(256, 1) k_apply(double2* A, double2* Z, int np, const int* pairs,
                                                  const double2* U, int b) {
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int nsym = b * (b + 1) / 2;
  if ((int)blockIdx.x >= nsym) {
    const int e = blockIdx.x - nsym;
    apply_z_block(Z, np, pairs, U, e % (np / S), e / (np / S), sm);
    return;
  }
  unsigned char* Xs = sm;                  // 64 KB: A_lk, then U_l (as U_l^H)
  unsigned char* Ys = sm + S * S * 16;     // 64 KB: U_k, then T1
  int idx = blockIdx.x, l = 0;
  while (idx >= b - l) { idx -= b - l; ++l; }
  const int k = l + idx;
  const int t = threadIdx.x;
  const double2* Uk = U + (int64_t)k * S * S;
  const double2* Ul = U + (int64_t)l * S * S;
  {
    // batched global loads (16 + 16 independent 16-byte loads in flight per thread), then stores
    double2 xa[16], ya[16];
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int e = t + 256 * it, i = e % S, j = e / S;
      xa[it] = A[gidx(pairs, l, i) + gidx(pairs, k, j) * np];
      ya[it] = Uk[i + j * S];
    }
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int e = t + 256 * it, i = e % S, j = e / S;
      tst(Xs, i, j, xa[it]);                                         // X[i][k=j]
      tst(Ys, j, i, ya[it]);                                         // Y[k=i][n=j]
    }
  }
  __syncthreads();
  double acc[4][2][2][2];
  tile_dmma<false>(smem_u32(Xs), smem_u32(Ys), acc);                 // T1 = A_lk U_k
  __syncthreads();
  const int w = t >> 5, lane = t & 31, wm = w >> 2, wn = w & 3, g = lane >> 2, tt = lane & 3;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j)   // T1[row][col] is Y'[k=row][n=col]
        tst(Ys, wn * 16 + nt * 8 + 2 * tt + j, wm * 32 + mt * 8 + g,
            make_double2(acc[mt][nt][0][j], acc[mt][nt][1][j]));
  {
    double2 ua[16];
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int e = t + 256 * it;
      ua[it] = Ul[e];
    }
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int e = t + 256 * it, kk = e % S, i = e / S;
      tst(Xs, i, kk, ua[it]);                                        // X'[i][k] = conj(U_l[k][i])
    }
  }
  __syncthreads();
  tile_dmma<true>(smem_u32(Xs), smem_u32(Ys), acc);                  // T = U_l^H T1
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int i = wm * 32 + mt * 8 + g, jj = wn * 16 + nt * 8 + 2 * tt + j;
        const int64_t gi = gidx(pairs, l, i), gj = gidx(pairs, k, jj);
        const double2 v = make_double2(acc[mt][nt][0][j], acc[mt][nt][1][j]);
        A[gi + gj * np] = v;
        if (l != k) A[gj + gi * np] = make_double2(v.x, -v.y);
      }
}

// Z[rows rt*64 .. +64, I_k] <- Z[rows, I_k] U_k
__device__ void apply_z_block(double2* Z, int np, const int* pairs, const double2* U, int rt, int k,
                              unsigned char* sm) {
  unsigned char* Xs = sm;
  unsigned char* Ys = sm + S * S * 16;
  const int t = threadIdx.x;
  const double2* Uk = U + (int64_t)k * S * S;
  {
    double2 xa[16], ya[16];
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int e = t + 256 * it, i = e % S, j = e / S;
      xa[it] = Z[(int64_t)(rt * S + i) + gidx(pairs, k, j) * np];
      ya[it] = Uk[i + j * S];
    }
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int e = t + 256 * it, i = e % S, j = e / S;
      tst(Xs, i, j, xa[it]);
      tst(Ys, j, i, ya[it]);
    }
  }
  __syncthreads();
  double acc[4][2][2][2];
  tile_dmma<false>(smem_u32(Xs), smem_u32(Ys), acc);
  const int w = t >> 5, lane = t & 31, wm = w >> 2, wn = w & 3, g = lane >> 2, tt = lane & 3;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        Z[(int64_t)(rt * S + wm * 32 + mt * 8 + g) + gidx(pairs, k, wn * 16 + nt * 8 + 2 * tt + j) * np] =
            make_double2(acc[mt][nt][0][j], acc[mt][nt][1][j]);
}

// partial sums of |A_ij|^2: off-diagonal and total, per block of rows (fixed order)
__global__ void k_offnorm(const double2* A, int np, double* part) {
  __shared__ double s_off[256], s_tot[256];
  const int col = blockIdx.x;
  double off = 0.0, tot = 0.0;
  for (int i = threadIdx.x; i < np; i += 256) {
    const double2 v = A[i + (int64_t)col * np];
    const double m2 = v.x * v.x + v.y * v.y;
    tot += m2;
    if (i != col) off += m2;
  }
  s_off[threadIdx.x] = off;
  s_tot[threadIdx.x] = tot;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) { s_off[threadIdx.x] += s_off[threadIdx.x + s]; s_tot[threadIdx.x] += s_tot[threadIdx.x + s]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { part[2 * col] = s_off[0]; part[2 * col + 1] = s_tot[0]; }
}

__global__ void k_extract(const double2* A, const double2* Zp, int np, int n, const int* order, double* theta,
                          double2* Z, int64_t ldz) {
  const int64_t total = (int64_t)n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    const int src = order[j];
    Z[i + (int64_t)j * ldz] = Zp[i + (int64_t)src * np];
    if (i == 0) theta[j] = A[src + (int64_t)src * np].x;
  }
}

}  // namespace

struct JacobiWork {
  void* A = nullptr; void* Zp = nullptr; void* U = nullptr; int* pairs = nullptr; int* order = nullptr;
  double* part = nullptr;
  size_t np = 0, b = 0;
  void ensure(int np_, cudaStream_t) {
    if ((size_t)np_ <= np) return;
    release();
    np = np_;
    b = np / S;
    CHASE_CUDA(cudaMalloc(&A, 16 * np * np));
    CHASE_CUDA(cudaMalloc(&Zp, 16 * np * np));
    CHASE_CUDA(cudaMalloc(&U, 16 * (size_t)S * S * b));
    CHASE_CUDA(cudaMalloc(&pairs, sizeof(int) * 2 * b * (2 * b)));
    CHASE_CUDA(cudaMalloc(&order, sizeof(int) * np));
    CHASE_CUDA(cudaMalloc(&part, sizeof(double) * 2 * np));
  }
  void release() {
    for (void* p : {A, Zp, U, (void*)pairs, (void*)order, (void*)part}) if (p) cudaFree(p);
    A = Zp = U = nullptr; pairs = order = nullptr; part = nullptr; np = b = 0;
  }
};

void heev_work_release(JacobiWork* w) {
  if (!w) return;
  w->release();
  delete w;
}

int heev_jacobi(void* G, int64_t ld, int n, double* theta, void* Z, int64_t ldz, cudaStream_t st, JacobiWork** work) {
  if (n <= 0) return 0;
  const int np = ceil_div(n, S) * S;
  const int b = np / S;           // pairs per round; 2b blocks of W
  const int nblocks = 2 * b;
  if (!*work) *work = new JacobiWork();
  JacobiWork& g_work = **work;
  g_work.ensure(np, st);
  static unsigned long long attr = 0;
  const int smem = (int)(2 * sizeof(double2) * S * LD);
  const int smem_apply = 2 * S * S * 16 + 1024;
  if (first_on_device(attr)) {
    CHASE_CUDA(cudaFuncSetAttribute(k_sub_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CHASE_CUDA(cudaFuncSetAttribute(k_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_apply));
  }
  // schedule: circle method over 2b blocks, 2b-1 rounds of b pairs
  const int rounds = nblocks - 1;
  std::vector<int> sched(2 * (size_t)b * rounds);
  for (int r = 0; r < rounds; ++r) {
    for (int i = 0; i < b; ++i) {
      int p, q;
      if (i == 0) { p = r; q = nblocks - 1; }
      else { p = (r + i) % (nblocks - 1); q = (r - i + (nblocks - 1)) % (nblocks - 1); }
      sched[2 * ((size_t)r * b + i)] = std::min(p, q);
      sched[2 * ((size_t)r * b + i) + 1] = std::max(p, q);
    }
  }
  CHASE_CUDA(cudaMemcpyAsync(g_work.pairs, sched.data(), sizeof(int) * sched.size(), cudaMemcpyHostToDevice, st));
  // padding above the spectrum: diagonal entries > ||G||_F >= ||G||_2, decoupled from G
  double2* A = reinterpret_cast<double2*>(g_work.A);
  double2* Zp = reinterpret_cast<double2*>(g_work.Zp);
  k_pad_init<<<148 * 8, 256, 0, st>>>(reinterpret_cast<const double2*>(G), ld, n, A, Zp, np, 0.0);
  CHASE_CHECK_LAUNCH();
  k_offnorm<<<np, 256, 0, st>>>(A, np, g_work.part);
  CHASE_CHECK_LAUNCH();
  std::vector<double> part(2 * (size_t)np);
  CHASE_CUDA(cudaMemcpyAsync(part.data(), g_work.part, sizeof(double) * 2 * np, cudaMemcpyDeviceToHost, st));
  CHASE_CUDA(cudaStreamSynchronize(st));
  double tot = 0.0;
  for (int j = 0; j < np; ++j) tot += part[2 * j + 1];
  const double fro = std::sqrt(tot);
  if (!std::isfinite(fro)) throw NumericError("Rayleigh-Ritz matrix is not finite");
  const double padbase = (fro > 0.0 ? fro : 1.0) * 1.1;   // > ||G||_F >= ||G||_2 >= every |eigenvalue|
  k_pad_init<<<148 * 8, 256, 0, st>>>(reinterpret_cast<const double2*>(G), ld, n, A, Zp, np, padbase);
  CHASE_CHECK_LAUNCH();

  // Inner sweeps per 64x64 subproblem: exact diagonalisation is wasted effort while the outer
  // iteration is still in its linear phase; one inner sweep per visit keeps the outer sweep count
  // (12 at n = 3000, measured) while making each round ~2x cheaper (CHASE_JACOBI_INNER overrides, for experiments).
  int max_inner = 1;
  if (const char* e = std::getenv("CHASE_JACOBI_INNER")) max_inner = std::max(1, std::atoi(e));
  int sweeps = 0;
  bool converged = false;
  for (; sweeps < 40; ++sweeps) {
    k_offnorm<<<np, 256, 0, st>>>(A, np, g_work.part);
    CHASE_CHECK_LAUNCH();
    CHASE_CUDA(cudaMemcpyAsync(part.data(), g_work.part, sizeof(double) * 2 * np, cudaMemcpyDeviceToHost, st));
    CHASE_CUDA(cudaStreamSynchronize(st));
    double off = 0.0, t2 = 0.0;
    for (int j = 0; j < np; ++j) { off += part[2 * j]; t2 += part[2 * j + 1]; }
    // off(A)_F <= max(1e-14, 4 n u) ||A||_F (A = padded G, unitarily invariant): the in-place
    // tile updates re-inject O(u ||A||) rounding into every off-diagonal entry, so off_F has a
    // floor ~ n u ||A||_F; asking for less only burns sweeps.
    const double tol_rel = std::max(1e-14, 4.0 * np * 1.1102230246251565e-16);
    if (std::getenv("CHASE_DEBUG_JACOBI"))
      std::fprintf(stderr, "[jacobi] n=%d sweep=%d off/||A||_F=%.3e tol=%.3e\n", n, sweeps, std::sqrt(off / t2), tol_rel);
    if (off <= tol_rel * tol_rel * t2) { converged = true; break; }
    for (int r = 0; r < rounds; ++r) {
      const int* pr = g_work.pairs + 2 * (size_t)r * b;
      double2* U = reinterpret_cast<double2*>(g_work.U);
      k_sub_eig<<<b, SUB_T, smem, st>>>(A, np, pr, U, max_inner);
      CHASE_CHECK_LAUNCH();
      k_apply<<<b * (b + 1) / 2 + (np / S) * b, 256, smem_apply, st>>>(A, Zp, np, pr, U, b);
      CHASE_CHECK_LAUNCH();
    }
  }
  if (!converged) throw NumericError("block Jacobi did not converge in 40 sweeps");
  // eigenvalues: diag(A); sort ascending, drop the padding (largest)
  std::vector<double2> diag(np);
  CHASE_CUDA(cudaMemcpy2DAsync(diag.data(), sizeof(double2), A, sizeof(double2) * (np + 1), sizeof(double2), np,
                               cudaMemcpyDeviceToHost, st));
  CHASE_CUDA(cudaStreamSynchronize(st));
  std::vector<int> order(np);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int c) { return diag[a].x < diag[c].x; });
  CHASE_CUDA(cudaMemcpyAsync(g_work.order, order.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
  k_extract<<<148 * 8, 256, 0, st>>>(A, Zp, np, n, g_work.order, theta, reinterpret_cast<double2*>(Z), ldz);
  CHASE_CHECK_LAUNCH();
  CHASE_CUDA(cudaStreamSynchronize(st));   // `order` / `diag` host buffers go out of scope
  return sweeps;
}

}  // namespace chase
