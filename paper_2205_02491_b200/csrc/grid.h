// 2D block distribution of H over an r x c grid (§3.2, Eq. distribution:AV)
// and the intersection ranges I_ij where the global diagonal crosses a shard (drives the fused
// shift A - gamma I of P:398/P:439-441 and the intersection sums of RR / residuals).
#pragma once
#include <algorithm>
#include <cstdint>

namespace chase {

struct Range {
  int64_t start = 0, len = 0;
};

// Block partition of [0, n) into `parts`; the first (n mod parts) blocks get one extra element
// (ledger #19).
inline Range block_range(int64_t n, int parts, int idx) {
  const int64_t base = n / parts, rem = n % parts;
  Range r;
  r.len = base + (idx < rem ? 1 : 0);
  r.start = idx * base + std::min<int64_t>(idx, rem);
  return r;
}

struct Grid {
  int r = 1, c = 1;       // grid shape
  int rank = 0;           // rank = i + j*r (column-major)
  int i = 0, j = 0;       // my grid coordinates
  int64_t N = 0;
  Range rows, cols;       // my shard: H[rows.start : +rows.len, cols.start : +cols.len]

  void setup(int64_t n, int rr, int cc, int rk) {
    N = n; r = rr; c = cc; rank = rk;
    i = rk % r; j = rk / r;
    rows = block_range(N, r, i);
    cols = block_range(N, c, j);
  }
  // Intersection of my row range with my column range, in global indices.
  Range diag() const {
    const int64_t lo = std::max(rows.start, cols.start);
    const int64_t hi = std::min(rows.start + rows.len, cols.start + cols.len);
    Range d;
    d.start = lo;
    d.len = std::max<int64_t>(0, hi - lo);
    return d;
  }
  // Designated ranks that add the beta term before the sum (exactly one per communicator).
  bool beta_owner_fwd() const { return j == (i % c); }     // forward sums over row comm i
  bool beta_owner_bwd() const { return i == (j % r); }     // backward sums over column comm j
};

}  // namespace chase
