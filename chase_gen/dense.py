"""Dense complex-Hermitian test matrices with an exactly known spectrum (§4.1).

SEEDED INPUT GENERATION ONLY -- no ChASE arithmetic lives here.  Both the CPU oracle tests and
the CUDA path consume these matrices; the device twin (`chase_gen/csrc/gen.cu`) evaluates the
very same entry formula on the GPU for the large benchmark shapes.

Two constructions:

G1 (paper's method, complexified per ledger #11): H = Q diag(lambda) Q^H with Q the
   Q factor of a Householder QR of a complex Gaussian n x n matrix (phases of R's diagonal
   absorbed, i.e. Haar-distributed Q).  O(n^3); used for n <= 4096.

G2 (any n): H = Phi P C P^H Phi^H, where
   * C = F diag(lambda_pi) F^H is circulant, F_{jk} = w^{jk}/sqrt(n), w = exp(2 pi i/n), and
     lambda_pi a seeded permutation of the spectrum, so C_{jl} = c_{(j-l) mod n} with
     c = ifft(lambda_pi);
   * P = H_1 ... H_k, H_t = I - 2 y_t y_t^H (unit complex Gaussian y_t), k = 4;
   * Phi = diag(exp(i theta_j)) with seeded random phases.
   Each reflector adds a rank-2 Hermitian term (M -> M + y w^H + w y^H, w = -2My + 2(y^H M y)y),
   so  H_{jl} = phi_j conj(phi_l) c_{(j-l) mod n} + sum_t U_{jt} conj(V_{lt})  with U, V of
   width 2k (phases folded in).  The spectrum is exact to FFT rounding and the eigenvector of
   lambda_pi[k] is Phi P f_k, computable in O(n k) -- an exact eigenvector pin at every n.
   Entries are evaluated with separate real multiplies/adds in a fixed order (no FMA), so the
   host and device evaluations are bitwise identical.
"""
from __future__ import annotations

import numpy as np

from .spectra import spectrum as _spectrum


class G2Matrix:
    """Description of a G2 matrix: O(n k) numbers from which any entry / block is evaluated."""

    def __init__(self, lam: np.ndarray, seed: int = 1, n_reflectors: int = 4):
        lam = np.asarray(lam, dtype=np.float64)
        n = lam.shape[0]
        self.n = n
        self.lam = np.sort(lam)
        rng = np.random.default_rng(seed)
        self.perm = rng.permutation(n)                 # lambda_pi[k] = lam[perm[k]]
        lam_p = self.lam[self.perm]
        self.lam_p = lam_p
        self.circ = np.fft.ifft(lam_p)                  # c_d, d = 0..n-1
        theta = rng.uniform(0.0, 2.0 * np.pi, size=n)
        self.phi = np.exp(1j * theta)
        ys = []
        for _ in range(n_reflectors):
            y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
            ys.append(y / np.linalg.norm(y))
        self.ys = ys
        U = np.zeros((n, 0), dtype=np.complex128)
        V = np.zeros((n, 0), dtype=np.complex128)
        # P C P^H = H_1 (H_2 ( ... H_k C H_k ... ) H_2) H_1  -> apply H_k first.
        for y in reversed(ys):
            z = np.fft.ifft(lam_p * np.fft.fft(y)) + U @ (V.conj().T @ y)   # z = M y
            s = np.vdot(y, z).real
            w = -2.0 * z + 2.0 * s * y
            U = np.concatenate([U, y[:, None], w[:, None]], axis=1)
            V = np.concatenate([V, w[:, None], y[:, None]], axis=1)
        self.U = self.phi[:, None] * U                  # Phi U
        self.V = self.phi[:, None] * V                  # Phi V
        self.rank = U.shape[1]

    # ---- entries -------------------------------------------------------------------------
    def block(self, r0: int, nr: int, c0: int, nc: int) -> np.ndarray:
        """H[r0:r0+nr, c0:c0+nc] as a complex128 array (evaluated like the device twin)."""
        rows = np.arange(r0, r0 + nr)
        cols = np.arange(c0, c0 + nc)
        d = (rows[:, None] - cols[None, :]) % self.n
        cr, ci = self.circ.real[d], self.circ.imag[d]
        pr_r, pr_i = self.phi.real[rows][:, None], self.phi.imag[rows][:, None]
        pc_r, pc_i = self.phi.real[cols][None, :], -self.phi.imag[cols][None, :]   # conj(phi_l)
        # s = phi_j * conj(phi_l)
        sr = pr_r * pc_r - pr_i * pc_i
        si = pr_r * pc_i + pr_i * pc_r
        # h = s * c_d
        hr = sr * cr - si * ci
        hi = sr * ci + si * cr
        Ur, Ui = self.U.real[rows], self.U.imag[rows]
        Vr, Vi = self.V.real[cols], -self.V.imag[cols]                               # conj(V)
        for t in range(self.rank):
            ar, ai = Ur[:, t][:, None], Ui[:, t][:, None]
            br, bi = Vr[:, t][None, :], Vi[:, t][None, :]
            hr = hr + (ar * br - ai * bi)
            hi = hi + (ar * bi + ai * br)
        return hr + 1j * hi

    def dense(self) -> np.ndarray:
        return self.block(0, self.n, 0, self.n)

    def params_for_device(self):
        """Flat float64 arrays the device twin consumes (see chase_gen/csrc/gen.cu)."""
        return dict(
            n=self.n, rank=self.rank,
            circ=np.ascontiguousarray(np.stack([self.circ.real, self.circ.imag], -1).ravel()),
            phi=np.ascontiguousarray(np.stack([self.phi.real, self.phi.imag], -1).ravel()),
            # row-major (n, rank) interleaved complex
            U=np.ascontiguousarray(np.stack([self.U.real, self.U.imag], -1).ravel()),
            V=np.ascontiguousarray(np.stack([self.V.real, self.V.imag], -1).ravel()),
        )

    # ---- exact eigenpairs ------------------------------------------------------------------
    def eigvecs(self, idx) -> np.ndarray:
        """Exact eigenvectors (columns) of H for eigenvalues self.lam[idx] (ascending order)."""
        idx = np.atleast_1d(np.asarray(idx))
        inv = np.empty(self.n, dtype=np.int64)
        inv[self.perm] = np.arange(self.n)
        ks = inv[idx]                                   # Fourier index of each eigenvalue
        j = np.arange(self.n)
        X = np.exp(2j * np.pi * np.outer(j, ks) / self.n) / np.sqrt(self.n)   # f_k
        for y in reversed(self.ys):                      # P f = H_1(...(H_k f))
            X = X - 2.0 * np.outer(y, y.conj() @ X)
        return self.phi[:, None] * X


class R2Matrix:
    """Real-symmetric analogue of G2 for the real variant (the paper's matrices are real,
    P:134):  H = S P C P^T S with C = Hc diag(lambda_pi) Hc, Hc the orthogonal, symmetric
    discrete Hartley matrix Hc_{jk} = cas(2 pi j k / n)/sqrt(n) (cas = cos + sin).  Since
    cas(a) cas(b) = cos(a - b) + sin(a + b),
        C_{jl} = u[(j - l) mod n] + w[(j + l) mod n],   u + i w = ifft(lambda_pi),
    P = four real Householder reflectors (rank-2 updates as in G2), S = diag(+-1) random signs.
    Exact spectrum; eigenvector of lambda_pi[k] = S P h_k (h_k = column k of Hc)."""

    def __init__(self, lam: np.ndarray, seed: int = 1, n_reflectors: int = 4):
        lam = np.asarray(lam, dtype=np.float64)
        n = lam.shape[0]
        self.n = n
        self.lam = np.sort(lam)
        rng = np.random.default_rng(seed)
        self.perm = rng.permutation(n)
        lam_p = self.lam[self.perm]
        self.lam_p = lam_p
        c = np.fft.ifft(lam_p)
        self.u, self.w = np.ascontiguousarray(c.real), np.ascontiguousarray(c.imag)
        self.sgn = np.where(rng.uniform(size=n) < 0.5, -1.0, 1.0)
        ys = []
        for _ in range(n_reflectors):
            y = rng.standard_normal(n)
            ys.append(y / np.linalg.norm(y))
        self.ys = ys
        U = np.zeros((n, 0))
        V = np.zeros((n, 0))

        def dht(x):                     # Hc x
            f = np.fft.fft(x)
            return (f.real - f.imag) / np.sqrt(n)

        for y in reversed(ys):
            z = dht(lam_p * dht(y)) + U @ (V.T @ y)                 # z = M y
            s = float(y @ z)
            w = -2.0 * z + 2.0 * s * y
            U = np.concatenate([U, y[:, None], w[:, None]], axis=1)
            V = np.concatenate([V, w[:, None], y[:, None]], axis=1)
        self.U = self.sgn[:, None] * U
        self.V = self.sgn[:, None] * V
        self.rank = U.shape[1]

    def block(self, r0, nr, c0, nc):
        rows = np.arange(r0, r0 + nr)
        cols = np.arange(c0, c0 + nc)
        dm = (rows[:, None] - cols[None, :]) % self.n
        dp = (rows[:, None] + cols[None, :]) % self.n
        h = self.sgn[rows][:, None] * self.sgn[cols][None, :]
        h = h * (self.u[dm] + self.w[dp])
        for t in range(self.rank):
            h = h + self.U[rows, t][:, None] * self.V[cols, t][None, :]
        return h

    def dense(self):
        return self.block(0, self.n, 0, self.n)

    def params_for_device(self):
        return dict(n=self.n, rank=self.rank, u=self.u.copy(), w=self.w.copy(), sgn=self.sgn.copy(),
                    U=np.ascontiguousarray(self.U.ravel()), V=np.ascontiguousarray(self.V.ravel()))

    def eigvecs(self, idx):
        idx = np.atleast_1d(np.asarray(idx))
        inv = np.empty(self.n, dtype=np.int64)
        inv[self.perm] = np.arange(self.n)
        ks = inv[idx]
        j = np.arange(self.n)
        ang = 2 * np.pi * np.outer(j, ks) / self.n
        X = (np.cos(ang) + np.sin(ang)) / np.sqrt(self.n)
        for y in reversed(self.ys):
            X = X - 2.0 * np.outer(y, y @ X)
        return self.sgn[:, None] * X


class G1Matrix:
    """Paper's construction A = Q^T D Q: Haar Q (complex by default -- ledger #11 --
    real orthogonal with real=True, the paper's own setting), n <= 4096."""

    def __init__(self, lam: np.ndarray, seed: int = 1, real: bool = False):
        lam = np.sort(np.asarray(lam, dtype=np.float64))
        n = lam.shape[0]
        if n > 4096:
            raise ValueError("G1 is O(n^3); use G2 for n > 4096")
        self.n = n
        self.lam = lam
        rng = np.random.default_rng(seed)
        if real:
            Z = rng.standard_normal((n, n))
        else:
            Z = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2.0)
        Q, R = np.linalg.qr(Z)
        dr = np.diag(R)
        Q = Q * (dr / np.abs(dr))[None, :]
        self.Q = Q
        H = (Q * lam[None, :]) @ Q.conj().T
        self._H = 0.5 * (H + H.conj().T)

    def dense(self) -> np.ndarray:
        return self._H.copy()

    def block(self, r0, nr, c0, nc):
        return self._H[r0:r0 + nr, c0:c0 + nc].copy()

    def eigvecs(self, idx):
        return self.Q[:, np.atleast_1d(idx)]


def make_matrix(family: str, n: int, kind: str = "g2", seed: int = 1,
                d_max: float = 1.0, eps: float = 1e-4):
    """Seeded test matrix of Table 1 `family` with exact spectrum `.lam`.
    kind: g1 / g2 (complex Hermitian), r1 / r2 (real symmetric: real Haar Q / Hartley-based)."""
    lam = _spectrum(family, n, d_max, eps)
    if kind == "g1":
        return G1Matrix(lam, seed)
    if kind == "g2":
        return G2Matrix(lam, seed)
    if kind == "r1":
        return G1Matrix(lam, seed, real=True)
    if kind == "r2":
        return R2Matrix(lam, seed)
    raise ValueError(kind)


def block_partition(n: int, parts: int):
    """Block partition of [0, n) into `parts` ranges; the first (n mod parts) get one extra
    (ledger #19).  Returns a list of (start, length)."""
    base, rem = divmod(n, parts)
    out, s = [], 0
    for i in range(parts):
        ln = base + (1 if i < rem else 0)
        out.append((s, ln))
        s += ln
    return out
