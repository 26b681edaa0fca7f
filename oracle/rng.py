"""Counter-based random block for ChASE's start vectors -- ORACLE SIDE implementation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The CUDA library implements the same
counter-based generator independently (paper_2205_02491_b200/csrc/rng.cuh); the two share no
code, only the definition below, and a GPU test checks they agree bit for bit.

Definition: Philox4x32-10 (Salmon et al., SC'11) with
  key     = (seed & 0xffffffff, seed >> 32)
  counter = (row & 0xffffffff, row >> 32, column, stream)
Entry (row, column) of the block is re + i*im with
  re = ((u0 << 21) | (u1 >> 11)) * 2^-52 - 1,   im = ((u2 << 21) | (u3 >> 11)) * 2^-52 - 1
(53-bit uniform in [-1, 1); the conversion is exact, so both sides agree bitwise).  Keying by
the GLOBAL row makes the block identical for every process-grid shape.
Alg. 1 "Require: ... vector V-hat" leaves V-hat to the caller; ChASE draws it at random.
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint32(0x9E3779B9)
_W1 = np.uint32(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)

STREAM_START_V = 0      # initial V-hat of the subspace iteration
STREAM_LANCZOS = 1      # Lanczos start vectors


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint32 arrays; returns four uint32 arrays."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3))
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    with np.errstate(over="ignore"):
        for r in range(10):
            if r > 0:
                k0 = np.uint32((int(k0) + int(_W0)) & 0xFFFFFFFF)
                k1 = np.uint32((int(k1) + int(_W1)) & 0xFFFFFFFF)
            p0 = _M0 * c0.astype(np.uint64)
            p1 = _M1 * c2.astype(np.uint64)
            hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
            lo0 = (p0 & _MASK).astype(np.uint32)
            hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
            lo1 = (p1 & _MASK).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def _to_unit(a, b):
    x = (a.astype(np.uint64) << np.uint64(21)) | (b.astype(np.uint64) >> np.uint64(11))
    return x.astype(np.float64) * 2.0 ** -52 - 1.0


def random_block(seed: int, row0: int, nrows: int, col0: int, ncols: int, stream: int) -> np.ndarray:
    """Rows [row0, row0+nrows) x columns [col0, col0+ncols) of the seeded complex block."""
    rows = np.arange(row0, row0 + nrows, dtype=np.uint64)
    cols = np.arange(col0, col0 + ncols, dtype=np.uint32)
    R = np.repeat(rows[:, None], ncols, axis=1)
    C = np.repeat(cols[None, :], nrows, axis=0)
    u0, u1, u2, u3 = philox4x32_10((R & _MASK).astype(np.uint32), (R >> np.uint64(32)).astype(np.uint32),
                                   C, np.full(R.shape, stream, dtype=np.uint32),
                                   seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    return _to_unit(u0, u1) + 1j * _to_unit(u2, u3)
