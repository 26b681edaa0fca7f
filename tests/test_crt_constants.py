"""CPU pins of the Ozaki scheme II constants in csrc/ozaki.cu: the moduli must be
pairwise coprime (the Chinese remainder theorem needs it), their product M must exceed twice the
largest |A'B'| the kernel can produce (|A'|, |B'| < 2^52, K <= 131071: A'B' must sit in the
balanced range (-M/2, M/2) to be rebuilt exactly), the balanced residues must fit int8 with the
int32 sums exact, and the Garner / Horner reconstruction written the way the kernel does it must
return A'B' exactly -- checked here in Python integers on random and extreme cases."""
import math
import os
import random
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _moduli():
    src = open(os.path.join(ROOT, "paper_2205_02491_b200", "csrc", "ozaki.cu")).read()
    m = re.search(r"constexpr int m\[NMOD\] = \{([^}]*)\}", src)
    nmod = int(re.search(r"constexpr int NMOD = (\d+);", src).group(1))
    mods = [int(x) for x in m.group(1).split(",")]
    assert len(mods) == nmod
    bits = int(re.search(r"constexpr int CRT_BITS = (\d+);", src).group(1))
    return mods, bits


def _balanced(r, m):
    hi = 127 if m == 256 else (m - 1) // 2
    r %= m
    return r - m if r > hi else r


def _garner(res, mods):
    """The kernel's reconstruction: digits v_j = (c_j - sum_{i<j} v_i P_i) P_j^-1 mod m_j, balanced,
    then Horner x = v_15; x = x m_j + v_j."""
    v = []
    for j, mj in enumerate(mods):
        P = 1
        R = 0
        for i in range(j):
            R += v[i] * (P % mj)
            P *= mods[i]
        t = (res[j] - R) % mj
        t = (t * pow(P % mj, -1, mj)) % mj
        v.append(_balanced(t, mj))
    x = v[-1]
    for j in range(len(mods) - 2, -1, -1):
        x = x * mods[j] + v[j]
    return x


def test_moduli_pairwise_coprime_and_range():
    mods, bits = _moduli()
    assert all(2 <= m <= 256 for m in mods)
    for i in range(len(mods)):
        for j in range(i + 1, len(mods)):
            assert math.gcd(mods[i], mods[j]) == 1, (mods[i], mods[j])
    M = math.prod(mods)
    kmax = 131071
    assert 2 * kmax * (2 ** bits) ** 2 < M            # |A'B'| < K 2^(2 bits) < M / 2
    assert 128 * 128 * kmax <= 2 ** 31 - 1             # balanced residues |r| <= 128: exact int32 sums
    assert 128 * 128 * (kmax + 1) > 2 ** 31 - 1        # ... and 131071 is the largest such K


def test_garner_reconstruction_is_exact():
    mods, bits = _moduli()
    rnd = random.Random(7)
    lim = 2 ** bits
    for trial in range(300):
        K = rnd.choice([1, 5, 300, 131071])
        if trial < 4:                                  # extremes: every term at its largest magnitude
            x = (lim - 1) * (lim - 1) * K * (1 if trial % 2 else -1)
        else:
            x = sum(rnd.randrange(-lim + 1, lim) * rnd.randrange(-lim + 1, lim) for _ in range(min(K, 8)))
        # what the GEMM drain stores: the int32 product mod m (here: of the exact integer)
        res = [x % m for m in mods]
        assert _garner(res, mods) == x
    assert _garner([0] * len(mods), mods) == 0
    assert _garner([(-1) % m for m in mods], mods) == -1
