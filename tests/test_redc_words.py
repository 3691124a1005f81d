"""CPU emulation of the MAC's word-level Montgomery recombination
(`redc_words` in csrc/he_kernels.cu, DESIGN.md §6 "MAC on tensor cores"):
the PTX sequence is replayed with 32-bit registers and an explicit carry
flag, and its result is checked against the definition V 2^-64 mod q and the
bound t < 2q, on adversarial and random diagonal sums S_d (byte-plane
products of K terms, S_d <= 7 K 255^2) with the largest 50-bit primes."""
import random

import pytest

M32 = (1 << 32) - 1


def _redc_words_emul(P0, P1, P2, P3, q):
    """The 20-instruction PTX block, one line per instruction."""
    qlo, qhi = q & M32, q >> 32
    qp = (-pow(q, -1, 1 << 64)) & M32            # low word of -q^-1 mod 2^64
    p0l, p0h = P0 & M32, P0 >> 32
    p1l, p1h = P1 & M32, P1 >> 32
    p2l, p2h = P2 & M32, P2 >> 32
    assert max(p0h, p1h, p2h, P3) <= M32
    m = (p0l * qp) & M32                          # mul.lo
    s = p1l + p0h; x0, c = s & M32, s >> 32       # add.cc
    x1 = (p1h + c) & M32                          # addc
    s = ((m * qhi) & M32) + x0; x0, c = s & M32, s >> 32     # mad.lo.cc
    x1 = (((m * qhi) >> 32) + x1 + c) & M32       # madc.hi
    s = ((m * qlo) & M32) + p0l; d, c = s & M32, s >> 32     # mad.lo.cc (d = 0)
    assert d == 0
    s = ((m * qlo) >> 32) + x0 + c; x0, c = s & M32, s >> 32  # madc.hi.cc
    x1 = (x1 + c) & M32                           # addc
    m = (x0 * qp) & M32                           # mul.lo
    s = p2l + x1; lo, c = s & M32, s >> 32        # add.cc
    hi = (p2h + P3 + c) & M32                     # addc
    s = ((m * qhi) & M32) + lo; lo, c = s & M32, s >> 32     # mad.lo.cc
    hi = (((m * qhi) >> 32) + hi + c) & M32       # madc.hi
    s = ((m * qlo) & M32) + x0; d, c = s & M32, s >> 32      # mad.lo.cc (d = 0)
    assert d == 0
    s = ((m * qlo) >> 32) + lo + c; lo, c = s & M32, s >> 32  # madc.hi.cc
    hi = (hi + c) & M32                           # addc
    return (hi << 32) | lo


def _partials(S, k16):
    """P_k as reduce13_mont forms them from the 13 diagonal sums."""
    P = []
    for k in range(3):
        if k16:
            a = (S[4 * k] + (S[4 * k + 1] << 8)) & M32
            b = (S[4 * k + 2] + (S[4 * k + 3] << 8)) & M32
            P.append(a + (b << 16))
        else:
            P.append(S[4 * k] + (S[4 * k + 1] << 8) + (S[4 * k + 2] << 16) + (S[4 * k + 3] << 24))
    return P[0], P[1], P[2], S[12]


def _diagonals(C, F):
    """S_d = sum_k sum_{i+j=d} byte_i(C_k) byte_j(F_k): the exact int8 MMA sums."""
    S = [0] * 13
    for c, f in zip(C, F):
        for i in range(7):
            for j in range(7):
                S[i + j] += ((c >> (8 * i)) & 255) * ((f >> (8 * j)) & 255)
    return S


QS = [(1 << 50) - 27 * (1 << 15) + 1,   # a 50-bit NTT-friendly shape (value only needs to be odd)
      1125899904679937, 1125899906826241, (1 << 29) + 11]


@pytest.mark.parametrize("K", [4, 16, 32, 64, 4096])
def test_redc_words_matches_definition(K):
    rng = random.Random(K)
    for q in QS:
        q |= 1
        R = 1 << 64
        for trial in range(40 if K < 4096 else 4):
            # lazy forward-NTT residues up to 3q/2 + 1, Montgomery filter planes < q
            if trial == 0:
                C = [3 * q // 2 + 1] * K
                F = [q - 1] * K
            elif trial == 1:
                C = [(1 << 56) - 1 if (3 * q // 2 + 1) >= (1 << 56) else 3 * q // 2 + 1] * K
                F = [q - 1] * K
            else:
                C = [rng.randrange(3 * q // 2 + 2) for _ in range(K)]
                F = [rng.randrange(q) for _ in range(K)]
            S = _diagonals(C, F)
            V = sum(s << (8 * d) for d, s in enumerate(S))
            assert V == sum(c * f for c, f in zip(C, F))
            t = _redc_words_emul(*_partials(S, K <= 16), q)
            assert t % q == V * pow(R, -1, q) % q
            assert t < 2 * q
