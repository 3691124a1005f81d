"""CPU checks of the FP64 modular-arithmetic bounds the CUDA transforms rely
on (he_internal.cuh: dp_mulmod, dp_reduce).  Not the oracle:
these emulate the kernels' exact double-precision operation sequence (an
FMA is one correctly rounded a*b + c, computed here with Fractions) on
adversarial operands and check the claimed ranges and congruences.
"""
from fractions import Fraction

import numpy as np

import synth

MAGIC = 6755399441055744.0          # 1.5 * 2^52


def fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def dp_mulmod(y, w, q, qinv):
    p = y * w
    e = fma(y, w, -p)
    k = fma(p, qinv, MAGIC) - MAGIC
    return fma(-k, q, p) + e


def dp_reduce(y, q, qinv):
    k = fma(y, qinv, MAGIC) - MAGIC
    return fma(-k, q, y)


def primes():
    return sorted(set(synth.PRIMES_N16384[:3] + synth.PRIMES_N32768[:2] +
                      synth.PRIMES_N8192[:2] + list(synth.PRIMES_CFG1)))


def test_mulmod_bound_with_centred_twiddles():
    """|y| <= 4q + 8 and |w| <= (q-1)/2 (centred tables): the product is
    exact mod q and |T| <= q."""
    rng = np.random.default_rng(5)
    for q in primes():
        qd, qinv = float(q), 1.0 / float(q)
        wmax = (q - 1) // 2
        ys = [4 * q + 8, -(4 * q + 8), 4 * q + 7, 2 * q, q - 1, 1, 0,
              3 * q + q // 2] + [int(v) for v in rng.integers(-(4 * q + 8), 4 * q + 9, 40)]
        ws = [wmax, -wmax, wmax - 1, 1, -1, 0] + \
            [int(v) for v in rng.integers(-wmax, wmax + 1, 12)]
        for y in ys:
            for w in ws:
                t = dp_mulmod(float(y), float(w), qd, qinv)
                assert t == int(t)
                assert abs(t) <= q, (q, y, w, t)
                assert (int(t) - y * w) % q == 0


def test_reduce_bound_up_to_2_53():
    """dp_reduce: |r| <= q/2 + 2 for integer-valued |y| < 2^53, so d2canon
    needs one conditional add.  (9q exceeds 2^53 for the 50-bit primes: the
    K4 writer reduces radix-16 outputs before adding the mask encoding.)"""
    rng = np.random.default_rng(6)
    for q in primes():
        qd, qinv = float(q), 1.0 / float(q)
        big = [y for y in (9 * q, 8 * q + 16, 5 * q + 8) if y < 2 ** 53]
        ys = [2 ** 53 - 1, -(2 ** 53 - 1), q // 2, q // 2 + 1, -(q // 2) - 1] + big + \
            [-y for y in big] + [int(v) for v in rng.integers(-(2 ** 53 - 1), 2 ** 53, 60)]
        for y in ys:
            r = dp_reduce(float(y), qd, qinv)
            assert r == int(r)
            assert abs(r) <= q / 2 + 2, (q, y, r)
            assert (int(r) - y) % q == 0
            canon = r + q if r < 0 else r
            assert 0 <= canon < q


def test_ct_radix16_pass_bounds():
    """A radix-16 CT pass on reduced inputs (|x| <= q/2 + 2) keeps every
    multiplicand below 4q and every output below 4.5q + 2 (worst case: all
    products at +q), within the exact range of doubles."""
    for q in primes():
        b = q / 2 + 2
        for r in range(4):
            assert b + r * q < 4 * q          # stage-r multiplicand
        assert b + 4 * q < 2 ** 53            # pass outputs exact
        # GS pass: |X - Y| <= 2^v (q + 4) at stage v; stages 0-2 multiply
        # directly (<= 4q + 16 only needs q <= 2^50 - 8: the bound used is
        # the mulmod test's 4q + 8 with the reduced start |x| <= q/2 + 2)
        assert 4 * (q + 4) <= 4 * q + 16
        assert 8 * (q / 2 + 2) < 2 ** 53      # radix-16 GS outputs exact
