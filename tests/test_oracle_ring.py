"""Pins for the oracle's ring arithmetic (not gpu).

Each test checks oracle/ against something other than itself: a brute-force
definition, a closed form, or an independent second path.
"""
import json
import os

import numpy as np
import pytest

import synth
from oracle import ref as R

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "spec_examples.json")))


def test_primes_match_r8_rule_and_tables():
    # R8: largest primes < 2^bits, q = 1 mod 2N; synth tables must agree.
    for c, cfg in synth.CONFIGS.items():
        bits = 30 if c == 1 else 50
        assert R.find_primes(cfg.N, bits, cfg.L) == list(cfg.primes)
        for q in cfg.primes:
            assert R.is_prime(q) and (q - 1) % (2 * cfg.N) == 0 and q < 2 ** bits


def test_is_prime_vs_trial_division():
    # independent brute force on small integers
    for n in range(2, 5000):
        bf = all(n % d for d in range(2, int(n ** 0.5) + 1))
        assert R.is_prime(n) == bf


def test_min_psi_brute_force_small():
    # R9 on small primes: brute-force the smallest x with x^N = -1
    for q, N in [(97, 8), (97, 16), (193, 32), (257, 64), (7681, 256)]:
        bf = min(x for x in range(2, q) if pow(x, N, q) == q - 1)
        assert R.min_psi(q, N) == bf


def test_psi_is_primitive_2n_root():
    for cfg in synth.CONFIGS.values():
        q = cfg.primes[0]
        psi = R.min_psi(q, cfg.N)
        assert pow(psi, cfg.N, q) == q - 1          # psi^N = -1
        assert pow(psi, 2 * cfg.N, q) == 1


def test_negacyclic_wrap_golden():
    g = GOLD["negacyclic_wrap"]
    N = g["N"]
    a = [0] * N
    b = [0] * N
    a[g["a_exp"]] = 1
    b[g["b_exp"]] = 1
    c = R.schoolbook_py(a, b, N)
    assert c[0] == g["expect_coeff0"] and all(x == 0 for x in c[1:])
    q = 97
    cc = R.negacyclic_at(np.array(a, np.uint64), np.array(b, np.uint64), q)
    assert int(cc[0]) == q - 1


def test_three_product_paths_agree():
    # schoolbook (Python ints) == C definition == sparse-direct
    rng = np.random.default_rng(1)
    for N, q in [(8, 97), (64, 7681), (256, 1073707009)]:
        a = rng.integers(0, q, N).astype(np.uint64)
        bsp = rng.integers(-8, 8, N) * (rng.random(N) < 0.2)
        ref = R.schoolbook_py(a, bsp, N, q)
        c_def = R.negacyclic_at(a, np.mod(bsp, q).astype(np.uint64), q)
        terms = [(i, int(bsp[i])) for i in range(N) if bsp[i]]
        c_sp = R.sparse_mul(a, terms, q)
        assert [int(x) for x in c_def] == ref
        assert [int(x) for x in c_sp] == ref


def test_ntt_definition_pins():
    q, N = 7681, 256
    psi = R.min_psi(q, N)
    rng = np.random.default_rng(2)
    a = rng.integers(0, q, N).astype(np.uint64)
    A = R.ntt_def(a, q, psi)
    # C definition equals the pure-Python definition on a tiny ring
    q2, N2 = 97, 16
    psi2 = R.min_psi(q2, N2)
    a2 = rng.integers(0, q2, N2)
    assert [int(x) for x in R.ntt_def(a2.astype(np.uint64), q2, psi2)] == \
        R.ntt_def_py(a2, q2, psi2)
    # INTT(NTT(a)) = a
    assert np.array_equal(R.intt_def(A, q, psi), a)
    # NTT(delta_0) = all ones
    d = np.zeros(N, np.uint64)
    d[0] = 1
    assert np.all(R.ntt_def(d, q, psi) == 1)
    # convolution theorem: pointwise product == schoolbook negacyclic product
    b = rng.integers(0, q, N).astype(np.uint64)
    B = R.ntt_def(b, q, psi)
    P = (A.astype(object) * B.astype(object)) % q
    assert [int(x) for x in R.intt_def(P.astype(np.uint64), q, psi)] == \
        R.schoolbook_py(a, b, N, q)


def test_encode_matches_bigint_definition():
    cfg = synth.CONFIGS[2]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    m = np.array([0, 1, 2, 255, 32768, 32769, 65535, 65536, 12345],
                 dtype=np.uint32)
    assert np.array_equal(R.encode(m, ring), R.encode_bigint(m, ring))
    ring1 = R.Ring(1024, synth.CONFIGS[1].primes, 65537)
    m1 = np.arange(0, 65537, 97, dtype=np.uint32)
    assert np.array_equal(R.encode(m1, ring1), R.encode_bigint(m1, ring1))


def test_encode_centred_remainder_identity():
    """The identity the K4 writer's FP64 mask encoding relies on (DESIGN.md
    §6, K4): Q m = t round(Q m / t) + c with c the centred remainder of r_t m
    mod t, and Q = 0 mod q_j, so enc_j(m) = -c t^{-1} mod q_j.  Checked
    against the literal R2 definition (big integers) for several t."""
    for c_idx, t in ((4, 65537), (1, 65537), (2, 257), (3, 3), (4, (1 << 20) - 3)):
        cfg = synth.CONFIGS[c_idx]
        ring = R.Ring(cfg.N, cfg.primes, t)
        rng = np.random.default_rng(t)
        m = np.unique(np.concatenate([[0, 1, t // 2, t // 2 + 1, t - 1],
                                      rng.integers(0, t, 200)])).astype(np.uint32)
        want = R.encode_bigint(m, ring)
        r_t = ring.Q % t
        for i, mv in enumerate(m):
            rem = (r_t * int(mv)) % t
            cen = rem - t if 2 * rem > t else rem
            assert abs(cen) <= t // 2
            for j, q in enumerate(ring.primes):
                assert (-cen * pow(t, -1, q)) % q == int(want[j, i])


def test_encode_decodes_exactly():
    # round(t * enc(m) / Q) = m: the encoding error is at most 1/2 (R2)
    for c in (1, 2, 4):
        cfg = synth.CONFIGS[c]
        ring = R.Ring(cfg.N, cfg.primes, cfg.t)
        m = np.array([0, 1, 7, 32768, 65536], dtype=np.uint32)
        enc = R.encode(m, ring)
        dec = R.crt_decode([enc[j] for j in range(ring.L)], ring)
        assert dec == [int(x) for x in m]


def test_splitmix64_phi1_stream():
    # SplitMix64 reference output for state 0 (Vigna's splitmix64.c): the
    # first value is 0xe220a8397b1dcdaf; the vectorised stream must match the
    # Python-int definition element by element.
    assert R.splitmix64_py(0, 0) == 0xE220A8397B1DCDAF
    for seed in (0, 1, 2 ** 63 + 12345, 2 ** 64 - 1):
        v = R.phi1_stream(seed, 257, 65537)
        assert [int(x) for x in v] == [R.splitmix64_py(seed, i) % 65537
                                       for i in range(257)]
        assert v.max() < 65537


def test_incomplete_ntt_definition_pins():
    # s = 1 is the full NTT in bit-reversed order; s = N is a mod (X^N + 1)
    # = a; and the fold identity of DESIGN.md §4: coefficient 0 of
    # c f mod (X^s - zeta_g), summed back through an (N/s)-point inverse
    # transform, gives the coefficients s j of the negacyclic product
    rng = np.random.default_rng(11)
    q, N = 7681, 64
    psi = R.min_psi(q, N)
    a = rng.integers(0, q, N).astype(np.uint64)
    full = R.ntt_def(a, q, psi)
    brv = [int(format(p, "06b")[::-1], 2) for p in range(N)]
    assert np.array_equal(R.incomplete_ntt_def(a, q, psi, 1), full[brv])
    assert np.array_equal(R.incomplete_ntt_def(a, q, psi, N), a)
    f = rng.integers(0, q, N).astype(np.uint64)
    prod = R.schoolbook_py(a, f, N, q)
    for s in (2, 4, 8):
        A = R.incomplete_ntt_def(a, q, psi, s)
        Fv = R.incomplete_ntt_def(f, q, psi, s)
        M = N // s
        T = M.bit_length() - 1
        for g in range(M):
            b = int(format(g, f"0{T}b")[::-1], 2)
            zeta = pow(psi, s * (2 * b + 1), q)
            c0 = (int(A[g * s]) * int(Fv[g * s]) + zeta * sum(
                int(A[g * s + u]) * int(Fv[g * s + s - u]) for u in range(1, s))) % q
            # = R_0(zeta) with R_0(Y) = sum_j prod[s j] Y^j
            assert c0 == sum(prod[s * j] * pow(zeta, j, q) for j in range(M)) % q
