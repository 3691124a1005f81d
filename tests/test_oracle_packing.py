"""Pins for the oracle's Conv/FC packing and server definition (not gpu).

Integer mode (no encryption): products of the packed polynomials, computed
by plain schoolbook, must carry the brute-force convolution Eq. (3)/(4) and
the FC output (Theorem 1) at the stated slots.
"""
import json
import os

import numpy as np
import pytest

import synth
from oracle import ref as R

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "spec_examples.json")))


def test_conv2d_ref_golden():
    g = GOLD["conv_2x2"]
    I = np.array(g["I"])[None]                        # c_i = 1
    F = np.array(g["F"])[None, None]                  # [1][1][2][1]
    Ly = synth.ConvLayer(1, 1, 2, 2, f_w=2, f_h=1, pad=0)
    plan = R.plan_conv(Ly, 16)
    assert R.conv2d_ref(I, F, plan).tolist() == [g["expect"]]


def test_single_pixel_golden():
    g = GOLD["single_pixel_input"]
    Ly = synth.ConvLayer(g["c_i"], 1, g["w_i"], g["h_i"], f_w=g["f_w"],
                         f_h=g["f_h"], pad=0)
    plan = R.plan_conv(Ly, g["N"], s_override=g["s"])
    p = R.pack_input_int(np.array([[[g["pixel"]]]]), plan)[0]
    e = g["expect"]["exponent"]
    assert p[e] == g["expect"]["coeff"] and np.count_nonzero(p) == 1


@pytest.mark.parametrize("key", ["valid_slots_2_2", "valid_slots_4_2"])
def test_valid_slot_offsets_golden(key):
    g = GOLD[key]
    Ly = synth.ConvLayer(g["c_i"], g["c_o"], 2, 2, f_w=1, f_h=1, pad=0)
    plan = R.plan_conv(Ly, 64, s_override=g["c_i"])
    assert [plan.t_n(n) for n in range(g["c_o"])] == g["expect_offsets"]


SHAPES = [
    # (layer, N, s_override)
    (synth.ConvLayer(1, 2, 4, 4), 256, 0),
    (synth.ConvLayer(3, 4, 4, 4), 256, 0),             # c_i not a power of 2
    (synth.ConvLayer(4, 4, 4, 4, stride=2), 256, 0),   # stride 2 (R12)
    (synth.ConvLayer(8, 2, 3, 3), 128, 0),             # n_ib = 2 (R13)
    (synth.ConvLayer(8, 8, 4, 4, stride=2), 256, 0),   # n_ib = n_ob = 2
    (synth.ConvLayer(4, 2, 2, 2, f_w=2, f_h=1, pad=0), 64, 4),  # paper-literal s=c_i
    (synth.ConvLayer(2, 2, 3, 3, f_w=2, f_h=2, pad=0), 64, 2),
    (synth.ConvLayer(2, 3, 5, 3, f_w=3, f_h=1), 256, 0),         # rectangular
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: str(s[0]))
def test_integer_mode_packing_equals_brute_force(shape):
    Ly, N, so = shape
    plan = R.plan_conv(Ly, N, so)
    rng = np.random.default_rng(7)
    img = rng.integers(0, 16, (Ly.c_i, Ly.w_i, Ly.h_i))
    W = rng.integers(-4, 4, (Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h))
    ref = R.conv2d_ref(img, W, plan)
    ipoly = R.pack_input_int(img, plan)
    pos = R.output_positions(plan)
    for ob in range(plan.n_ob):
        for nl in range(plan.c_ob):
            n = ob * plan.c_ob + nl
            if n >= plan.c_o:
                continue
            prod = np.zeros(N, dtype=object)
            for beta in range(plan.n_ib):
                f = R.filter_poly_int(W, plan, n, beta, shifted=True)
                prod += np.array(R.schoolbook_py(ipoly[beta], f, N), object)
            got = prod[pos[nl::plan.c_ob]].astype(np.int64)
            assert np.array_equal(got.reshape(plan.w_o, plan.h_o), ref[n])


def test_shift_consistency():
    # coefficient s*P + t_n with the shifted filter == coefficient s*P with
    # the unshifted one (Eq. (7) factored form)
    Ly = synth.ConvLayer(4, 4, 3, 3)
    plan = R.plan_conv(Ly, 256)
    rng = np.random.default_rng(3)
    img = rng.integers(0, 16, (4, 3, 3))
    W = rng.integers(-4, 4, (4, 4, 3, 3))
    ip = R.pack_input_int(img, plan)[0]
    for n in range(4):
        a = R.schoolbook_py(ip, R.filter_poly_int(W, plan, n, 0, True), 256)
        b = R.schoolbook_py(ip, R.filter_poly_int(W, plan, n, 0, False), 256)
        for P in range(256 // plan.s):
            assert a[plan.s * P + plan.t_n(n)] == b[plan.s * P]


def test_plans_of_configs():
    # SURVEY §8 plan table (R11)
    expect = {1: [(8, 1, 1, 2, 1)], 2: [(4, 3, 1, 4, 4)],
              3: [(16, 16, 2, 16, 2)], 5: [(256, 64, 1, 64, 1)]}
    for c, rows in expect.items():
        cfg = synth.CONFIGS[c]
        for Ly, row in zip(cfg.conv, rows):
            p = R.plan_conv(Ly, cfg.N)
            assert (p.s, p.c_ib, p.n_ib, p.c_ob, p.n_ob) == row
    p4 = [R.plan_conv(Ly, 16384) for Ly in synth.CONFIGS[4].conv]
    assert [(p.s, p.n_ib, p.n_ob) for p in p4[:2]] == [(8, 1, 2), (8, 2, 2)]
    assert (p4[7].s, p4[7].n_ob, p4[7].w_o) == (8, 4, 16)
    assert (p4[13].s, p4[13].n_ob, p4[13].w_o) == (32, 2, 8)
    assert (p4[18].s, p4[18].c_ob) == (128, 64)


def test_output_positions_unique_and_ordered():
    for cfg in synth.CONFIGS.values():
        for Ly in cfg.conv:
            p = R.plan_conv(Ly, cfg.N)
            pos = R.output_positions(p)
            assert len(pos) == p.n_valid == len(set(pos.tolist()))
            assert np.all(np.diff(pos) > 0) and pos[-1] < cfg.N


# ---------------------------------------------------------------- FC -----
def test_fc_golden():
    g = GOLD["fc_pack_2x2"]
    assert R.fc_weight_eq10_literal(np.array(g["W"])).tolist() == g["expect_w"]
    w = np.zeros(g["N"], np.int64)
    for e, c in R.fc_weight_terms(np.array(g["W"]), g["N"]):
        w[e] += c
    assert w.tolist() == g["expect_w"]
    g = GOLD["fc_product_2x2"]
    ip = R.fc_input_int(np.array(g["I"]), 2, g["N"])
    assert ip.tolist() == g["expect_input_poly"]
    prod = R.schoolbook_py(ip, w, g["N"])
    assert prod[:2] == g["expect"]


def test_theorem1_exhaustive():
    # Theorem 1 for (n_i, n_o) in {1..8}^2 at N = n_i n_o
    # (literal Eq. 10) and at the next power of two (R17).
    rng = np.random.default_rng(11)
    for n_i in range(1, 9):
        for n_o in range(1, 9):
            for trial in range(6):
                W = rng.integers(-8, 8, (n_o, n_i))
                I = rng.integers(0, 256, n_i)
                Bv = rng.integers(-8, 8, n_o)
                N0 = n_i * n_o
                w_lit = R.fc_weight_eq10_literal(W)
                for N in (N0, 1 << (N0 - 1).bit_length(), 2 * N0 + 3):
                    w = np.zeros(N, np.int64)
                    for e, c in R.fc_weight_terms(W, N):
                        w[e] += c
                    if N == N0:
                        assert np.array_equal(w, w_lit)
                    prod = R.schoolbook_py(R.fc_input_int(I, n_o, N), w, N)
                    got = np.array(prod[:n_o]) + Bv
                    assert np.array_equal(got, W @ I + Bv)


# ---------------------------------------------------- server definition --
def test_conv_server_integer_mode():
    """c0 = packed input (no noise, no scale) mod q: the C server definition
    must return conv mod q at the valid slots and 0 elsewhere."""
    Ly = synth.ConvLayer(8, 8, 4, 4, stride=2)
    N = 256
    plan = R.plan_conv(Ly, N)
    ring = R.Ring(N, (7681, 12289), 65537)
    rng = np.random.default_rng(5)
    B = 2
    imgs = rng.integers(0, 256, (B, 8, 4, 4))
    W = rng.integers(-8, 8, (8, 8, 3, 3))
    c0 = np.stack([R.signed_to_residues(R.pack_input_int(imgs[b], plan), ring)
                   for b in range(B)])
    out = R.conv_server(c0, W, plan, ring)
    pos = R.output_positions(plan)
    mask = np.ones(N, bool)
    mask[[plan.s * j + plan.t_n(n) for j in range(N // plan.s)
          for n in range(plan.c_ob)]] = False
    for b in range(B):
        ref = R.conv2d_ref(imgs[b], W, plan)
        for ob in range(plan.n_ob):
            for j, q in enumerate(ring.primes):
                got = out[b, ob, j, pos].astype(np.int64)
                want = np.stack([ref[ob * plan.c_ob + nl].ravel()
                                 for nl in range(plan.c_ob)], 1).ravel() % q
                assert np.array_equal(got, want)
                assert np.all(out[b, ob, j, mask] == 0)


def test_fc_server_integer_mode():
    n_i, n_o, N = 6, 5, 64
    ring = R.Ring(N, (7681, 12289), 65537)
    rng = np.random.default_rng(9)
    W = rng.integers(-8, 8, (n_o, n_i))
    I = rng.integers(0, 256, (3, n_i))
    c0 = np.stack([R.signed_to_residues(R.fc_input_int(I[b], n_o, N), ring)
                   for b in range(3)])
    out = R.fc_server(c0, W, None, ring)
    for b in range(3):
        for j, q in enumerate(ring.primes):
            assert np.array_equal(out[b, j].astype(np.int64), (W @ I[b]) % q)


def test_conv_reads_only_input_channel_columns():
    """DESIGN.md §4 (k_u): the filter's exponents are -m mod s (m < c_ib), so
    the server output at the valid slots depends on c0 only through the
    coefficients g s + u with u < c_ib.  Zeroing every other coefficient of
    c0 leaves the oracle's full output unchanged (on all s j + t_n slots)."""
    for Ly, N in [(synth.ConvLayer(3, 8, 8, 8), 1024), (synth.ConvLayer(5, 6, 4, 4), 1024),
                  (synth.ConvLayer(3, 4, 6, 6, pad=0), 1024)]:
        ring = R.Ring(N, synth.PRIMES_CFG1, 65537)
        plan = R.plan_conv(Ly, N)
        assert plan.c_ib < plan.s
        rng = np.random.default_rng(N + Ly.c_i)
        W = rng.integers(-8, 8, (Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h))
        c0 = synth.uniform_residues((2, plan.n_ib, ring.L, N), ring.primes, 4, "misc", Ly.c_i)
        full = R.conv_server(c0, W, plan, ring, None)
        mask = (np.arange(N) % plan.s) < plan.c_ib
        sparse = R.conv_server(np.where(mask, c0, 0).astype(np.uint64), W, plan, ring, None)
        assert np.array_equal(full, sparse)
