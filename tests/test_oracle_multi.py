"""Pins for the oracle's multi-image packing (reading
R31, a protocol extension): P images at offsets p*D of one ciphertext give,
at image p's shifted valid slots, exactly image p's brute-force convolution
Eq. (3)/(4); the spacing D = s h_p (w_p + 1) is needed; and
a trivially encrypted multi-image ciphertext through the server definition
decrypts to every image's conv mod t."""
import numpy as np
import pytest

import synth
from oracle import ref as R


def negacyclic_int(a, f):
    """a(X) f(X) mod X^N + 1 over Z by the textbook definition (numpy
    convolution, then X^N = -1 folding) -- independent of the oracle's
    modular product routines."""
    N = a.shape[-1]
    full = np.convolve(a.astype(np.int64), f.astype(np.int64))
    out = full[:N].copy()
    out[: len(full) - N] -= full[N:]
    return out


CASES = [
    (synth.ConvLayer(2, 3, 4, 4), 1024, 2),            # s = 2, D = 84, P = 12
    (synth.ConvLayer(3, 2, 5, 4), 1024, 4),            # rectangular, c_i < s
    (synth.ConvLayer(4, 4, 4, 4, stride=2), 2048, 4),  # stride 2
    (synth.ConvLayer(6, 2, 3, 3), 1024, 4),            # n_ib = 2 (c_ib = 4)
    (synth.ConvLayer(2, 2, 4, 4, pad=0), 512, 2),      # valid padding
]


def _check(Ly, N, so, D, P=None):
    plan = R.plan_conv(Ly, N, so)
    D0, P0 = R.multi_image_spacing(plan)
    P = P0 if P is None else P
    rng = np.random.default_rng(N + so)
    imgs = rng.integers(-9, 10, (P, Ly.c_i, Ly.w_i, Ly.h_i))
    W = rng.integers(-8, 8, (Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h))
    c = R.pack_input_multi_int(imgs, plan, D)
    pos = R.output_positions(plan)
    ok = True
    for n in range(plan.c_o):
        prod = sum(negacyclic_int(c[beta], R.filter_poly_int(W, plan, n, beta))
                   for beta in range(plan.n_ib))
        nl = n % plan.c_ob
        for p in range(P):
            want = R.conv2d_ref(imgs[p], W, plan)[n].reshape(-1)
            got = prod[p * D + pos[nl::plan.c_ob]]
            ok &= bool(np.array_equal(got, want))
    return ok, plan, P


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-N{c[1]}-s{c[2]}")
def test_multi_image_slots_equal_bruteforce_conv(case):
    Ly, N, so = case
    plan = R.plan_conv(Ly, N, so)
    D, P = R.multi_image_spacing(plan)
    assert P >= 2
    ok, _, _ = _check(Ly, N, so, D)
    assert ok


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-N{c[1]}-s{c[2]}")
def test_tighter_spacing_breaks(case):
    # two s-steps below D the neighbour images' partial sums reach the valid
    # slots: the spacing rule is (nearly) tight, not vacuous
    Ly, N, so = case
    plan = R.plan_conv(Ly, N, so)
    D, P = R.multi_image_spacing(plan)
    ok, _, _ = _check(Ly, N, so, D - 2 * plan.s, P)
    assert not ok


def test_multi_image_trivial_encryption_decrypts_to_conv():
    cfg = synth.CONFIGS[1]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    Ly = synth.ConvLayer(1, 2, 4, 4)
    plan = R.plan_conv(Ly, cfg.N, 8)
    D, P = R.multi_image_spacing(plan)
    assert P >= 3
    rng = np.random.default_rng(9)
    imgs = rng.integers(0, 16, (P, 1, 4, 4))
    W = rng.integers(-4, 4, (2, 1, 3, 3))
    pt = np.mod(R.pack_input_multi_int(imgs, plan, D), cfg.t).astype(np.uint32)
    c0 = R.encode(pt[0], ring)[None, None]            # trivial encryption (c1 = 0)
    out = R.conv_server(c0, W, plan, ring)
    m = R.decrypt_round(R.compact_multi(out, plan, P, D), ring)   # [1][n_ob][P n_valid]
    got = R.centered_mod_t(m.astype(np.int64), cfg.t).reshape(plan.n_ob, P, -1)
    for p in range(P):
        want = R.conv2d_ref(imgs[p], W, plan)              # [c_o][w_o][h_o]
        # compact order within an image: (K, L, n)
        want_c = np.moveaxis(want, 0, -1).reshape(-1)
        assert np.array_equal(got[0, p], R.centered_mod_t(want_c, cfg.t))
