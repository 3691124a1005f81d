"""Protocol pins (not gpu): the oracle's server output, decrypted by the
oracle's client side of Algorithms 1/2, equals the brute-force layer output
mod t.  This pins the BFV encoding R2, the mask R15 and the server
definition end to end (configs 1 and 2 of BASELINE.json)."""
import numpy as np
import pytest

import synth
from oracle import ref as R


def _conv_protocol(cfg_idx: int, B: int = 1):
    cfg = synth.CONFIGS[cfg_idx]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    Ly = cfg.conv[0]
    plan = R.plan_conv(Ly, cfg.N)
    seed = cfg.seed
    s_key = synth.secret_key(cfg.N, cfg.h, seed)
    a = synth.uniform_residues((ring.L, cfg.N), cfg.primes, seed, "a")
    e = synth.gauss_poly(cfg.N, cfg.sigma, seed, "e0", 999)
    b_pk = R.keygen(ring, s_key, a, e)
    imgs = synth.images(cfg, 0, B)
    W = synth.weights(cfg, 0)
    phi = synth.phi1((B, plan.n_ob, cfg.N), cfg.t, seed)
    c0 = np.empty((B, plan.n_ib, ring.L, cfg.N), np.uint64)
    vs = {}
    for b in range(B):
        ip = R.pack_input_int(imgs[b], plan)
        for beta in range(plan.n_ib):
            v = synth.v_poly(cfg.N, seed, b, beta)
            e0 = synth.gauss_poly(cfg.N, cfg.sigma, seed, "e0", b, beta)
            vs[(b, beta)] = v
            c0[b, beta] = R.encrypt_c0(ring, ip[beta], b_pk, v, e0)
    out = R.conv_server(c0, W, plan, ring, phi)
    ef = {(n, beta): synth.gauss_poly(cfg.N, cfg.sigma, seed, "ef", n, beta)
          for n in range(plan.c_o) for beta in range(plan.n_ib)}
    for b in range(B):
        dec = R.conv_protocol_decrypt(ring, plan, W, out[b], s_key, a,
                                      [vs[(b, beta)] for beta in range(plan.n_ib)],
                                      ef, phi[b])
        ref = R.centered_mod_t(R.conv2d_ref(imgs[b], W, plan), cfg.t)
        assert np.array_equal(dec, ref), \
            f"{np.count_nonzero(dec != ref)} of {dec.size} slots wrong"
    # the compact payload is exactly the valid slots
    comp = R.compact(out, plan)
    assert comp.shape == (B, plan.n_ob, ring.L, plan.n_valid)


def test_config1_protocol_decrypts_to_conv():
    _conv_protocol(1)


@pytest.mark.slow
def test_config2_protocol_decrypts_to_conv():
    _conv_protocol(2)


def test_fc_protocol_decrypts_to_wi_plus_b():
    # FC 64 -> 100 (config 4's layer) on config 2's ring (N=8192 >= 6400)
    cfg = synth.CONFIGS[2]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    seed = 77
    n_i, n_o = 64, 100
    rng = np.random.default_rng(seed)
    W = rng.integers(-8, 8, (n_o, n_i))
    Bv = rng.integers(-8, 8, n_o)
    I = rng.integers(0, 256, n_i)
    s_key = synth.secret_key(cfg.N, cfg.h, seed)
    a = synth.uniform_residues((ring.L, cfg.N), cfg.primes, seed, "a")
    b_pk = R.keygen(ring, s_key, a, synth.gauss_poly(cfg.N, 3.2, seed, "e0", 9))
    v = synth.v_poly(cfg.N, seed, 0)
    c0 = R.encrypt_c0(ring, R.fc_input_int(I, n_o, cfg.N), b_pk, v,
                      synth.gauss_poly(cfg.N, 3.2, seed, "e0", 0))
    phi = synth.phi1((1, n_o), cfg.t, seed)
    out = R.fc_server(c0[None], W, Bv, ring, phi)
    ef = synth.gauss_poly(cfg.N, 3.2, seed, "ef", 0)
    dec = R.fc_protocol_decrypt(ring, W, out[0], s_key, a, v, ef, phi[0])
    assert np.array_equal(dec, R.centered_mod_t(W @ I + Bv, cfg.t))
