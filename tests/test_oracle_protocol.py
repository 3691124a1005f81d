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


def _client_steps(cfg_idx: int, layer, B: int = 2):
    """The client mirror path as separate oracle steps (server_p,
    client_c1r, decrypt_round) decrypts to the brute-force conv mod t."""
    cfg = synth.CONFIGS[cfg_idx]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    plan = R.plan_conv(layer, cfg.N)
    seed = cfg.seed + 5
    s_key = synth.secret_key(cfg.N, cfg.h, seed)
    a = synth.uniform_residues((ring.L, cfg.N), cfg.primes, seed, "a")
    b_pk = R.keygen(ring, s_key, a, synth.gauss_poly(cfg.N, cfg.sigma, seed, "e0", 9))
    rng = np.random.default_rng(seed)
    # the config's value ranges keep the noise inside Delta/2 (config 1 has
    # a single 30-bit limb)
    imgs = rng.integers(cfg.img_lo, cfg.img_hi + 1,
                        (B, layer.c_i, layer.w_i, layer.h_i))
    W = rng.integers(cfg.w_lo, cfg.w_hi + 1,
                     (layer.c_o, layer.c_i, layer.f_w, layer.f_h))
    phi = synth.phi1((B, plan.n_ob, cfg.N), cfg.t, seed)
    c0 = np.empty((B, plan.n_ib, ring.L, cfg.N), np.uint64)
    vs = np.empty_like(c0)
    for b in range(B):
        ip = R.pack_input_int(imgs[b], plan)
        for beta in range(plan.n_ib):
            v = synth.v_poly(cfg.N, seed, b, beta)
            c0[b, beta] = R.encrypt_c0(ring, ip[beta], b_pk, v, synth.gauss_poly(
                cfg.N, cfg.sigma, seed, "e0", b, beta))
            vs[b, beta] = R.signed_to_residues(
                np.array(R.schoolbook_py(v, s_key, cfg.N)), ring)
    out = R.conv_server(c0, W, plan, ring, phi)
    ef = {(n, beta): synth.gauss_poly(cfg.N, cfg.sigma, seed, "ef", n, beta)
          for n in range(plan.c_o) for beta in range(plan.n_ib)}
    p = R.server_p(W, plan, ring, a, ef)
    c1 = R.client_c1r(vs, p, plan, ring)
    # c1^r is zero outside the slots s j + t_n (R14), like the full c0^r
    for ob in range(plan.n_ob):
        mask = np.ones(cfg.N, bool)
        for nl in range(plan.c_ob):
            if ob * plan.c_ob + nl < plan.c_o:
                mask[plan.t_n(ob * plan.c_ob + nl)::plan.s] = False
        assert not c1[:, ob][..., mask].any()
    pos = R.output_positions(plan)
    qo = np.array(ring.primes, dtype=object)[None, None, :, None]
    m = R.decrypt_round((out.astype(object) + c1.astype(object)) % qo, ring)
    for b in range(B):
        ref = R.centered_mod_t(R.conv2d_ref(imgs[b], W, plan), cfg.t)
        for ob in range(plan.n_ob):
            got = (m[b, ob, pos].astype(np.int64) - phi[b, ob, pos]) % cfg.t
            got = np.where(got > cfg.t // 2, got - cfg.t, got)
            for nl in range(plan.c_ob):
                n = ob * plan.c_ob + nl
                if n < plan.c_o:
                    assert np.array_equal(got[nl::plan.c_ob],
                                          ref[n].ravel()), (b, n)


def test_client_steps_config1():
    _client_steps(1, synth.CONFIGS[1].conv[0])


def test_client_steps_two_blocks_each_way():
    # n_ib = n_ob = 2 on config 1's ring: c_i = c_o = 2 s
    L0 = synth.CONFIGS[1].conv[0]
    plan0 = R.plan_conv(L0, 1024)
    Ly = synth.ConvLayer(c_i=2 * plan0.s, c_o=2 * plan0.s, w_i=L0.w_i, h_i=L0.h_i,
                         f_w=3, f_h=3, stride=1, pad=1)
    plan = R.plan_conv(Ly, 1024)
    assert plan.n_ib == 2 and plan.n_ob == 2
    _client_steps(1, Ly, B=1)


def test_decrypt_round_definition():
    # round(t r / Q) mod t by exact rationals with an independent CRT on
    # random residues, and Delta m + small noise decrypts to m (Eq. (2) in
    # the BFV reading R1)
    from fractions import Fraction
    cfg = synth.CONFIGS[2]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    rng = np.random.default_rng(3)
    r = np.stack([rng.integers(0, q, cfg.N, dtype=np.uint64) for q in ring.primes])
    got = R.decrypt_round(r, ring)
    Q = 1
    for q in ring.primes:
        Q *= q
    for k in range(0, cfg.N, 97):
        val = 0
        for j, q in enumerate(ring.primes):
            Qj = Q // q
            val += int(r[j, k]) * Qj * pow(Qj, -1, q)
        val %= Q
        want = (Fraction(cfg.t * val, Q) + Fraction(1, 2)).__floor__() % cfg.t
        assert int(got[k]) == want
    m = rng.integers(0, cfg.t, cfg.N).astype(np.uint32)
    enc = R.encode(m, ring)
    noise = rng.integers(-1000, 1000, cfg.N)
    enc_n = np.stack([(enc[j].astype(object) + noise) % q
                      for j, q in enumerate(ring.primes)]).astype(np.uint64)
    assert np.array_equal(R.decrypt_round(enc_n, ring), m)


@pytest.mark.parametrize("n_i,n_o", [(20, 30), (300, 5), (16, 16), (7, 200), (257, 3)])
def test_fc_tiled_decrypts_to_wi_plus_b(n_i, n_o):
    """R27 sub-matrix tiling for n_i n_o > N: with the
    trivial-key ciphertexts c0_beta = enc(i_beta) (Eq. (9) per input block),
    round(t c0^r / Q) - phi1 = W I + B mod t (Thm. 1 per sub-matrix, summed
    over input blocks)."""
    N, primes = 256, (7681, 12289, 40961)
    ring = R.Ring(N, primes, 65537)
    rng = np.random.default_rng(n_i * 1000 + n_o)
    W = rng.integers(-8, 8, (n_o, n_i))
    Bv = rng.integers(-8, 8, n_o)
    I = rng.integers(0, 256, (2, n_i))
    fp = R.plan_fc(n_i, n_o, N)
    assert fp.n_it * fp.n_ot <= N and fp.n_ib * fp.n_it >= n_i and fp.n_t * fp.n_ot >= n_o
    c0 = np.stack([np.stack([R.encode(np.mod(blk, ring.t).astype(np.uint32), ring)
                             for blk in R.fc_input_blocks(I[b], fp)]) for b in range(2)])
    phi = synth.phi1((2, n_o), ring.t, 5)
    out = R.fc_server_tiled(c0, W, Bv, ring, phi)
    m = R.decrypt_round(out, ring).astype(np.int64)
    got = R.centered_mod_t(m - phi, ring.t)
    assert np.array_equal(got, R.centered_mod_t(I @ W.T + Bv, ring.t))


def test_mod_switch_definition_and_protocol():
    """R28: round(Q' x / Q) by exact rationals, and the switched shares of a
    real protocol run (config 2, L = 3 -> L' = 1) still decrypt, under Q',
    to the brute-force conv mod t."""
    from fractions import Fraction
    cfg = synth.CONFIGS[2]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    rng = np.random.default_rng(8)
    r = np.stack([rng.integers(0, q, 50, dtype=np.uint64) for q in ring.primes])
    for Lk in (1, 2):
        sw = R.mod_switch(r, ring, Lk)
        Qp = 1
        for q in ring.primes[:Lk]:
            Qp *= q
        for k in range(0, 50, 7):
            x = 0
            for j, q in enumerate(ring.primes):
                Qj = ring.Q // q
                x += int(r[j, k]) * Qj * pow(Qj, -1, q)
            x %= ring.Q
            want = (Fraction(Qp * x, ring.Q) + Fraction(1, 2)).__floor__() % Qp
            assert [int(sw[j, k]) for j in range(Lk)] == [want % q for q in ring.primes[:Lk]]
    # protocol: switch c0^r (server) and c1^r (client) to one limb
    Ly = cfg.conv[0]
    plan = R.plan_conv(Ly, cfg.N)
    seed = cfg.seed + 9
    s_key = synth.secret_key(cfg.N, cfg.h, seed)
    a = synth.uniform_residues((ring.L, cfg.N), cfg.primes, seed, "a")
    b_pk = R.keygen(ring, s_key, a, synth.gauss_poly(cfg.N, cfg.sigma, seed, "e0", 9))
    img = synth.images(cfg, 0, 1)
    W = synth.weights(cfg, 0)
    v = synth.v_poly(cfg.N, seed, 0, 0)
    c0 = R.encrypt_c0(ring, R.pack_input_int(img[0], plan)[0], b_pk, v,
                      synth.gauss_poly(cfg.N, cfg.sigma, seed, "e0", 0, 0))[None, None]
    phi = synth.phi1((1, plan.n_ob, cfg.N), cfg.t, seed)
    comp0 = R.compact(R.conv_server(c0, W, plan, ring, phi), plan)
    ef = {(n, 0): synth.gauss_poly(cfg.N, cfg.sigma, seed, "ef", n, 0) for n in range(Ly.c_o)}
    vs = R.signed_to_residues(np.array(R.schoolbook_py(v, s_key, cfg.N)), ring)[None, None]
    comp1 = R.compact(R.client_c1r(vs, R.server_p(W, plan, ring, a, ef), plan, ring), plan)
    ring1 = R.Ring(cfg.N, cfg.primes[:1], cfg.t)
    s0, s1 = R.mod_switch(comp0, ring, 1), R.mod_switch(comp1, ring, 1)
    m = R.decrypt_round((s0.astype(object) + s1.astype(object)) % cfg.primes[0], ring1)
    got = R.centered_mod_t(m[0, 0].astype(np.int64) - phi[0, 0, R.output_positions(plan)], cfg.t)
    ref = R.centered_mod_t(R.conv2d_ref(img[0], W, plan), cfg.t)
    want = np.stack([ref[nl].ravel() for nl in range(plan.c_ob)], 1).ravel()
    assert np.array_equal(got, want)


def test_chained_protocol_matches_plain_chain():
    """R29: two Conv layers (the second with stride 2) and the FC, each run
    through the oracle's encrypted protocol (c0-only encryption, server,
    client c1^r, decryption) with the stub between layers, reproduce the
    plaintext chain exactly (Fig. 5)."""
    cfg = synth.CONFIGS[1]
    N, t = cfg.N, cfg.t
    ring = R.Ring(N, cfg.primes, t)
    layers = [synth.ConvLayer(1, 2, 8, 8), synth.ConvLayer(2, 2, 8, 8, stride=2)]
    rng = np.random.default_rng(3)
    Ws = [rng.integers(-4, 4, (Ly.c_o, Ly.c_i, 3, 3)) for Ly in layers]
    fcW, fcB = rng.integers(-4, 4, (3, 2)), rng.integers(-4, 4, 3)
    img = rng.integers(0, 16, (1, 8, 8))
    shift, qmax = 2, 15
    acts, logits = R.plain_chain(img, Ws, layers, N, t, shift, qmax, fcW, fcB)
    seed = 77
    s_key = synth.secret_key(N, cfg.h, seed)
    a = synth.uniform_residues((ring.L, N), cfg.primes, seed, "a")
    b_pk = R.keygen(ring, s_key, a, synth.gauss_poly(N, cfg.sigma, seed, "e0", 9))
    x = img
    for li, (W, Ly) in enumerate(zip(Ws, layers)):
        plan = R.plan_conv(Ly, N)
        ip = R.pack_input_int(x, plan)
        vs = [synth.v_poly(N, seed, li, beta) for beta in range(plan.n_ib)]
        c0 = np.stack([R.encrypt_c0(ring, ip[beta], b_pk, vs[beta],
                                    synth.gauss_poly(N, cfg.sigma, seed, "e0", li, beta))
                       for beta in range(plan.n_ib)])[None]
        phi = synth.phi1((1, plan.n_ob, N), t, seed, li)
        out = R.conv_server(c0, W, plan, ring, phi)
        ef = {(n, beta): synth.gauss_poly(N, cfg.sigma, seed, "ef", li, n, beta)
              for n in range(plan.c_o) for beta in range(plan.n_ib)}
        dec = R.conv_protocol_decrypt(ring, plan, W, out[0], s_key, a, vs, ef, phi[0])
        x = np.minimum(qmax, np.maximum(dec, 0) >> shift)
        assert np.array_equal(x, acts[li]), li
    v_in = R.avgpool(x)
    v = synth.v_poly(N, seed, 99)
    c0 = R.encrypt_c0(ring, R.fc_input_int(v_in, 3, N), b_pk, v,
                      synth.gauss_poly(N, cfg.sigma, seed, "e0", 99))
    phi = synth.phi1((1, 3), t, seed, 99)
    out = R.fc_server(c0[None], fcW, fcB, ring, phi)
    dec = R.fc_protocol_decrypt(ring, fcW, out[0], s_key, a, v,
                                synth.gauss_poly(N, cfg.sigma, seed, "ef", 99), phi[0])
    assert np.array_equal(dec, logits)
