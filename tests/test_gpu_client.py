"""GPU parity for the client mirror path (first "next" row):
server initialisation p = fhat a + e_f (Alg. 1 Line 5), the client's
c1^r (Lines 21-24) through he_pack_client_p + he_conv, negacyclic products,
and the decryption rounding of Eq. (2) -- each against the CPU oracle, and
the whole protocol decrypted on the GPU against the brute-force conv mod t.
Bit-exact on every residue and every decoded value.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import ref as R

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(),
                                 reason="needs a CUDA GPU")]


@pytest.fixture(scope="module")
def he():
    import paper_2409_05205_b200 as he
    return he


def u64(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)


def dev(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


_CTX = {}


def ctx_for(he, N, primes, t=65537):
    key = (N, tuple(primes), t)
    if key not in _CTX:
        _CTX[key] = he.Context(primes, N.bit_length() - 1, t)
    return _CTX[key]


RINGS = {
    256: (7681, 12289, 40961),
    1024: tuple(synth.PRIMES_CFG1) + (R.find_primes(1024, 50, 1)[0],),
    8192: tuple(synth.PRIMES_N8192[:3]),
    32768: tuple(synth.PRIMES_N32768[:2]),
}


@pytest.mark.parametrize("N", sorted(RINGS))
@pytest.mark.parametrize("ybc", [True, False])
def test_poly_mul_and_residues_from_int(he, N, ybc):
    primes = RINGS[N]
    ring = R.Ring(N, primes, 65537)
    ctx = ctx_for(he, N, primes)
    rng = np.random.default_rng(N + ybc)
    B = 3
    xi = rng.integers(-2 ** 20, 2 ** 20, (B, N)).astype(np.int32)
    xi[0, :4] = [-2 ** 31, 2 ** 31 - 1, 0, -1]                 # extremes
    xr = ctx.residues_from_int(dev(xi))
    got_r = u64(xr)
    for b in range(B):
        assert np.array_equal(got_r[b], R.signed_to_residues(xi[b].astype(np.int64), ring))
    y = synth.uniform_residues((1 if ybc else B, ring.L, N), primes, 5, "misc", N)
    out = u64(ctx.poly_mul(xr, dev(y)))
    pos = np.arange(N) if N <= 1024 else np.unique(
        np.concatenate([[0, 1, N - 1], rng.integers(0, N, 24)]))
    for b in (0, B - 1):
        for j, q in enumerate(primes):
            want = R.negacyclic_at(got_r[b, j], y[0 if ybc else b, j], q, pos)
            assert np.array_equal(out[b, j, pos], want), (b, j)


def _layer_cases():
    L1 = synth.CONFIGS[1].conv[0]
    two = synth.ConvLayer(c_i=16, c_o=16, w_i=8, h_i=8)   # n_ib = n_ob = 2 at N=1024
    valid = synth.ConvLayer(c_i=3, c_o=5, w_i=9, h_i=7, pad=0)
    return [("cfg1", 1024, L1), ("two_blocks", 1024, two), ("valid_ragged", 1024, valid),
            ("n8192", 8192, synth.ConvLayer(c_i=20, c_o=12, w_i=16, h_i=16))]


@pytest.mark.parametrize("name,N,layer", _layer_cases(), ids=lambda v: str(v)
                         if isinstance(v, (str, int)) else "")
def test_server_p_and_client_c1r(he, name, N, layer):
    primes = RINGS[N]
    ring = R.Ring(N, primes, 65537)
    ctx = ctx_for(he, N, primes)
    plan = R.plan_conv(layer, N)
    p = ctx.plan(layer.c_i, layer.c_o, layer.w_i, layer.h_i, layer.f_w, layer.f_h,
                 layer.stride, layer.pad)
    seed = 31 + N
    rng = np.random.default_rng(seed)
    W = rng.integers(-8, 8, (layer.c_o, layer.c_i, layer.f_w, layer.f_h)).astype(np.int32)
    a = synth.uniform_residues((ring.L, N), primes, seed, "a")
    ef = np.stack([np.stack([synth.gauss_poly(N, 3.2, seed, "ef", n, beta)
                             for beta in range(plan.n_ib)]) for n in range(plan.c_o)])
    p_gpu = ctx.server_init_p(p, dev(W), dev(a), dev(ef.astype(np.int32)))
    efd = {(n, beta): ef[n, beta] for n in range(plan.c_o) for beta in range(plan.n_ib)}
    p_ref = R.server_p(W, plan, ring, a, efd)
    assert np.array_equal(u64(p_gpu), p_ref)
    # client: vs = v_beta s (residues), c1^r through the conv machinery
    B = 2
    vs = synth.uniform_residues((B, plan.n_ib, ring.L, N), primes, seed, "misc", 77)
    pspec = ctx.pack_client_p(p, p_gpu)
    c1 = u64(ctx.conv(ctx.dense_plan(p), dev(vs), pspec))
    want = R.client_c1r(vs, p_ref, plan, ring)
    assert np.array_equal(c1, want)


@pytest.mark.parametrize("cfg_idx", [1, 2, 4])
def test_decrypt_round_matches_oracle(he, cfg_idx):
    cfg = synth.CONFIGS[cfg_idx]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    n, ln = 3, 777                                     # ragged length
    r0 = synth.uniform_residues((n, ring.L, ln), cfg.primes, 3, "misc", cfg_idx)
    r1 = synth.uniform_residues((n, ring.L, ln), cfg.primes, 4, "misc", cfg_idx)
    m = ctx.decrypt_round(dev(r0), dev(r1)).cpu().numpy().view(np.uint32)
    qo = np.array(cfg.primes, dtype=object)[None, :, None]
    rs = ((r0.astype(object) + r1.astype(object)) % qo).astype(np.uint64)
    want = np.stack([R.crt_decode([rs[i, j] for j in range(ring.L)], ring)
                     for i in range(n)]).astype(np.uint32)
    assert np.array_equal(m, want)
    m0 = ctx.decrypt_round(dev(r0)).cpu().numpy().view(np.uint32)
    want0 = np.stack([R.crt_decode([r0[i, j] for j in range(ring.L)], ring)
                      for i in range(n)]).astype(np.uint32)
    assert np.array_equal(m0, want0)
    # enc(m) + small noise decodes to m (Eq. (2))
    msg = np.random.default_rng(cfg_idx).integers(0, cfg.t, (1, cfg.N)).astype(np.uint32)
    enc = R.encode(msg[0], ring)
    noise = np.random.default_rng(9).integers(-500, 500, cfg.N)
    enc_n = np.stack([(enc[j].astype(object) + noise) % q
                      for j, q in enumerate(cfg.primes)]).astype(np.uint64)
    assert np.array_equal(ctx.decrypt_round(dev(enc_n[None])).cpu().numpy()
                          .view(np.uint32), msg)


@pytest.mark.parametrize("cfg_idx", [1, 2])
def test_protocol_end_to_end_on_gpu(he, cfg_idx):
    """Alg. 1 with every ring operation on the GPU: client encryption
    (v b + e0 via he_poly_mul), server conv + mask (a1-a7), server init p
    (Line 5), client c1^r (Lines 21-24), decryption (Eq. 2); the decrypted
    valid slots minus phi1 equal the brute-force conv mod t.  Checked on the
    full output rows and on the compact payload."""
    cfg = synth.CONFIGS[cfg_idx]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    Ly = cfg.conv[0]
    plan = R.plan_conv(Ly, cfg.N)
    p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride, Ly.pad)
    seed = cfg.seed + 17
    B = 2
    s_key = synth.secret_key(cfg.N, cfg.h, seed)
    a = synth.uniform_residues((ring.L, cfg.N), cfg.primes, seed, "a")
    b_pk = R.keygen(ring, s_key, a, synth.gauss_poly(cfg.N, cfg.sigma, seed, "e0", 999))
    imgs = synth.images(cfg, 0, B).astype(np.int32)
    W = synth.weights(cfg, 0).astype(np.int32)
    v = np.stack([np.stack([synth.v_poly(cfg.N, seed, b, beta) for beta in range(plan.n_ib)])
                  for b in range(B)]).astype(np.int32)
    e0 = np.stack([np.stack([synth.gauss_poly(cfg.N, cfg.sigma, seed, "e0", b, beta)
                             for beta in range(plan.n_ib)]) for b in range(B)]).astype(np.int32)
    ef = np.stack([np.stack([synth.gauss_poly(cfg.N, cfg.sigma, seed, "ef", n, beta)
                             for beta in range(plan.n_ib)])
                   for n in range(plan.c_o)]).astype(np.int32)
    phi = synth.phi1((B, plan.n_ob, cfg.N), cfg.t, seed)
    qd = torch.tensor(cfg.primes, dtype=torch.int64, device="cuda")[:, None]
    # client: encryption randomness v b + e0 (Alg. 1 Line 10), then Eq. (5)
    vr = ctx.residues_from_int(dev(v))
    vb = ctx.poly_mul(vr, dev(b_pk[None]))
    ve = (vb + ctx.residues_from_int(dev(e0))) % qd
    c0 = ctx.pack_input(p, dev(imgs), ve)
    # server
    fspec = ctx.pack_filters(p, dev(W))
    comp = ctx.empty_u64(B, p.n_ob, ctx.L, p.n_valid)
    c0r = ctx.conv(p, c0, fspec, dev(phi.astype(np.uint32)), compact=comp)
    pp = ctx.server_init_p(p, dev(W), dev(a), dev(ef))
    # client: v s, c1^r, decryption
    sr = ctx.residues_from_int(dev(s_key.astype(np.int32)[None]))
    vs = ctx.poly_mul(vr.reshape(B * plan.n_ib, ctx.L, cfg.N), sr).reshape(
        B, plan.n_ib, ctx.L, cfg.N)
    pspec = ctx.pack_client_p(p, pp)
    comp1 = ctx.empty_u64(B, p.n_ob, ctx.L, p.n_valid)
    c1r = ctx.conv(ctx.dense_plan(p), vs, pspec, compact=comp1)
    m_full = ctx.decrypt_round(c0r, c1r).cpu().numpy().view(np.uint32)
    m_comp = ctx.decrypt_round(comp, comp1).cpu().numpy().view(np.uint32)
    # modulus switching of both shares to one limb (R28), decrypted under Q'
    ctx1 = ctx_for(he, cfg.N, cfg.primes[:1], cfg.t)
    m_sw = ctx1.decrypt_round(ctx.mod_switch(comp, 1), ctx.mod_switch(comp1, 1)) \
        .cpu().numpy().view(np.uint32)
    pos = R.output_positions(plan)
    for b in range(B):
        ref = R.centered_mod_t(R.conv2d_ref(imgs[b], W, plan), cfg.t)
        for ob in range(plan.n_ob):
            for m_row, sel in ((m_full[b, ob, pos], pos), (m_comp[b, ob], pos),
                               (m_sw[b, ob], pos)):
                got = (m_row.astype(np.int64) - phi[b, ob, sel]) % cfg.t
                got = np.where(got > cfg.t // 2, got - cfg.t, got)
                for nl in range(plan.c_ob):
                    n = ob * plan.c_ob + nl
                    if n < plan.c_o:
                        assert np.array_equal(got[nl::plan.c_ob], ref[n].ravel()), (b, n)


@pytest.mark.parametrize("cfg_idx", [2, 4, 5])
def test_mod_switch_matches_oracle(he, cfg_idx):
    cfg = synth.CONFIGS[cfg_idx]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    x = synth.uniform_residues((2, ring.L, 97), cfg.primes, 6, "misc", cfg_idx)
    for Lk in sorted({1, 2, ring.L - 1, ring.L}):
        got = u64(ctx.mod_switch(dev(x), Lk))
        assert np.array_equal(got, R.mod_switch(x, ring, Lk)), Lk


@pytest.mark.parametrize("cfg_idx,li", [(5, 0), (4, 0), (4, 14), (1, 0)])
def test_sparse_c0_upload(he, cfg_idx, li):
    """Protocol extension: the client sends only the k_u columns of c0
    (he_c0_compact); the server expands them (he_c0_expand, zeros elsewhere)
    and he_conv returns exactly the oracle's output for the full c0."""
    cfg = synth.CONFIGS[cfg_idx]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    Ly = cfg.conv[li]
    plan = R.plan_conv(Ly, cfg.N)
    p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride, Ly.pad)
    B = 4
    W = synth.weights(cfg, li)
    c0 = synth.uniform_residues((B, p.n_ib, ring.L, cfg.N), cfg.primes, 12, "misc", li)
    phi = synth.phi1((B, p.n_ob, cfg.N), cfg.t, 12)
    fspec = ctx.pack_filters(p, dev(W))
    c0c = ctx.c0_compact(p, dev(c0))
    assert c0c.shape[-1] == (cfg.N // p.s) * p.k_u
    c0x = ctx.c0_expand(p, c0c)
    out = u64(ctx.conv(p, c0x, fspec, dev(phi.astype(np.uint32))))
    for b in (0, B - 1):
        assert np.array_equal(out[b], R.conv_server(c0[b:b + 1], W, plan, ring, phi[b:b + 1])[0])


def test_pk_mask_vs_matches_separate_products(he):
    """he_pk_mask_vs (shared NTT(v)) equals v b + e and v s computed by the
    oracle's negacyclic products."""
    cfg = synth.CONFIGS[2]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    v = np.stack([synth.v_poly(cfg.N, 5, i) for i in range(3)]).astype(np.int32)
    e = np.stack([synth.gauss_poly(cfg.N, 3.2, 5, "e0", i) for i in range(3)]).astype(np.int32)
    b = synth.uniform_residues((ring.L, cfg.N), cfg.primes, 5, "a")
    s_key = synth.secret_key(cfg.N, cfg.h, 5)
    s_res = R.signed_to_residues(s_key, ring)
    ve, vs = ctx.pk_mask_vs(dev(v), dev(e), dev(b), dev(s_res))
    ve, vs = u64(ve), u64(vs)
    pos = np.array([0, 1, 2, 100, cfg.N // 2, cfg.N - 1])
    for i in range(3):
        vr = R.signed_to_residues(v[i].astype(np.int64), ring)
        er = R.signed_to_residues(e[i].astype(np.int64), ring)
        for j, q in enumerate(cfg.primes):
            want_ve = (R.negacyclic_at(vr[j], b[j], q, pos).astype(object) +
                       er[j][pos].astype(object)) % q
            assert [int(x) for x in ve[i, j, pos]] == [int(x) for x in want_ve]
            assert np.array_equal(vs[i, j, pos], R.negacyclic_at(vr[j], s_res[j], q, pos))
