"""GPU parity of multi-image packing (reading R31):
he_multi_image_spacing / he_pack_input_multi / he_conv /
he_mask_extract_multi against the oracle (bit-exact), and a trivially
encrypted config-5 multi-image ciphertext decrypting to every image's
brute-force convolution mod t."""
import numpy as np
import pytest
import torch

import synth
from oracle import ref as R

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA GPU")]


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


CASES = [
    (synth.ConvLayer(2, 3, 4, 4), 1024, 2, 40),
    (synth.ConvLayer(3, 2, 5, 4), 1024, 4, 9),
    (synth.ConvLayer(4, 4, 4, 4, stride=2), 2048, 4, 20),
    (synth.ConvLayer(6, 2, 3, 3), 1024, 4, 13),
    (synth.ConvLayer(2, 2, 4, 4, pad=0), 512, 2, 15),
    (synth.ConvLayer(16, 24, 5, 5), 8192, 16, 11),   # n_ob = 2, c_o = 24
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-N{c[1]}-s{c[2]}-B{c[3]}")
def test_multi_image_path(case):
    import paper_2409_05205_b200 as he
    Ly, N, so, B = case
    primes = R.find_primes(N, 50, 2)
    ring = R.Ring(N, primes, 65537)
    ctx = he.Context(primes, N.bit_length() - 1, 65537)
    plan = R.plan_conv(Ly, N, so)
    p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride, Ly.pad, so)
    D, P = R.multi_image_spacing(plan)
    assert ctx.multi_image_spacing(p) == (D, P)
    rng = np.random.default_rng(B + N)
    imgs = rng.integers(0, 256, (B, Ly.c_i, Ly.w_i, Ly.h_i)).astype(np.int32)
    W = rng.integers(-8, 8, (Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h)).astype(np.int32)
    Bc = -(-B // P)
    ve = synth.uniform_residues((Bc, plan.n_ib, ring.L, N), primes, 5, "ve", B)
    c0 = ctx.pack_input_multi(p, dev(imgs), P, D, ve=dev(ve))
    got_c0 = u64(c0)
    pad_imgs = np.zeros((Bc * P,) + imgs.shape[1:], np.int32)
    pad_imgs[:B] = imgs
    for c in range(Bc):
        pt = R.pack_input_multi_int(pad_imgs[c * P:(c + 1) * P], plan, D)
        for beta in range(plan.n_ib):
            enc = R.encode(np.mod(pt[beta], 65537).astype(np.uint32), ring)
            want = (enc.astype(object) + ve[c, beta].astype(object)) % \
                ring.q_arr.astype(object)[:, None]
            assert np.array_equal(got_c0[c, beta], want.astype(np.uint64)), (c, beta)
    phi = synth.phi1((Bc, plan.n_ob, N), 65537, 6, B)
    out = ctx.conv(p, c0, ctx.pack_filters(p, dev(W)), dev(phi))
    comp = ctx.mask_extract_multi(p, out, P, D)
    ref = R.conv_server(got_c0, W, plan, ring, phi)
    assert np.array_equal(u64(out), ref)
    assert np.array_equal(u64(comp), R.compact_multi(ref, plan, P, D))
    # the mask added by the extraction instead of the conv
    out2 = ctx.conv(p, c0, ctx.pack_filters(p, dev(W)))
    comp2 = ctx.mask_extract_multi(p, out2, P, D, phi1=dev(phi))
    assert np.array_equal(u64(comp2), R.compact_multi(ref, plan, P, D))


def test_multi_image_config5_decrypts():
    """Config 5's layer at the paper's s = c_i = 64: P = 5 images per
    ciphertext (D = 5760 of N = 32768).  Trivial encryption (c1 = 0) of the
    GPU-packed images, GPU server, oracle decryption: every image's slots
    equal its brute-force conv mod t."""
    import paper_2409_05205_b200 as he
    cfg = synth.CONFIGS[5]
    primes = cfg.primes[:2]
    ring = R.Ring(cfg.N, primes, cfg.t)
    ctx = he.Context(primes, cfg.log2N, cfg.t)
    Ly = cfg.conv[0]
    plan = R.plan_conv(Ly, cfg.N, 64)
    p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, s_override=64)
    D, P = ctx.multi_image_spacing(p)
    assert (D, P) == R.multi_image_spacing(plan) and P == 5
    imgs = synth.images(cfg, 0, P)
    W = synth.weights(cfg, 0)
    c0 = ctx.pack_input_multi(p, dev(imgs), P, D)
    out = ctx.conv(p, c0, ctx.pack_filters(p, dev(W)))
    comp = u64(ctx.mask_extract_multi(p, out, P, D))
    m = R.decrypt_round(comp, ring).astype(np.int64).reshape(plan.n_ob, P, -1)
    for pi in (0, P - 1):
        want = np.moveaxis(R.conv2d_ref(imgs[pi], W, plan), 0, -1).reshape(-1)
        assert np.array_equal(R.centered_mod_t(m[0, pi], cfg.t), R.centered_mod_t(want, cfg.t))
