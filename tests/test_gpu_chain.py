"""GPU chained pipeline: three Conv layers (one with
stride 2) and the FC run encrypted layer to layer on the GPU -- client
encryption, server Conv/FC with masks, client share, decryption, the R29 stub
-- and every layer's activations and the logits equal the oracle's
plaintext chain exactly."""
import numpy as np
import pytest
import torch

import synth
from oracle import ref as R

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(),
                                 reason="needs a CUDA GPU")]


def dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(a).cuda()


@pytest.mark.parametrize("cfg_idx,B", [(2, 2), (3, 3)])
def test_chain_matches_plain_reference(cfg_idx, B):
    import paper_2409_05205_b200 as he
    from paper_2409_05205_b200.chain import Chain
    cfg = synth.CONFIGS[cfg_idx]
    N, t = cfg.N, cfg.t
    ctx = he.Context(cfg.primes, cfg.log2N, t)
    ring = R.Ring(N, cfg.primes, t)
    layers = [synth.ConvLayer(3, 8, 16, 16), synth.ConvLayer(8, 16, 16, 16, stride=2),
              synth.ConvLayer(16, 16, 8, 8)]
    rng = np.random.default_rng(cfg_idx)
    Ws = [rng.integers(-8, 8, (Ly.c_o, Ly.c_i, 3, 3)).astype(np.int32) for Ly in layers]
    fcW = rng.integers(-8, 8, (10, 16)).astype(np.int32)
    fcB = rng.integers(-8, 8, 10).astype(np.int32)
    img = rng.integers(0, 256, (B, 3, 16, 16)).astype(np.int32)
    shift, qmax = 6, 255
    seed = 1234
    s_key = synth.secret_key(N, cfg.h, seed)
    a = synth.uniform_residues((ring.L, N), cfg.primes, seed, "a")
    b_pk = R.keygen(ring, s_key, a, synth.gauss_poly(N, cfg.sigma, seed, "e0", 9))
    plans = [R.plan_conv(Ly, N) for Ly in layers]
    ef = [np.stack([np.stack([synth.gauss_poly(N, cfg.sigma, seed, "ef", li, n, beta)
                              for beta in range(p.n_ib)]) for n in range(p.c_o)]).astype(np.int32)
          for li, p in enumerate(plans)]
    fp = R.plan_fc(16, 10, N)
    ef_fc = np.stack([np.stack([synth.gauss_poly(N, cfg.sigma, seed, "ef", 99, bb, tt)
                                for tt in range(fp.n_t)]) for bb in range(fp.n_ib)]).astype(np.int32)
    ch = Chain(ctx, layers, [dev(W) for W in Ws], dev(fcW), dev(fcB),
               dev(s_key.astype(np.int32)), dev(a), dev(b_pk), [dev(e) for e in ef], dev(ef_fc))
    v = [dev(np.stack([np.stack([synth.v_poly(N, seed, li, b, beta) for beta in range(p.n_ib)])
                       for b in range(B)]).astype(np.int32)) for li, p in enumerate(plans)]
    e0 = [dev(np.stack([np.stack([synth.gauss_poly(N, cfg.sigma, seed, "e0", li, b, beta)
                                  for beta in range(p.n_ib)]) for b in range(B)]).astype(np.int32))
          for li, p in enumerate(plans)]
    v_fc = dev(np.stack([[synth.v_poly(N, seed, 99, b, bb) for bb in range(fp.n_ib)]
                         for b in range(B)]).astype(np.int32))
    e_fc = dev(np.stack([[synth.gauss_poly(N, cfg.sigma, seed, "e0", 99, b, bb)
                          for bb in range(fp.n_ib)] for b in range(B)]).astype(np.int32))
    acts, logits = ch.run(dev(img), v, e0, 5, shift, qmax, v_fc, e_fc, keep=True)
    for b in range(B):
        ref_acts, ref_logits = R.plain_chain(img[b], Ws, layers, N, t, shift, qmax, fcW, fcB)
        for li in range(len(layers)):
            assert 0.05 < (ref_acts[li] > 0).mean() < 0.95      # non-degenerate
            assert np.array_equal(acts[li][b].cpu().numpy(), ref_acts[li]), (b, li)
        assert np.array_equal(logits[b].cpu().numpy(), ref_logits), b
