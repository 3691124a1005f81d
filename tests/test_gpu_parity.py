"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bit-exact on every compared residue (integer work).  Sizes: small rings
with several tiles and ragged batches, every BASELINE.json config (configs
1-5 in full -- every image and limb at the bench batch), plus edge cases (B = 0, valid padding, s_override, stride 2,
n_ib / n_ob > 1, masks on/off, N = 256 .. 32768).
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


def brv(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


_CTX = {}


def ctx_for(he, N, primes, t=65537):
    key = (N, tuple(primes), t)
    if key not in _CTX:
        _CTX[key] = he.Context(primes, N.bit_length() - 1, t)
    return _CTX[key]


RINGS = {
    256: (7681, 12289, 40961),
    1024: tuple(synth.PRIMES_CFG1) + (R.find_primes(1024, 50, 1)[0],),
    8192: tuple(synth.PRIMES_N8192[:2]),
    16384: tuple(synth.PRIMES_N16384[:2]),
    32768: tuple(synth.PRIMES_N32768[:2]),
}


# ------------------------------------------------------------- transforms
@pytest.mark.parametrize("N", sorted(RINGS))
def test_ntt_forward_matches_definition(he, N):
    primes = RINGS[N]
    ctx = ctx_for(he, N, primes)
    logN = N.bit_length() - 1
    for j, q in enumerate(primes):
        assert ctx.psi(j) == R.min_psi(q, N)          # R9, independently
    batch = 3
    x = synth.uniform_residues((batch, len(primes), N), primes, 1, "misc", N)
    d = dev(x)
    ctx.ntt_forward(d)
    got = u64(d)
    rng = np.random.default_rng(N)
    pos = np.arange(N) if N <= 1024 else np.unique(
        np.concatenate([[0, 1, N - 1], rng.integers(0, N, 40)]))
    for b in (0, batch - 1):
        for j, q in enumerate(primes):
            ks = np.array([brv(int(p), logN) for p in pos], np.int32)
            want = R.ntt_def(x[b, j], q, ctx.psi(j), ks)
            assert np.array_equal(got[b, j, pos], want)


@pytest.mark.parametrize("N", sorted(RINGS))
def test_ntt_roundtrip(he, N):
    primes = RINGS[N]
    ctx = ctx_for(he, N, primes)
    x = synth.uniform_residues((5, len(primes), N), primes, 2, "misc", N)
    d = dev(x)
    ctx.ntt_forward(d)
    assert not np.array_equal(u64(d), x)
    ctx.ntt_inverse(d)
    assert np.array_equal(u64(d), x)


@pytest.mark.parametrize("N", [2048, 4096])
def test_ntt_roundtrip_cluster_sizes(he, N):
    """The FP64 inverse kernel's other single-CTA sizes (log2 N - 1 = 10, 11
    in-segment stages before its fused register step), forward pinned to the
    definition on sampled outputs, inverse by the round trip."""
    primes = tuple(R.find_primes(N, 50, 2))
    ctx = ctx_for(he, N, primes)
    logN = N.bit_length() - 1
    x = synth.uniform_residues((3, len(primes), N), primes, 4, "misc", N)
    d = dev(x)
    ctx.ntt_forward(d)
    got = u64(d)
    pos = np.array([0, 1, 5, N // 2, N - 1])
    ks = np.array([brv(int(p), logN) for p in pos], np.int32)
    for j, q in enumerate(primes):
        assert np.array_equal(got[2, j, pos], R.ntt_def(x[2, j], q, ctx.psi(j), ks))
    ctx.ntt_inverse(d)
    assert np.array_equal(u64(d), x)


def test_ntt_inverse_matches_definition(he):
    N, primes = 256, RINGS[256]
    ctx = ctx_for(he, N, primes)
    X = synth.uniform_residues((1, 3, N), primes, 3, "misc")
    d = dev(X)
    ctx.ntt_inverse(d)
    got = u64(d)
    for j, q in enumerate(primes):
        nat = np.empty(N, np.uint64)         # bit-reversed -> natural order
        for p in range(N):
            nat[brv(p, 8)] = X[0, j, p]
        assert np.array_equal(got[0, j], R.intt_def(nat, q, ctx.psi(j)))


def extreme_residues(shape, primes, kind):
    """Structured worst-case magnitudes, [..., L, N]: every residue q - 1,
    q - 1 / 0 alternating, (q - 1) / 2 + (i & 1), or q - 1 - (i mod 7)."""
    N = shape[-1]
    q = np.array(primes, np.uint64)[:, None]
    i = np.arange(N, dtype=np.uint64)[None, :]
    if kind == "max":
        v = q - 1 + 0 * i
    elif kind == "alt":
        v = np.where(i % 2 == 0, q - 1, 0).astype(np.uint64)
    elif kind == "half":
        v = (q - 1) // 2 + (i & 1)
    else:
        v = q - 1 - i % 7
    return np.ascontiguousarray(np.broadcast_to(v, shape)).astype(np.uint64)


EXTREME = ["max", "alt", "half", "ramp"]


@pytest.mark.parametrize("N", [1024, 16384, 32768])
def test_ntt_extreme_inputs(he, N):
    """The FP64 transforms keep unreduced values up to 4q + 8 (centred
    twiddles, he_internal.cuh): structured maximal inputs with the largest
    50-bit primes still transform exactly (forward vs the definition on
    sampled outputs; inverse round trip)."""
    primes = RINGS[N]
    ctx = ctx_for(he, N, primes)
    logN = N.bit_length() - 1
    x = np.stack([extreme_residues((len(primes), N), primes, k) for k in EXTREME])
    d = dev(x)
    ctx.ntt_forward(d)
    got = u64(d)
    rng = np.random.default_rng(7 * N)
    pos = np.unique(np.concatenate([[0, 1, 2, N // 2, N - 1], rng.integers(0, N, 24)]))
    ks = np.array([brv(int(p), logN) for p in pos], np.int32)
    for b in range(len(EXTREME)):
        for j, q in enumerate(primes):
            assert np.array_equal(got[b, j, pos], R.ntt_def(x[b, j], q, ctx.psi(j), ks))
    ctx.ntt_inverse(d)
    assert np.array_equal(u64(d), x)


@pytest.mark.parametrize("kind", EXTREME)
def test_conv_extreme_inputs(he, kind):
    """Config 4 layer 1 (s = 8, n_ib = 2) with structured maximal c0 and
    extreme filter taps (+7 / -8): the whole path (forward NTT, folded MAC,
    inverse NTT + scatter + mask) stays exact."""
    cfg = synth.CONFIGS[4]
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    Ly = cfg.conv[1]
    p = R.plan_conv(Ly, cfg.N)
    B = 2
    c0 = extreme_residues((B, p.n_ib, ring.L, cfg.N), ring.primes, kind)
    W = np.where(np.arange(Ly.c_o * Ly.c_i * Ly.f_w * Ly.f_h) % 3 == 0, -8, 7)
    W = W.reshape(Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h).astype(np.int32)
    run_conv(he, ctx, ring, Ly, B, seed=5, c0=c0, W=W)


# -------------------------------------------------------------- conv path
def run_conv(he, ctx, ring, Ly, B, seed, mask=True, s_override=0,
             ve=False, check_b=None, c0=None, W=None):
    """GPU: pack_input -> pack_filters -> conv -> mask_extract; oracle: the
    same on the sampled images (c0 / W: fixed inputs instead of the seeded
    ones).  Returns the plan."""
    N = ring.N
    plan_o = R.plan_conv(Ly, N, s_override)
    p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride,
                 Ly.pad, s_override)
    assert (p.s, p.c_ib, p.n_ib, p.c_ob, p.n_ob, p.w_o, p.h_o, p.n_valid) == \
        (plan_o.s, plan_o.c_ib, plan_o.n_ib, plan_o.c_ob, plan_o.n_ob,
         plan_o.w_o, plan_o.h_o, plan_o.n_valid)
    rng = np.random.default_rng(seed)
    if W is None:
        W = rng.integers(-8, 8, (Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h)).astype(np.int32)
    if c0 is None:
        c0 = synth.uniform_residues((B, p.n_ib, ring.L, N), ring.primes, seed)
    phi = synth.phi1((B, p.n_ob, N), ring.t, seed) if mask else None
    fspec = ctx.pack_filters(p, dev(W))
    d_c0, d_phi = dev(c0), (dev(phi) if mask else None)
    out = ctx.conv(p, d_c0, fspec, d_phi)
    comp = ctx.mask_extract(p, out)
    # fused payload (he_conv_ex): full + compact, and compact only
    comp2 = ctx.empty_u64(B, p.n_ob, ring.L, p.n_valid)
    out2 = ctx.conv(p, d_c0, fspec, d_phi, compact=comp2)
    comp3 = ctx.empty_u64(B, p.n_ob, ring.L, p.n_valid)
    ctx.conv(p, d_c0, fspec, d_phi, compact=comp3, full=False)
    torch.cuda.synchronize()
    g_out, g_comp = u64(out), u64(comp)
    bs = list(range(B)) if check_b is None else check_b
    ref = R.conv_server(c0[bs], W, plan_o, ring,
                        phi[bs] if mask else None)
    ref_c = R.compact(ref, plan_o)
    assert np.array_equal(g_out[bs], ref)
    assert np.array_equal(g_comp[bs], ref_c)
    assert np.array_equal(u64(out2)[bs], ref)
    assert np.array_equal(u64(comp2)[bs], ref_c)
    assert np.array_equal(u64(comp3)[bs], ref_c)
    return p


SMALL = [
    (synth.ConvLayer(1, 2, 4, 4), 256, 0, 3),
    (synth.ConvLayer(3, 4, 4, 4), 256, 0, 2),
    (synth.ConvLayer(4, 4, 4, 4, stride=2), 256, 0, 5),
    (synth.ConvLayer(8, 2, 3, 3), 256, 0, 1),
    (synth.ConvLayer(8, 8, 4, 4, stride=2), 256, 0, 17),
    (synth.ConvLayer(4, 2, 2, 2, f_w=2, f_h=1, pad=0), 256, 4, 2),
    (synth.ConvLayer(2, 3, 5, 3, f_w=3, f_h=1), 1024, 0, 33),
    (synth.ConvLayer(5, 7, 6, 5), 1024, 0, 19),
    (synth.ConvLayer(40, 70, 4, 4), 1024, 0, 35),   # n_ib = 3, n_ob = 5
    (synth.ConvLayer(16, 16, 6, 6), 1024, 16, 7),   # s_override
    (synth.ConvLayer(3, 5, 14, 14, f_w=5, f_h=5), 1024, 0, 9),  # fills ring
    # one K4 chunk wider than the 256-thread CTA (s >= 512)
    (synth.ConvLayer(4, 4, 2, 2, f_w=2, f_h=2, pad=0), 16384, 0, 3),   # s = 4096
    (synth.ConvLayer(64, 64, 8, 8, pad=0), 32768, 0, 2),                # s = 512
]


@pytest.mark.parametrize("case", SMALL, ids=lambda c: f"{c[0]}-N{c[1]}")
@pytest.mark.parametrize("mask", [True, False])
def test_conv_small(he, case, mask):
    Ly, N, so, B = case
    primes = RINGS[N]
    ctx = ctx_for(he, N, primes)
    ring = R.Ring(N, primes, 65537)
    run_conv(he, ctx, ring, Ly, B, seed=B * 7 + N, mask=mask, s_override=so)


@pytest.mark.parametrize("cfg_idx", [1, 2, 3])
def test_conv_configs_full(he, cfg_idx):
    cfg = synth.CONFIGS[cfg_idx]
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    run_conv(he, ctx, ring, cfg.conv[0], cfg.B, seed=cfg.seed)


def _distinct_layers(cfg):
    seen, out = set(), []
    for i, Ly in enumerate(cfg.conv):
        if Ly not in seen:
            seen.add(Ly)
            out.append((i, Ly))
    return out


@pytest.mark.parametrize("li", [i for i, _ in _distinct_layers(synth.CONFIGS[4])])
def test_conv_config4_layers(he, li):
    """Config 4 at the bench batch (B = 32): every image, every limb."""
    cfg = synth.CONFIGS[4]
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    run_conv(he, ctx, ring, cfg.conv[li], cfg.B, seed=cfg.seed + li)


def test_conv_config5_full(he):
    """Config 5 (N = 32768, L = 12, B = 256): every image, every limb."""
    cfg = synth.CONFIGS[5]
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    run_conv(he, ctx, ring, cfg.conv[0], cfg.B, seed=cfg.seed)


def test_conv_config5_paper_literal_s(he):
    """Config 5 with s = c_i = 64 (the paper's own layout)."""
    cfg = synth.CONFIGS[5]
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    run_conv(he, ctx, ring, cfg.conv[0], 8, seed=5, s_override=64,
             check_b=[0, 7])


# ------------------------------------------------------------ packing a1
@pytest.mark.parametrize("cfg_idx", [1, 2, 3, 4])
def test_pack_input(he, cfg_idx):
    cfg = synth.CONFIGS[cfg_idx]
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    Ly = cfg.conv[-1]
    plan = R.plan_conv(Ly, cfg.N)
    p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride,
                 Ly.pad)
    B = 2
    img = synth.images(cfg, len(cfg.conv) - 1, B)
    ve = synth.uniform_residues((B, p.n_ib, ring.L, cfg.N), cfg.primes, 4, "ve")
    got = u64(ctx.pack_input(p, dev(img)))
    got_ve = u64(ctx.pack_input(p, dev(img), ve=dev(ve)))
    for b in range(B):
        ip = R.pack_input_int(img[b], plan)
        for beta in range(plan.n_ib):
            enc = R.encode(np.mod(ip[beta], cfg.t).astype(np.uint32), ring)
            assert np.array_equal(got[b, beta], enc)
            want = (enc.astype(object) + ve[b, beta].astype(object)) % \
                ring.q_arr.astype(object)[:, None]
            assert np.array_equal(got_ve[b, beta], want.astype(np.uint64))


def test_protocol_config1_gpu_server(he):
    """Client (oracle) -> GPU server -> client decrypt == conv mod t."""
    cfg = synth.CONFIGS[1]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    Ly = cfg.conv[0]
    plan = R.plan_conv(Ly, cfg.N)
    p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i)
    s_key = synth.secret_key(cfg.N, cfg.h, cfg.seed)
    a = synth.uniform_residues((1, cfg.N), cfg.primes, cfg.seed, "a")
    b_pk = R.keygen(ring, s_key, a, synth.gauss_poly(cfg.N, 3.2, cfg.seed, "e0", 9))
    img = synth.images(cfg, 0)
    W = synth.weights(cfg, 0)
    v = synth.v_poly(cfg.N, cfg.seed, 0, 0)
    e0 = synth.gauss_poly(cfg.N, 3.2, cfg.seed, "e0", 0, 0)
    # c0 = v b + e0 + enc(i): the GPU packs/encodes i and adds v b + e0
    vbe = R.encrypt_c0(ring, np.zeros(cfg.N, np.int64), b_pk, v, e0)
    c0 = ctx.pack_input(p, dev(img), ve=dev(vbe[None, None]))
    assert np.array_equal(u64(c0)[0, 0], R.encrypt_c0(
        ring, R.pack_input_int(img[0], plan)[0], b_pk, v, e0))
    phi = synth.phi1((1, p.n_ob, cfg.N), cfg.t, cfg.seed)
    out = ctx.conv(p, c0, ctx.pack_filters(p, dev(W)), dev(phi))
    ef = {(n, 0): synth.gauss_poly(cfg.N, 3.2, cfg.seed, "ef", n, 0)
          for n in range(Ly.c_o)}
    dec = R.conv_protocol_decrypt(ring, plan, W, u64(out)[0], s_key, a, [v],
                                  ef, phi[0])
    assert np.array_equal(dec, R.centered_mod_t(R.conv2d_ref(img[0], W, plan),
                                                cfg.t))


# ----------------------------------------------------------------- FC a9
@pytest.mark.parametrize("N,n_i,n_o,B", [(256, 6, 5, 3), (1024, 10, 100, 2),
                                         (16384, 64, 100, 32),
                                         # sub-matrix tiling (R27): n_i n_o > N
                                         (256, 20, 30, 3), (256, 300, 5, 2),
                                         (1024, 512, 100, 2), (16384, 512, 1000, 4),
                                         # N = 32768 (2-CTA cluster inverse)
                                         (32768, 64, 100, 3), (32768, 1024, 100, 2)])
@pytest.mark.parametrize("ntt", ["", "int"])
def test_fc(he, N, n_i, n_o, B, ntt, monkeypatch):
    if ntt:
        monkeypatch.setenv("HE_NTT", ntt)
    primes = {16384: synth.PRIMES_N16384[:3],
              32768: synth.PRIMES_N32768[:3]}.get(N, RINGS[N])
    ctx = he.Context(primes, N.bit_length() - 1, 65537) if ntt else ctx_for(he, N, primes)
    ring = R.Ring(N, tuple(primes), 65537)
    fp = R.plan_fc(n_i, n_o, N)
    assert ctx.fc_plan(n_i, n_o) == (fp.n_it, fp.n_ib, fp.n_ot, fp.n_t)
    rng = np.random.default_rng(N + n_o)
    W = rng.integers(-8, 8, (n_o, n_i)).astype(np.int32)
    bias = rng.integers(-8, 8, n_o).astype(np.int32)
    inp = rng.integers(0, 256, (B, n_i)).astype(np.int32)
    c0 = synth.uniform_residues((B, fp.n_ib, ring.L, N), primes, N)
    phi = synth.phi1((B, n_o), 65537, N)
    wspec, benc = ctx.fc_pack_weights(dev(W), dev(bias))
    out = u64(ctx.fc(n_i, n_o, dev(c0), wspec, benc, dev(phi)))
    bs = [0, B - 1]
    assert np.array_equal(out[bs], R.fc_server_tiled(c0[bs], W, bias, ring, phi[bs]))
    # packed input: enc(Eq. 9) per input block
    pk = u64(ctx.fc_pack_input(n_i, n_o, dev(inp)))
    for b in bs:
        blocks = R.fc_input_blocks(inp[b], fp)
        for beta in range(fp.n_ib):
            enc = R.encode(np.mod(blocks[beta], 65537).astype(np.uint32), ring)
            assert np.array_equal(pk[b, beta], enc)


# --------------------------------------------------------------- errors
def test_errors(he):
    with pytest.raises(he.HeError) as e:
        he.Context([7681, 7681], 8)
    assert e.value.status == he.HE_EPARAM
    with pytest.raises(he.HeError):
        he.Context([7683], 8)                      # not prime
    with pytest.raises(he.HeError):
        he.Context([(1 << 50) + 1], 8)
    ctx = ctx_for(he, 256, RINGS[256])
    with pytest.raises(he.HeError) as e:
        ctx.plan(1, 1, 17, 17)                     # 19*19 > 256
    assert e.value.status == he.HE_ESHAPE
    with pytest.raises(he.HeError):
        ctx.plan(1, 1, 4, 4, s_override=3)
    p = ctx.plan(2, 2, 4, 4)
    c0 = ctx.empty_u64(2, p.n_ib, 3, 256)
    fspec = ctx.pack_filters(p, torch.zeros(2, 2, 3, 3, dtype=torch.int32,
                                            device="cuda"))
    small_ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(he.HeError) as e:
        ctx.conv(p, c0, fspec, ws=small_ws)
    assert e.value.status == he.HE_ENOMEM
    # B = 0 is a no-op
    ctx.conv(p, ctx.empty_u64(0, p.n_ib, 3, 256), fspec)


def test_conv_imad_mac_path(he, monkeypatch):
    """HE_MAC=imad selects the IMAD (25-bit split) MAC kernel instead of the
    int8 tensor-core MAC; both must be bit-exact."""
    monkeypatch.setenv("HE_MAC", "imad")
    for cfg_idx, li, B in [(3, 0, 64), (4, 1, 32), (4, 14, 32)]:
        cfg = synth.CONFIGS[cfg_idx]
        ctx = he.Context(cfg.primes, cfg.log2N, cfg.t)      # fresh: reads HE_MAC
        ring = R.Ring(cfg.N, cfg.primes, cfg.t)
        run_conv(he, ctx, ring, cfg.conv[li], B, seed=cfg.seed + 7 * li,
                 check_b=[0, B - 1])


# ------------------------------------------------------------ wire format
def _pack50_ref(x: np.ndarray) -> np.ndarray:
    """Bit-level definition of the 50-bit little-endian wire stream."""
    acc, nbits, out = 0, 0, bytearray()
    for v in x.tolist():
        acc |= int(v) << nbits
        nbits += 50
        while nbits >= 8:
            out.append(acc & 0xFF)
            acc >>= 8
            nbits -= 8
    assert nbits == 0
    return np.frombuffer(bytes(out), dtype=np.uint8)


@pytest.mark.parametrize("n", [32, 4096, 4096 + 96, 3 * 4096 + 32])
def test_pack50_roundtrip_and_layout(he, n):
    ctx = ctx_for(he, 256, RINGS[256])
    rng = np.random.default_rng(n)
    x = rng.integers(0, 2 ** 50, n, dtype=np.uint64)
    pk = ctx.pack50(dev(x))
    got = pk.cpu().numpy()
    assert got.size == n * 50 // 8
    if n <= 4096 + 96:
        assert np.array_equal(got, _pack50_ref(x))
    back = torch.empty(n, dtype=torch.int64, device="cuda")
    ctx.unpack50(pk, back)
    assert np.array_equal(u64(back), x)


def test_phi1_generate_matches_oracle(he):
    ctx = ctx_for(he, 256, RINGS[256])
    for seed, n in [(0, 1000), (2 ** 63 + 7, 65536 + 3)]:
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        ctx.phi1_generate(seed, out)
        assert np.array_equal(out.cpu().numpy().view(np.uint32),
                              R.phi1_stream(seed, n, 65537))


def test_integer_transform_path(he, monkeypatch):
    """HE_NTT=int selects the integer (Shoup) transforms instead of the FP64
    ones; both must be bit-exact (conv, FC, NTT round trip)."""
    monkeypatch.setenv("HE_NTT", "int")
    cfg = synth.CONFIGS[4]
    ctx = he.Context(cfg.primes, cfg.log2N, cfg.t)
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    for li in (1, 14):
        run_conv(he, ctx, ring, cfg.conv[li], cfg.B, seed=cfg.seed + 11 * li,
                 check_b=[0, cfg.B - 1])
    x = synth.uniform_residues((2, cfg.L, cfg.N), cfg.primes, 3, "misc")
    d = dev(x)
    ctx.ntt_forward(d)
    ctx.ntt_inverse(d)
    assert np.array_equal(u64(d), x)
    cfg5 = synth.CONFIGS[5]
    ctx5 = he.Context(cfg5.primes, cfg5.log2N, cfg5.t)
    run_conv(he, ctx5, R.Ring(cfg5.N, cfg5.primes, cfg5.t), cfg5.conv[0], 32,
             seed=9, check_b=[0, 31])


@pytest.mark.parametrize("N", [256, 1024, 16384, 32768])
def test_ntt_forward_partial_matches_definition(he, N):
    """The incomplete forward transform the conv fold runs
    against the oracle's definition: blocks of 2^skip outputs = a mod
    (X^{2^skip} - zeta_g).  Sampled blocks for large N."""
    primes = RINGS[N]
    ctx = ctx_for(he, N, primes)
    logN = N.bit_length() - 1
    x = synth.uniform_residues((2, len(primes), N), primes, 4, "misc", N)
    skips = range(logN + 1) if N <= 1024 else (1, 3, 5, 7, logN)
    for skip in skips:
        d = dev(x)
        ctx.ntt_forward_partial(d, skip)
        got = u64(d)
        s = 1 << skip
        M = N // s
        gs = range(M) if N <= 1024 else sorted(g for g in {0, 1, M - 1, M // 2 + 1} if g < M)
        for j, q in enumerate(primes):
            psi = ctx.psi(j)
            T = M.bit_length() - 1
            for g in gs:
                b = int(format(g, f"0{T}b")[::-1], 2) if T else 0
                want = R.reduce_mod_binomial(x[1, j], s, pow(psi, s * (2 * b + 1), q), q)
                assert np.array_equal(got[1, j, g * s:(g + 1) * s], want), (skip, j, g)


def test_conv_cluster_ntt_path_for_large_s(he, monkeypatch):
    """HE_NTT_COLS=0 keeps the 4-CTA cluster forward NTT for s >= 256 (config
    5) instead of the column-tiled incomplete transform; both bit-exact."""
    monkeypatch.setenv("HE_NTT_COLS", "0")
    cfg = synth.CONFIGS[5]
    ctx = he.Context(cfg.primes, cfg.log2N, cfg.t)
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    run_conv(he, ctx, ring, cfg.conv[0], 16, seed=cfg.seed + 3, check_b=[0, 15])


@pytest.mark.parametrize("t", [3, 257, (1 << 21) + 7, 4294967291])
def test_conv_and_fc_other_plaintext_moduli(he, t):
    """The mask encoding enc_j(phi1) for t other than 65537: tables for
    t <= 2^20, the arithmetic enc_plain path above (t up to 2^32 - 5)."""
    N = 1024
    primes = RINGS[N]
    ring = R.Ring(N, primes, t)
    ctx = ctx_for(he, N, primes, t)
    run_conv(he, ctx, ring, synth.ConvLayer(5, 7, 6, 5), 3, seed=t % 1000, mask=True)
    rng = np.random.default_rng(t % 997)
    n_i, n_o, B = 10, 30, 2
    W = rng.integers(-8, 8, (n_o, n_i)).astype(np.int32)
    bias = rng.integers(-8, 8, n_o).astype(np.int32)
    c0 = synth.uniform_residues((B, 1, ring.L, N), primes, 7, "misc", 3)
    phi = (rng.integers(0, t, (B, n_o), dtype=np.int64)).astype(np.uint32)
    wspec, benc = ctx.fc_pack_weights(dev(W), dev(bias))
    out = u64(ctx.fc(n_i, n_o, dev(c0), wspec, benc, dev(phi)))
    assert np.array_equal(out, R.fc_server_tiled(c0, W, bias, ring, phi))


def test_conv_column_ntt_forced(he, monkeypatch):
    """HE_NTT_COLS=1 runs the column-tiled incomplete transform for every
    s >= 4 (config 4 layers 0, 1, 8, 14 and config 3); bit-exact."""
    monkeypatch.setenv("HE_NTT_COLS", "1")
    for cfg_idx, li, B in [(4, 0, 32), (4, 1, 32), (4, 8, 32), (4, 14, 32), (3, 0, 16)]:
        cfg = synth.CONFIGS[cfg_idx]
        ctx = he.Context(cfg.primes, cfg.log2N, cfg.t)
        ring = R.Ring(cfg.N, cfg.primes, cfg.t)
        run_conv(he, ctx, ring, cfg.conv[li], B, seed=cfg.seed + 11 * li, check_b=[0, B - 1])


def test_conv_in_bench_launch_configuration(he):
    """The bench step's launch configuration -- config 4 layer jobs dealt to
    six streams, the FC job last on the next stream, captured once as a CUDA
    graph and replayed -- gives bit-exact full outputs, payloads and FC
    outputs (sampled images vs the oracle)."""
    cfg = synth.CONFIGS[4]
    ctx = ctx_for(he, cfg.N, cfg.primes, cfg.t)
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    B = cfg.B
    lis = [0, 1, 7, 8, 13, 14]
    jobs = []
    for li in lis:
        Ly = cfg.conv[li]
        p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride, Ly.pad)
        W = synth.weights(cfg, li)
        c0 = synth.uniform_residues((B, p.n_ib, ring.L, cfg.N), cfg.primes, cfg.seed, "c0", li)
        phi = synth.phi1((B, p.n_ob, cfg.N), cfg.t, cfg.seed, li)
        jobs.append(dict(li=li, p=p, W=W, c0=c0, phi=phi, fspec=ctx.pack_filters(p, dev(W)),
                         c0_d=dev(c0), phi_d=dev(phi), out=ctx.empty_u64(B, p.n_ob, ring.L, cfg.N),
                         comp=ctx.empty_u64(B, p.n_ob, ring.L, p.n_valid)))
    fc = cfg.fc
    fp = R.plan_fc(fc.n_i, fc.n_o, cfg.N)
    fW, fbias = synth.fc_weights(cfg), synth.fc_bias(cfg)
    fc0 = synth.uniform_residues((B, fp.n_ib, ring.L, cfg.N), cfg.primes, cfg.seed, "c0", 99)
    fphi = synth.phi1((B, fc.n_o), cfg.t, cfg.seed, 99)
    fwspec, fbenc = ctx.fc_pack_weights(dev(fW), dev(fbias))
    fjob = dict(c0_d=dev(fc0), phi_d=dev(fphi), out=ctx.empty_u64(B, ring.L, fc.n_o),
                ws=ctx.fc_workspace(fc.n_i, fc.n_o, B))
    nstr = 6
    main = torch.cuda.Stream()
    side = [main] + [torch.cuda.Stream() for _ in range(nstr - 1)]
    ws = [ctx.conv_workspace(j["p"], B) for j in jobs]
    wsk = [torch.empty(max(w.numel() for w in ws), dtype=torch.uint8, device="cuda")
           for _ in range(nstr)]
    fork = [torch.cuda.Event() for _ in range(nstr)]

    def step():
        fork[0].record(main)
        for k in range(1, nstr):
            side[k].wait_event(fork[0])
        for i, j in enumerate(jobs):
            k = i % nstr
            ctx.conv(j["p"], j["c0_d"], j["fspec"], j["phi_d"], j["out"], wsk[k],
                     compact=j["comp"], stream=side[k])
        ctx.fc(fc.n_i, fc.n_o, fjob["c0_d"], fwspec, fbenc, fjob["phi_d"], fjob["out"],
               fjob["ws"], stream=side[len(jobs) % nstr])
        for k in range(1, nstr):
            fork[k].record(side[k])
            main.wait_event(fork[k])

    torch.cuda.synchronize()
    with torch.cuda.stream(main):
        step()                                   # warm-up outside capture
    torch.cuda.synchronize()
    for j in jobs:
        j["out"].zero_()
        j["comp"].zero_()
    fjob["out"].zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        step()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for j in jobs:                          # every image of every job
        plan = R.plan_conv(cfg.conv[j["li"]], cfg.N)
        ref = R.conv_server(j["c0"], j["W"], plan, ring, j["phi"])
        assert np.array_equal(u64(j["out"]), ref), j["li"]
        assert np.array_equal(u64(j["comp"]), R.compact(ref, plan)), j["li"]
    assert np.array_equal(u64(fjob["out"]),
                          R.fc_server_tiled(fc0, fW, fbias, ring, fphi))


@pytest.mark.parametrize("case", SMALL + [
    (synth.ConvLayer(16, 24, 5, 5), 1024, 0, 130),        # two 128-image tiles, ragged
    (synth.ConvLayer(64, 64, 8, 8), 8192, 0, 129),         # K = 64, c_o = 64
    # TMA-staged operands (B % 8 == 0, K a multiple of 32, c_o % 8 == 0):
    (synth.ConvLayer(64, 64, 8, 8), 8192, 0, 136),         # second tile: 8 images
    (synth.ConvLayer(32, 40, 8, 8), 8192, 0, 16)],         # c_o = 40: 8 zero channel rows
    ids=lambda c: f"{c[0]}-N{c[1]}-B{c[3]}")
def test_conv_tcgen05_mac_path(he, case, monkeypatch):
    """The tcgen05 MAC (k_mac_tc, the default for >= 128 images) forced on
    every shape, including batches below one 128-image tile."""
    monkeypatch.setenv("HE_MAC_TC", "1")
    Ly, N, so, B = case
    ring = R.Ring(N, RINGS[N] if N in RINGS else synth.PRIMES_N8192[:2], 65537)
    ctx = he.Context(ring.primes, N.bit_length() - 1, 65537)   # fresh: reads HE_MAC_TC
    check = list(range(B)) if B <= 8 else [0, 1, B // 2, B - 2, B - 1]
    run_conv(he, ctx, ring, Ly, B, seed=B + N, s_override=so, check_b=check)


@pytest.mark.parametrize("B", [20, 32, 45])
def test_conv_k16_mac_tma_path(he, B):
    """The K = 16 int8 MAC instance (16 channels, four groups per CTA, 32-image
    tiles) with its operands staged by TMA tensor copies: a ragged last tile
    (images past B arrive as TMA out-of-bounds zeros), every image checked."""
    N = 8192
    primes = synth.PRIMES_N8192[:2]
    ctx = he.Context(primes, N.bit_length() - 1, 65537)
    ring = R.Ring(N, tuple(primes), 65537)
    run_conv(he, ctx, ring, synth.ConvLayer(8, 16, 16, 16), B, seed=B + 16)


def test_conv_wide_layer_over_256_channels(he):
    """c_o > 256: the IMAD MAC path (the tensor-core kernel keeps all of a
    group's output channels in one CTA); n_ob > 1 blocks, bit-exact."""
    N = 1024
    primes = RINGS[N]
    ctx = ctx_for(he, N, primes)
    ring = R.Ring(N, primes, 65537)
    run_conv(he, ctx, ring, synth.ConvLayer(8, 300, 4, 4), 3, seed=300, mask=True)


@pytest.mark.parametrize("case", SMALL[:6], ids=lambda c: f"{c[0]}-N{c[1]}")
def test_filter_coefficients_eq6_eq7(he, case):
    """a2 directly: the coefficient-domain filter polynomials of Eq. (6) and
    the Eq. (7)-shifted ones against the oracle's sparse term lists."""
    Ly, N, so, _ = case
    primes = RINGS[N]
    ctx = ctx_for(he, N, primes)
    ring = R.Ring(N, primes, 65537)
    plan = R.plan_conv(Ly, N, so)
    p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride, Ly.pad, so)
    W = np.random.default_rng(N + Ly.c_o).integers(-8, 8, (Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h))
    for shifted in (False, True):
        got = u64(ctx.filter_coeffs(p, dev(W.astype(np.int32)), shifted))
        for n in range(plan.c_o):
            for beta in range(plan.n_ib):
                want = np.zeros(N, dtype=np.int64)
                for e, w in R.filter_terms(W, plan, n, beta, shifted=shifted):
                    want[e] += w
                assert np.array_equal(got[n, beta], R.signed_to_residues(want, ring)), \
                    (shifted, n, beta)


@pytest.mark.parametrize("case", SMALL[3:8], ids=lambda c: f"{c[0]}-N{c[1]}")
def test_conv_plain_unfolded_path(he, case):
    """The unfolded reference path (full N-point products and inverse, then
    extraction) equals the oracle and he_conv's folded output."""
    Ly, N, so, B = case
    primes = RINGS[N]
    ctx = ctx_for(he, N, primes)
    ring = R.Ring(N, primes, 65537)
    plan = R.plan_conv(Ly, N, so)
    p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride, Ly.pad, so)
    W = np.random.default_rng(B + N).integers(-8, 8, (Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h)).astype(np.int32)
    c0 = synth.uniform_residues((B, p.n_ib, ring.L, N), primes, 41, "misc", B)
    phi = synth.phi1((B, p.n_ob, N), ring.t, 41)
    out_p = u64(ctx.conv_plain(p, dev(c0), ctx.pack_filters_plain(p, dev(W)), dev(phi)))
    out_f = u64(ctx.conv(p, dev(c0), ctx.pack_filters(p, dev(W)), dev(phi)))
    assert np.array_equal(out_p, out_f)
    assert np.array_equal(out_p, R.conv_server(c0, W, plan, ring, phi))
