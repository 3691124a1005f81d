"""Memory-safety checks of our own, in place of compute-sanitizer (closed on the
GPU pool: the pool refuses to run it).

Every buffer the library writes sits between two guard bands filled with a
canary word; every output and workspace is pre-filled with random garbage;
every input sits between guard bands of random garbage.  Each call runs twice
with two different garbage fills.  Checked:
* the guard bands around outputs and workspaces still hold the canary
  (no out-of-bounds write);
* the two runs give identical outputs (no result depends on unwritten
  workspace or output memory, nor on memory next to an input);
* the result equals the oracle (so the identical outputs are the right ones).
Shapes: the small parity cases, every compile-time instance shape of the
plain-20 stack (config 4 layers at B = 4), config 5's layer (tcgen05 MAC at
B = 128), FC with and without tiling, the standalone transforms.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import ref as R

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(),
                                 reason="needs a CUDA GPU")]

G = 4096                                       # guard words on each side
CANARY = 0x5A5A_A5A5_5A5A_A5A5            # < 2^63: a valid int64


@pytest.fixture(scope="module")
def he():
    import paper_2409_05205_b200 as he
    return he


class Guarded:
    """A [G | body | G] int64 device buffer; `body` is a contiguous view."""

    def __init__(self, shape, garbage_seed, guard="canary", dtype=torch.int64):
        n = int(np.prod(shape))
        g = torch.Generator(device="cpu").manual_seed(garbage_seed)
        self.n = n
        if guard == "canary":
            self.buf = torch.full((n + 2 * G,), CANARY, dtype=torch.int64)
        else:                                   # random garbage neighbours
            self.buf = torch.randint(-(1 << 62), 1 << 62, (n + 2 * G,), generator=g)
        self.buf[G:G + n] = torch.randint(-(1 << 62), 1 << 62, (n,), generator=g)
        self.buf = self.buf.cuda()
        self.body = self.buf[G:G + n].view(shape)
        if dtype != torch.int64:                # e.g. uint8 workspaces
            self.body = self.buf[G:G + n].view(dtype)

    def guards_ok(self):
        torch.cuda.synchronize()
        lo, hi = self.buf[:G].cpu(), self.buf[G + self.n:].cpu()
        return bool((lo == CANARY).all()) and bool((hi == CANARY).all())


def guarded_input(a: np.ndarray, garbage_seed):
    """Input `a` (uint64 / uint32 / int32) between random garbage bands."""
    a = np.ascontiguousarray(a)
    b = a.view(np.int64) if a.dtype == np.uint64 else a.view(np.int32)
    t = torch.from_numpy(b.copy())
    g = torch.Generator(device="cpu").manual_seed(garbage_seed)
    lo = torch.randint(-(1 << 30), 1 << 30, (G,), generator=g).to(t.dtype)
    hi = torch.randint(-(1 << 30), 1 << 30, (G,), generator=g).to(t.dtype)
    buf = torch.cat([lo, t.reshape(-1), hi]).cuda()
    return buf[G:G + t.numel()].view(t.shape)


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def ws_guarded(nbytes, seed):
    words = (nbytes + 7) // 8
    w = Guarded((words,), seed)
    return w, w.buf[G:G + words].view(torch.uint8)[:nbytes]


def conv_guarded_run(he, ctx, p, c0, fspec, phi, seed):
    B = c0.shape[0]
    out = Guarded((B, p.n_ob, ctx.L, ctx.N), seed)
    comp = Guarded((B, p.n_ob, ctx.L, p.n_valid), seed + 1)
    nb = ctx.conv_workspace(p, B).numel()
    wsg, ws = ws_guarded(nb, seed + 2)
    d_c0 = guarded_input(c0, seed + 3)
    d_phi = guarded_input(phi, seed + 4) if phi is not None else None
    ctx.conv(p, d_c0, fspec, d_phi, out=out.body, ws=ws, compact=comp.body)
    assert out.guards_ok() and comp.guards_ok() and wsg.guards_ok()
    return u64(out.body), u64(comp.body)


CONV_CASES = [
    ("small-256", synth.ConvLayer(8, 8, 4, 4, stride=2), 256, (7681, 12289, 40961), 5),
    ("small-1024-nib3", synth.ConvLayer(40, 70, 4, 4), 1024, None, 3),
    ("s4096", synth.ConvLayer(4, 4, 2, 2, f_w=2, f_h=2, pad=0), 16384, "c4", 3),
] + [(f"cfg4-layer{i}", synth.CONFIGS[4].conv[i], 16384, "c4", 4) for i in (0, 1, 7, 8, 13, 14)]


@pytest.mark.parametrize("case", CONV_CASES, ids=lambda c: c[0])
def test_conv_guard_bands(he, case):
    _, Ly, N, primes, B = case
    if primes == "c4":
        primes = synth.CONFIGS[4].primes
    elif primes is None:
        primes = tuple(synth.PRIMES_CFG1) + (R.find_primes(1024, 50, 1)[0],)
    ctx = he.Context(list(primes), N.bit_length() - 1, 65537)
    ring = R.Ring(N, tuple(primes), 65537)
    p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride, Ly.pad)
    plan_o = R.plan_conv(Ly, N)
    rng = np.random.default_rng(N + B)
    W = rng.integers(-8, 8, (Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h)).astype(np.int32)
    c0 = synth.uniform_residues((B, p.n_ib, ring.L, N), ring.primes, 11)
    phi = synth.phi1((B, p.n_ob, N), ring.t, 11)
    fspec = ctx.pack_filters(p, torch.from_numpy(W).cuda())
    o1, c1 = conv_guarded_run(he, ctx, p, c0, fspec, phi, 100)
    o2, c2 = conv_guarded_run(he, ctx, p, c0, fspec, phi, 200)
    assert np.array_equal(o1, o2) and np.array_equal(c1, c2)
    ref = R.conv_server(c0, W, plan_o, ring, phi)
    assert np.array_equal(o1, ref)
    assert np.array_equal(c1, R.compact(ref, plan_o))


def test_conv_guard_bands_tcgen05(he):
    """Config 5's layer at B = 128 (the tcgen05 MAC), two garbage fills."""
    cfg = synth.CONFIGS[5]
    Ly, B, N = cfg.conv[0], 128, cfg.N
    ctx = he.Context(list(cfg.primes), N.bit_length() - 1, cfg.t)
    ring = R.Ring(N, tuple(cfg.primes), cfg.t)
    p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride, Ly.pad)
    W = np.random.default_rng(3).integers(-8, 8, (Ly.c_o, Ly.c_i, 3, 3)).astype(np.int32)
    c0 = synth.uniform_residues((B, p.n_ib, ring.L, N), ring.primes, 12)
    phi = synth.phi1((B, p.n_ob, N), ring.t, 12)
    fspec = ctx.pack_filters(p, torch.from_numpy(W).cuda())
    o1, c1 = conv_guarded_run(he, ctx, p, c0, fspec, phi, 300)
    o2, c2 = conv_guarded_run(he, ctx, p, c0, fspec, phi, 400)
    assert np.array_equal(o1, o2) and np.array_equal(c1, c2)
    bs = [0, 77, B - 1]
    ref = R.conv_server(c0[bs], W, R.plan_conv(Ly, N), ring, phi[bs])
    assert np.array_equal(c1[bs], R.compact(ref, R.plan_conv(Ly, N)))


@pytest.mark.parametrize("N,n_i,n_o,B", [(16384, 64, 100, 4), (16384, 512, 1000, 2),
                                         (32768, 64, 100, 2)])
def test_fc_guard_bands(he, N, n_i, n_o, B):
    primes = {16384: synth.PRIMES_N16384[:3], 32768: synth.PRIMES_N32768[:3]}[N]
    ctx = he.Context(list(primes), N.bit_length() - 1, 65537)
    ring = R.Ring(N, tuple(primes), 65537)
    fp = R.plan_fc(n_i, n_o, N)
    rng = np.random.default_rng(N + n_i)
    W = rng.integers(-8, 8, (n_o, n_i)).astype(np.int32)
    bias = rng.integers(-8, 8, n_o).astype(np.int32)
    c0 = synth.uniform_residues((B, fp.n_ib, ring.L, N), primes, 13)
    phi = synth.phi1((B, n_o), 65537, 13)
    wspec, benc = ctx.fc_pack_weights(torch.from_numpy(W).cuda(),
                                      torch.from_numpy(bias).cuda())
    outs = []
    for seed in (500, 600):
        out = Guarded((B, ring.L, n_o), seed)
        wsg, ws = ws_guarded(ctx.fc_workspace(n_i, n_o, B).numel(), seed + 1)
        ctx.fc(n_i, n_o, guarded_input(c0, seed + 2), wspec, benc,
               guarded_input(phi, seed + 3), out=out.body, ws=ws)
        assert out.guards_ok() and wsg.guards_ok()
        outs.append(u64(out.body))
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], R.fc_server_tiled(c0, W, bias, ring, phi))


@pytest.mark.parametrize("N", [1024, 8192, 16384, 32768])
def test_ntt_guard_bands(he, N):
    """In-place transforms: the bands around the data keep the canary and a
    forward + inverse round trip returns the input."""
    primes = {1024: tuple(synth.PRIMES_CFG1) + (R.find_primes(1024, 50, 1)[0],),
              8192: synth.PRIMES_N8192[:2], 16384: synth.PRIMES_N16384[:2],
              32768: synth.PRIMES_N32768[:2]}[N]
    ctx = he.Context(list(primes), N.bit_length() - 1, 65537)
    x = synth.uniform_residues((3, len(primes), N), primes, N)
    d = Guarded((3, len(primes), N), 700)
    d.body.copy_(torch.from_numpy(x.view(np.int64)).cuda())
    ctx.ntt_forward(d.body)
    assert d.guards_ok()
    ctx.ntt_inverse(d.body)
    assert d.guards_ok()
    assert np.array_equal(u64(d.body), x)


def test_guard_detects_overrun():
    """Negative control: one word written past the body is seen."""
    g = Guarded((100,), 1)
    assert g.guards_ok()
    g.buf[G + 100] = 0
    assert not g.guards_ok()
    g = Guarded((100,), 2)
    g.buf[G - 1] = 0
    assert not g.guards_ok()
