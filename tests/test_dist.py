"""Multi-rank host logic on CPU (gloo, world_size 2): batch sharding and
the payload gather reproduce the single-process result bit for bit."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_05205_b200.dist import gather_payload, shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 32, 256, 257):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # every rank "serves" its shard: a deterministic per-image payload of
    # the same shape as a compact output [b][n_ob][L][n_valid]
    full = torch.arange(total * 2 * 3 * 5, dtype=torch.int64).reshape(total, 2, 3, 5)
    lo, hi = shard_range(total, rank, world)
    got = gather_payload(full[lo:hi].clone(), total)
    q.put((rank, bool(torch.equal(got, full))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [8, 7])
def test_gather_payload_gloo_world2(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + total
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)


# ---- real shards: each rank's payload comes from the oracle's server
# definition (orc_conv_server) on its part of the work; the assembled
# payload must equal the single-process payload.
def _oracle_payload(Ly, W, c0, phi, N, primes, t=65537):
    from oracle import ref as R
    ring = R.Ring(N, primes, t)
    plan = R.plan_conv(Ly, N)
    return R.compact(R.conv_server(c0, W, plan, ring, phi), plan)


def _shard_worker(rank, world, port, case, q):
    import synth
    from oracle import ref as R
    from paper_2409_05205_b200.dist import (choose_axis, gather_blocks, gather_payload,
                                            shard_out_blocks, sub_layer_weights)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    Ly, N, primes, B = case
    plan = R.plan_conv(Ly, N)
    W = np.random.default_rng(3).integers(-8, 8, (Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h)).astype(np.int32)
    c0 = synth.uniform_residues((B, plan.n_ib, len(primes), N), primes, 11, "c0", 1)
    phi = synth.phi1((B, plan.n_ob, N), 65537, 11, 1)
    axis = choose_axis(B, plan.n_ob, world)
    if axis == "batch":
        lo, hi = shard_range(B, rank, world)
        local = _oracle_payload(Ly, W, c0[lo:hi], phi[lo:hi], N, primes)
        got = gather_payload(torch.from_numpy(local.view(np.int64)), B)
    else:
        lo, hi = shard_out_blocks(plan.n_ob, rank, world)
        import synth as S
        sub = S.ConvLayer(Ly.c_i, (hi - lo) * plan.c_ob, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h,
                          Ly.stride, Ly.pad)
        sp = R.plan_conv(sub, N)
        assert (sp.s, sp.c_ob, sp.n_valid) == (plan.s, plan.c_ob, plan.n_valid)
        Ws = sub_layer_weights(W, plan.c_ob, lo, hi)
        local = _oracle_payload(sub, Ws, c0, np.ascontiguousarray(phi[:, lo:hi]), N, primes)
        got = gather_blocks(torch.from_numpy(np.ascontiguousarray(local).view(np.int64)),
                            plan.n_ob)
    want = _oracle_payload(Ly, W, c0, phi, N, primes)
    q.put((rank, axis, bool(np.array_equal(got.numpy().view(np.uint64), want))))
    dist.barrier()
    dist.destroy_process_group()


SHARD_CASES = [
    # batch axis: config 2's layer, 3 images over 2 ranks (ragged)
    ("batch", lambda: (__import__("synth").CONFIGS[2].conv[0], 8192,
                       __import__("synth").PRIMES_N8192[:2], 3)),
    # output-block axis: config 2 itself (B = 1, n_ob = 4)
    ("out_block", lambda: (__import__("synth").CONFIGS[2].conv[0], 8192,
                           __import__("synth").PRIMES_N8192[:3], 1)),
    # output-block axis with a partial last block (c_o = 14, c_ob = 8)
    ("out_block", lambda: (__import__("synth").ConvLayer(3, 14, 8, 8), 1024,
                           __import__("oracle.ref").ref.find_primes(1024, 50, 2), 1)),
]


@pytest.mark.parametrize("case", range(len(SHARD_CASES)))
def test_sharded_oracle_payload_gloo_world2(case):
    axis_want, mk = SHARD_CASES[case]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() % 1000) + case
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, mk(), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(a == axis_want for _, a, _ in res), res
    assert all(ok for _, _, ok in res), res


def test_sub_layer_weights_blocks():
    from paper_2409_05205_b200.dist import sub_layer_weights
    W = np.arange(14 * 2 * 3 * 3).reshape(14, 2, 3, 3)
    s = sub_layer_weights(W, 8, 1, 2)           # block 1: channels 8..13, padded to 8
    assert s.shape == (8, 2, 3, 3)
    assert np.array_equal(s[:6], W[8:14]) and not s[6:].any()
    assert np.array_equal(sub_layer_weights(W, 8, 0, 2)[:14], W)
