#!/usr/bin/env python
"""bench.py -- throughput of the rotation-free HE Conv/FC server hot path.

Workload (default, BASELINE.json configs[3]): the full plain-20 stack
(19 Conv layers + FC 64->100), ring N = 16384, L = 6 primes of 50 bits,
B = 32 images per GPU (weak scaling: every rank serves its own batch, no
data-path collective).  One step = the server evaluation of
every layer for the batch: he_conv_ex (forward NTT of c0, folded NTT-domain
MAC, inverse NTT + slot scatter + enc(phi1) mask, full output and fused
valid-slot payload) for each Conv layer, then he_fc.  Default launch
configuration (--streams 6 --overlap layers): the 20 independent layer jobs
are dealt round-robin to six CUDA streams (layer i on stream i % 6, the FC
job on stream 19 % 6), the whole step captured once as a CUDA graph and
replayed; --overlap batch instead splits every layer's batch across the
streams.  A second, sequential pass (one launch sequence per layer, stage
events) measures every kernel for the roofline.  Inputs are seeded
synthetic residues (synth/); the per-layer filter spectra (server init,
Alg. 1 Line 4) are prepared before the timed region and timed separately.

Metric: ct x pt evals / s (one eval = one c0_beta x fhat_beta^{(n)} product
with its extraction; B*c_o*n_ib per Conv layer, B per FC) plus ms per
plain-20 image and NTT limbs / s against the roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload plain20|cfg5|cfg3]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK_GBS = 6650.0           # B200_PROFILING.md fallback
# FP64 operations of one exact modular butterfly (dp_mulmod: DMUL + 3 DFMA +
# 2 DADD, plus the add and subtract): the DFMA-pipe roof is DFMA/s / 8
DP_OPS_PER_BFLY = 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["plain20", "cfg5", "cfg3", "cfg2"],
                    default="plain20")
    ap.add_argument("--scaling", choices=["auto", "weak", "strong"], default="auto",
                    help="weak: every rank serves the config's own batch (plain20 and "
                         "cfg3 default); strong: one global batch split over the ranks "
                         "by image, or by output-channel block when it has fewer "
                         "images than ranks (cfg5 and cfg2 default)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the client / chain / ablation / FC-variant sections")
    ap.add_argument("--streams", type=int, default=6,
                    help="split every layer's image batch into this many "
                         "sub-batches, each on its own CUDA stream (1 = one launch "
                         "sequence per layer)")
    ap.add_argument("--overlap", choices=["batch", "layers"], default="layers",
                    help="with --streams > 1: split each layer's batch across the "
                         "streams (batch) or put whole layers on alternating streams "
                         "(layers: independent layer jobs overlap)")
    ap.add_argument("--schedule", choices=["lpt", "rr"], default="rr",
                    help="--overlap layers: deal the layer jobs (and the FC job) to "
                         "the streams longest-first onto the least-loaded stream, by "
                         "their measured stand-alone times (lpt), or round-robin (rr; "
                         "default -- lpt measured equal, 1.6995 vs 1.697 ms: the step "
                         "is throughput-limited, not tail-limited)")
    ap.add_argument("--graph", type=int, default=1,
                    help="1: replay the step as a captured CUDA graph")
    ap.add_argument("--payload-only", type=int, default=0,
                    help="1: the step writes only the masked valid-slot payload "
                         "(he_conv_ex with d_out = NULL), not the full c0^r")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-client", action="store_true",
                    help="skip the client mirror-path measurement")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no e2e / cpu baseline / clocks")
    return ap.parse_args()


WORKLOADS = {"plain20": 4, "cfg5": 5, "cfg3": 3, "cfg2": 2}
DEFAULT_SCALING = {"plain20": "weak", "cfg3": "weak", "cfg5": "strong", "cfg2": "strong"}


def self_launch(args) -> int:
    """--gpus N > 1 without a torchrun environment: re-run this command under
    torch.distributed.run with one rank per GPU (127.0.0.1 rendezvous); rank 0
    prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def peaks():
    try:
        d = json.load(open(MEASURED))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------- workload def
class LayerWork:
    def __init__(self, idx, Ly, plan, N, L, B):
        self.idx, self.Ly, self.p = idx, Ly, plan
        M = N // plan.s
        ku = plan.k_u                      # fold-group columns the MAC uses
        nlimb = B * plan.n_ib * L
        self.evals = B * Ly.c_o * plan.n_ib
        # the fold runs the incomplete transform, log2(N/s) stages, and needs
        # only the k_u columns of each group
        self.ntt_bfly = nlimb * ku * (M // 2) * (M.bit_length() - 1)
        self.ntt_bytes = nlimb * M * ku * 16
        self.macs = L * M * plan.n_ib * ku * B * Ly.c_o
        self.mac_bytes = 8 * (nlimb * M * ku + Ly.c_o * plan.n_ib * ku * L * M +
                              L * M * B * Ly.c_o)
        logM = M.bit_length() - 1
        self.intt_bfly = B * plan.n_ob * plan.c_ob * L * (M // 2) * logM
        self.intt_bytes = 8 * (L * M * B * Ly.c_o + B * plan.n_ob * L * N) + \
            4 * B * plan.n_ob * N
        self.c0_bytes = nlimb * N * 8
        self.comp_bytes = B * plan.n_ob * L * plan.n_valid * 8
        self.phi_bytes = B * plan.n_ob * N * 4


def u1_peaks(device_index=0):
    """Run the U1 register-resident microbenchmarks (libhe_u1.so) on this
    GPU: rates per second (whole GPU, CUDA-event timed) and the implied rate
    per clock per SM at the GPU's maximum SM clock."""
    import ctypes
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2409_05205_b200",
                                   "libhe_u1.so"))
    lib.u1_run.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p] * 3
    out = {}
    import torch
    nsm = torch.cuda.get_device_properties(device_index).multi_processor_count
    try:
        max_mhz = float(subprocess.run(
            ["nvidia-smi", "--query-gpu=clocks.max.sm", "--format=csv,noheader,nounits",
             "-i", str(device_index)], capture_output=True, text=True,
            timeout=20).stdout.strip().splitlines()[0])
    except Exception:
        max_mhz = 1965.0
    names = ["imad", "imad_wide", "modmac", "ct_bfly", "gs_bfly", "imma_u8",
             "dfma", "dp_ct_bfly", "dp_gs_bfly",
             # tcgen05.mma kind::i8 (int8 MAC/s), one issuing thread per SM
             "tc_i8_m128n16", "tc_i8_m128n32", "tc_i8_m128n64"]
    iters = {0: 20000, 1: 20000, 2: 20000, 3: 2000, 4: 2000, 5: 2000, 6: 20000,
             7: 2000, 8: 2000, 9: 4000, 10: 4000, 11: 4000}
    for w, name in enumerate(names):
        ms, cyc, ops = ctypes.c_float(), ctypes.c_longlong(), ctypes.c_double()
        blocks, threads = (nsm, 128) if w >= 9 else (148 * 8, 256)
        rc = lib.u1_run(w, blocks, threads, iters[w], ctypes.byref(ms),
                        ctypes.byref(cyc), ctypes.byref(ops))
        if rc:
            raise RuntimeError(f"u1 {name} rc={rc}")
        rate = ops.value / (ms.value * 1e-3)
        out[name] = {"per_s": rate,
                     "per_clk_per_sm_at_max_clock": rate / (max_mhz * 1e6) / nsm}
    return out


class ClockSampler:
    def __init__(self, idx):
        self.idx = idx
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for r in self.rows:
            for n, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_single_thread(cfg_idx: int, max_s: float = 20.0) -> None:
    """cpu_baseline leg (child process, OMP_NUM_THREADS=1): the oracle's server
    work for ONE image through every layer of the config, repeated up to
    max_s; prints one JSON object."""
    from oracle import ref as R
    cfg = synth.CONFIGS[cfg_idx]
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    plans = [R.plan_conv(Ly, cfg.N) for Ly in cfg.conv]
    Ws = [synth.weights(cfg, i) for i in range(len(cfg.conv))]
    c0s = [synth.uniform_residues((1, p.n_ib, ring.L, cfg.N), cfg.primes, cfg.seed, "c0", i)
           for i, p in enumerate(plans)]
    phis = [synth.phi1((1, p.n_ob, cfg.N), cfg.t, cfg.seed, i) for i, p in enumerate(plans)]
    fc = cfg.fc
    evals = sum(Ly.c_o * p.n_ib for Ly, p in zip(cfg.conv, plans)) + (1 if fc else 0)
    t0, reps = time.perf_counter(), 0
    while True:
        for p, W, c0, ph in zip(plans, Ws, c0s, phis):
            R.compact(R.conv_server(c0, W, p, ring, ph), p)
        if fc:
            R.fc_server(synth.uniform_residues((1, ring.L, cfg.N), cfg.primes, cfg.seed, "c0", 99),
                        synth.fc_weights(cfg), synth.fc_bias(cfg), ring,
                        synth.phi1((1, fc.n_o), cfg.t, cfg.seed, 99))
        reps += 1
        if time.perf_counter() - t0 > max_s or reps >= 4:
            break
    dt = time.perf_counter() - t0
    res = {"value": reps * evals / dt, "unit": "ct×pt evals/s", "cores": 1,
           "s_per_image": dt / reps, "cpu_model": cpu_model(),
           "sample": f"{reps} x 1 image x all {len(plans)} conv"
                     f"{' + FC' if fc else ''} layers ({dt:.1f} s wall, OMP_NUM_THREADS=1)"}
    # the CPU textbook-NTT path on one thread, conv layers only
    from oracle import cpu_baseline as CB
    fsp = [CB.prepare_filters(W, p, ring) for W, p in zip(Ws, plans)]
    t0, reps = time.perf_counter(), 0
    while True:
        for p, f, c0, ph in zip(plans, fsp, c0s, phis):
            R.compact(CB.conv_server(c0, f, p, ring, ph), p)
        reps += 1
        if time.perf_counter() - t0 > max_s or reps >= 4:
            break
    dtn = time.perf_counter() - t0
    evc = sum(Ly.c_o * p.n_ib for Ly, p in zip(cfg.conv, plans))
    res["ntt_path"] = {"value": reps * evc / dtn, "unit": "ct×pt evals/s", "cores": 1,
                       "s_per_image_conv_layers": dtn / reps,
                       "sample": f"{reps} x 1 image x all {len(plans)} conv layers "
                                 f"({dtn:.1f} s wall, OMP_NUM_THREADS=1)"}
    print(json.dumps(res))


# ------------------------------------------------------------ reference
def run_reference(args, cfg, rank):
    """--impl reference: the CPU oracle as it stands (test infrastructure),
    rank 0 only, one image through the whole stack per step."""
    if rank != 0:
        return
    from oracle import ref as R
    ring = R.Ring(cfg.N, cfg.primes, cfg.t)
    plans = [R.plan_conv(Ly, cfg.N) for Ly in cfg.conv]
    Ws = [synth.weights(cfg, i) for i in range(len(cfg.conv))]
    c0s = [synth.uniform_residues((1, p.n_ib, ring.L, cfg.N), cfg.primes,
                                  cfg.seed, "c0", i) for i, p in enumerate(plans)]
    phis = [synth.phi1((1, p.n_ob, cfg.N), cfg.t, cfg.seed, i)
            for i, p in enumerate(plans)]
    fc = None
    if cfg.fc is not None:
        fc = (synth.fc_weights(cfg), synth.fc_bias(cfg),
              synth.uniform_residues((1, ring.L, cfg.N), cfg.primes, cfg.seed,
                                     "c0", 99),
              synth.phi1((1, cfg.fc.n_o), cfg.t, cfg.seed, 99))
    evals = sum(Ly.c_o * p.n_ib for Ly, p in zip(cfg.conv, plans)) + \
        (1 if fc else 0)

    def step():
        for p, W, c0, ph in zip(plans, Ws, c0s, phis):
            R.compact(R.conv_server(c0, W, p, ring, ph), p)
        if fc:
            R.fc_server(fc[2], fc[0], fc[1], ring, fc[3])

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    v = evals / dt
    line = {"metric": "Conv+FC layer ct×pt evals/sec", "value": v,
            "unit": "ct×pt evals/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic",
            "config": {"workload": f"cfg{cfg.idx} {cfg.name}", "N": cfg.N,
                       "L": cfg.L, "images_per_step": 1},
            "ms_per_plain20_image": dt * 1e3,
            "cpu_baseline": {"value": v, "unit": "ct×pt evals/s",
                             "cores": os.cpu_count(), "kind": "oracle",
                             "sample": f"1 image x {len(plans)} conv"
                                       f"{' + FC' if fc else ''} layers per step"},
            "e2e": {"value": v, "unit": "ct×pt evals/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours
def main():
    args = parse()
    cfg = synth.CONFIGS[WORKLOADS[args.workload]]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, cfg, rank)
    scaling = DEFAULT_SCALING[args.workload] if args.scaling == "auto" else args.scaling
    if args.profile:
        args.streams = 1            # profiling runs: one launch sequence per layer

    import torch
    import torch.distributed as dist
    import paper_2409_05205_b200 as he

    # HE_BENCH_GLOO_CHECK=1 (host-logic check only, never a measurement):
    # every rank on cuda:0 with gloo collectives on host copies, so the
    # multi-rank partition / gather / timing code runs on a one-GPU box
    gloo_check = os.environ.get("HE_BENCH_GLOO_CHECK") == "1"
    if gloo_check:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if gloo_check:
            dist.init_process_group("gloo")
        else:
            # NCCL's init log (rank, nRanks) is the evidence of the communicator
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier(device_ids=[local])
        print(f"[bench] rank {rank}/{world} on cuda:{local}, backend "
              f"{dist.get_backend()}", file=sys.stderr, flush=True)
    dev = torch.device("cuda", local)
    cdev = torch.device("cpu") if gloo_check else dev     # where collectives run
    N, L = cfg.N, cfg.L
    from paper_2409_05205_b200.dist import (choose_axis, shard_out_blocks, shard_range,
                                            sub_layer_weights)
    # ---- partition: weak = every rank its own cfg.B images
    # (seeded per rank); strong = one global batch of cfg.B images split by
    # image, or by output-channel block when it has fewer images than ranks
    ctx0 = he.Context(cfg.primes, cfg.log2N, cfg.t, local)
    Ly0 = cfg.conv[0]
    n_ob0 = ctx0.plan(Ly0.c_i, Ly0.c_o, Ly0.w_i, Ly0.h_i, Ly0.f_w, Ly0.f_h, Ly0.stride,
                      Ly0.pad).n_ob
    axis = "batch" if scaling == "weak" else choose_axis(cfg.B, n_ob0, world)
    if scaling == "weak":
        B, b_lo, seed_r = cfg.B, 0, cfg.seed + 1000 * rank
        B_global = cfg.B * world
    elif axis == "batch":
        b_lo, b_hi = shard_range(cfg.B, rank, world)
        B, seed_r, B_global = b_hi - b_lo, cfg.seed, cfg.B
    else:
        B, b_lo, seed_r, B_global = cfg.B, 0, cfg.seed, cfg.B
    del ctx0
    if B == 0 or (axis == "out_block" and n_ob0 < world):
        raise SystemExit(f"{args.workload} with {scaling} scaling leaves rank {rank} of "
                         f"{world} without work (batch {cfg.B}, {n_ob0} output blocks)")
    ctx = he.Context(cfg.primes, cfg.log2N, cfg.t, local)
    # all work on a dedicated (non-default) stream: CUDA-graph capture needs it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    def d(a):
        a = np.ascontiguousarray(a)
        if a.dtype == np.uint64:
            a = a.view(np.int64)
        elif a.dtype == np.uint32:
            a = a.view(np.int32)
        return torch.from_numpy(a).to(dev)

    # ---- server init (Alg. 1 Line 4 / Alg. 2 Lines 3-4), timed separately
    layers, fspecs, c0_h, c0_d, phi_d, phi_h, outs, comps = [], [], [], [], [], [], [], []
    t_init0 = time.perf_counter()
    init_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    init_ev[0].record()
    ob_span = []
    for i, Ly in enumerate(cfg.conv):
        W = synth.weights(cfg, i)
        if axis == "out_block":
            pf = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride, Ly.pad)
            o_lo, o_hi = shard_out_blocks(pf.n_ob, rank, world)
            ob_span.append((o_lo, o_hi, pf.n_ob))
            W = sub_layer_weights(W, pf.c_ob, o_lo, o_hi)
            Ly = synth.ConvLayer(Ly.c_i, W.shape[0], Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h,
                                 Ly.stride, Ly.pad)
        p = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride,
                     Ly.pad)
        layers.append(LayerWork(i, Ly, p, N, L, B))
        fspecs.append(ctx.pack_filters(p, d(W)) if Ly.c_o > 0 else None)
    init_ev[1].record()
    torch.cuda.synchronize()
    init_ms = init_ev[0].elapsed_time(init_ev[1])
    for lw in layers:
        p = lw.p
        Bg = B if scaling == "weak" else cfg.B
        c0 = synth.uniform_residues((Bg, p.n_ib, L, N), cfg.primes,
                                    seed_r, "c0", lw.idx)[b_lo:b_lo + B]
        if axis == "out_block":          # this rank's blocks of the full layer's mask
            o_lo, o_hi, n_ob_full = ob_span[lw.idx]
            ph = synth.phi1((Bg, n_ob_full, N), cfg.t, seed_r, lw.idx)[:, o_lo:o_hi]
        else:
            ph = synth.phi1((Bg, p.n_ob, N), cfg.t, seed_r, lw.idx)[b_lo:b_lo + B]
        c0, ph = np.ascontiguousarray(c0), np.ascontiguousarray(ph)
        c0_h.append(torch.from_numpy(c0.view(np.int64)).pin_memory())
        phi_h.append(torch.from_numpy(ph.view(np.int32)).pin_memory())
        c0_d.append(c0_h[-1].to(dev))
        phi_d.append(phi_h[-1].to(dev))
        outs.append(ctx.empty_u64(B, p.n_ob, L, N))
        comps.append(ctx.empty_u64(B, p.n_ob, L, p.n_valid))
    nstr = max(1, args.streams)
    # workspaces cover the dense (client) plans too
    ws_all = [torch.empty(max(ctx.conv_workspace(p, B).numel() for p in
                              [lw.p for lw in layers] + [ctx.dense_plan(lw.p) for lw in layers]),
                          dtype=torch.uint8, device=dev)
              for _ in range(nstr)]
    ws = ws_all[0]
    side = [stream] + [torch.cuda.Stream(dev) for _ in range(nstr - 1)]
    fc = None
    if cfg.fc is not None:
        n_i, n_o = cfg.fc.n_i, cfg.fc.n_o
        wspec, benc = ctx.fc_pack_weights(d(synth.fc_weights(cfg)),
                                          d(synth.fc_bias(cfg)))
        Bg = B if scaling == "weak" else cfg.B
        fc_c0 = np.ascontiguousarray(synth.uniform_residues(
            (Bg, L, N), cfg.primes, seed_r, "c0", 99)[b_lo:b_lo + B])
        fc_ph = np.ascontiguousarray(synth.phi1((Bg, n_o), cfg.t, seed_r, 99)[b_lo:b_lo + B])
        fc = dict(n_i=n_i, n_o=n_o, wspec=wspec, benc=benc,
                  c0_h=torch.from_numpy(fc_c0.view(np.int64)).pin_memory(),
                  ph_h=torch.from_numpy(fc_ph.view(np.int32)).pin_memory())
        fc["c0_d"] = fc["c0_h"].to(dev)
        fc["ph_d"] = fc["ph_h"].to(dev)
        fc["out"] = ctx.empty_u64(B, L, n_o)
        fc["ws"] = ctx.fc_workspace(n_i, n_o, B)
        fc["out_h"] = torch.empty((B, L, n_o), dtype=torch.int64).pin_memory()
    comp_h = [torch.empty(c.shape, dtype=torch.int64).pin_memory() for c in comps]
    torch.cuda.synchronize()

    evals_step = sum(lw.evals for lw in layers) + (B if fc else 0)
    evals_all = evals_step                # every rank's work (value = all ranks / max time)
    if world > 1:
        _t = torch.tensor([evals_step], dtype=torch.float64, device=cdev)
        dist.all_reduce(_t)
        evals_all = int(_t.item())
    launches_step = 3 * len(layers) * (nstr if args.overlap == "batch" else 1) + \
        (2 if fc else 0)

    fork_ev = [torch.cuda.Event() for _ in range(nstr)]
    from paper_2409_05205_b200.dist import shard_range
    sub = [shard_range(B, k, nstr) for k in range(nstr)]

    po_flag = [bool(args.payload_only)]
    order = list(enumerate(layers))     # heavy layers first (reversed: 2.36 vs 2.34 ms)
    # job -> stream: round-robin (layer i on stream i % nstr, the FC job on the
    # next one), or LPT: every job timed alone once (after one warm-up call),
    # then dealt longest first to the stream with the least work so far, so
    # no stream is left running alone at the end of the step (round-robin put
    # layers 1, 7, 13 and the FC, the heaviest mix, on one stream)
    job_stream = {i: i % nstr for i in range(len(layers))}
    job_stream["fc"] = len(layers) % nstr
    job_ms = None
    if nstr > 1 and args.overlap == "layers" and args.schedule == "lpt":
        def run_job(j):
            if j == "fc":
                ctx.fc(fc["n_i"], fc["n_o"], fc["c0_d"], fc["wspec"], fc["benc"],
                       fc["ph_d"], fc["out"], fc["ws"])
            else:
                lw = layers[j]
                ctx.conv(lw.p, c0_d[j], fspecs[j], phi_d[j], outs[j], ws, compact=comps[j])
        jobs = list(range(len(layers))) + (["fc"] if fc else [])
        job_ms = {}
        for j in jobs:
            run_job(j)
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run_job(j)
            b_.record()
            b_.synchronize()
            job_ms[j] = a.elapsed_time(b_)
        load = [0.0] * nstr
        lpt = sorted(jobs, key=lambda j: -job_ms[j])
        for j in lpt:
            k = min(range(nstr), key=lambda k: load[k])
            job_stream[j] = k
            load[k] += job_ms[j]
        order = [(j, layers[j]) for j in lpt if j != "fc"]

    def step():
        po = po_flag[0]
        if nstr == 1:
            for i, lw in enumerate(layers):
                ctx.conv(lw.p, c0_d[i], fspecs[i], phi_d[i], None if po else outs[i], ws,
                         compact=comps[i], full=not po)
        else:
            fork_ev[0].record(stream)
            for k in range(1, nstr):
                side[k].wait_event(fork_ev[0])
            for i, lw in order:
                if args.overlap == "layers":
                    k = job_stream[i]
                    ctx.conv(lw.p, c0_d[i], fspecs[i], phi_d[i], None if po else outs[i],
                             ws_all[k], compact=comps[i], full=not po, stream=side[k])
                    continue
                for k, (lo, hi) in enumerate(sub):
                    ctx.conv(lw.p, c0_d[i][lo:hi], fspecs[i], phi_d[i][lo:hi],
                             None if po else outs[i][lo:hi], ws_all[k],
                             compact=comps[i][lo:hi], full=not po, stream=side[k])
            if fc and args.overlap == "layers":
                # the FC job is independent of the conv jobs (R22): it is
                # the 20th layer job, dealt to the next stream in turn
                ctx.fc(fc["n_i"], fc["n_o"], fc["c0_d"], fc["wspec"], fc["benc"],
                       fc["ph_d"], fc["out"], fc["ws"], stream=side[job_stream["fc"]])
            for k in range(1, nstr):
                fork_ev[k].record(side[k])
                stream.wait_event(fork_ev[k])
        if fc and (nstr == 1 or args.overlap != "layers"):
            ctx.fc(fc["n_i"], fc["n_o"], fc["c0_d"], fc["wspec"], fc["benc"],
                   fc["ph_d"], fc["out"], fc["ws"])

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            if gloo_check:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    graph = None
    if args.graph and not args.profile:
        # the whole step (both sub-batch streams, every layer) as one graph
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step()
        graph.replay()
        torch.cuda.synchronize()
    run_step = graph.replay if graph is not None else step
    mk = lambda: torch.cuda.Event(enable_timing=True)
    # ---- timed region 1 (the headline value): the step as configured
    e0, e1 = mk(), mk()
    barrier()
    sampler = ClockSampler(local)
    with (sampler if not args.profile else _Null()):
        e0.record()
        for k in range(args.steps):
            run_step()
        e1.record()
        barrier()
    ms_step = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    # ---- the same step writing only the masked valid-slot payload (what the
    # server sends), reported beside the headline
    payload_only = None
    if not args.profile and not args.payload_only:
        po_flag[0] = True
        step()
        g2 = None
        if args.graph:
            torch.cuda.synchronize()
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2, stream=stream):
                step()
            g2.replay()
        run2 = g2.replay if g2 is not None else step
        barrier()
        e0.record()
        for k in range(args.steps):
            run2()
        e1.record()
        barrier()
        ms_po = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        payload_only = {"ms_per_step": ms_po, "value": evals_all / (ms_po * 1e-3),
                        "what": "he_conv_ex with d_out = NULL: extraction, mask and "
                                "payload fused, full c0^r not materialised"}
        po_flag[0] = False
        del g2
    # ---- timed region 2 (kernel analysis): one launch sequence per layer
    # (streams = 1) with stage events from he_conv_ex / he_fc_ex, so each
    # kernel's duration is measured without overlap
    evs = [[[mk() for _ in range(4)] for _ in layers] + ([[mk() for _ in range(3)]] if fc else [])
           for _ in range(args.steps)]
    for E in evs:                    # torch creates the cudaEvent_t lazily
        for grp in E:
            for ev in grp:
                ev.record()

    def step_seq(E):
        for i, lw in enumerate(layers):
            ctx.conv(lw.p, c0_d[i], fspecs[i], phi_d[i], outs[i], ws, events=E[i],
                     compact=comps[i])
        if fc:
            ctx.fc(fc["n_i"], fc["n_o"], fc["c0_d"], fc["wspec"], fc["benc"],
                   fc["ph_d"], fc["out"], fc["ws"], events=E[len(layers)])

    s0, s1 = mk(), mk()
    barrier()
    s0.record()
    for k in range(args.steps):
        step_seq(evs[k])
    s1.record()
    barrier()
    ms_seq = max_over_ranks(s0.elapsed_time(s1) / args.steps)
    # stage sums (ms per step, averaged over the analysis steps)
    st = {"ntt_fwd": 0.0, "mac_fold": 0.0, "intt_scatter": 0.0,
          "gaps": 0.0, "fc_ntt_fwd": 0.0, "fc_inv": 0.0}
    for k in range(args.steps):
        E = evs[k]
        for i in range(len(layers)):
            a = E[i]
            st["ntt_fwd"] += a[0].elapsed_time(a[1])
            st["mac_fold"] += a[1].elapsed_time(a[2])
            st["intt_scatter"] += a[2].elapsed_time(a[3])
            nxt = E[i + 1][0] if i + 1 < len(E) else None
            if nxt is not None:
                st["gaps"] += a[3].elapsed_time(nxt)
        if fc:
            f = E[len(layers)]
            st["fc_ntt_fwd"] += f[0].elapsed_time(f[1])
            st["fc_inv"] += f[1].elapsed_time(f[2])
    st = {k: v / args.steps for k, v in st.items()}
    per_layer = []
    for i, lw in enumerate(layers):
        t = [0.0, 0.0, 0.0]
        for k in range(args.steps):
            a = evs[k][i]
            t[0] += a[0].elapsed_time(a[1])
            t[1] += a[1].elapsed_time(a[2])
            t[2] += a[2].elapsed_time(a[3])
        p = lw.p
        per_layer.append({"layer": i, "s": p.s, "n_ib": p.n_ib, "n_ob": p.n_ob,
                          "c_o": lw.Ly.c_o, "ntt_ms": t[0] / args.steps,
                          "mac_ms": t[1] / args.steps, "intt_ms": t[2] / args.steps})

    # ---- algorithmic work per step
    W_ntt_bfly = sum(lw.ntt_bfly for lw in layers)
    W_ntt_bytes = sum(lw.ntt_bytes for lw in layers)
    W_macs = sum(lw.macs for lw in layers)
    W_mac_bytes = sum(lw.mac_bytes for lw in layers)
    W_intt_bfly = sum(lw.intt_bfly for lw in layers)
    W_intt_bytes = sum(lw.intt_bytes for lw in layers)

    hbm_gbs, hbm_src = peaks()
    u1 = u1_peaks(local)
    # U1 rates were measured at the in-kernel clock; they are the alu roofs.
    # transforms run FP64 butterflies by default (HE_NTT=int: integer Shoup)
    ntt_int = os.environ.get("HE_NTT", "")[:1] == "i"
    ct_roof = u1["ct_bfly"]["per_s"] if ntt_int else u1["dp_ct_bfly"]["per_s"]
    gs_roof = u1["gs_bfly"]["per_s"] if ntt_int else u1["dp_gs_bfly"]["per_s"]
    # int8 tensor-core MAC: 49 u8 x u8 products per 50-bit modMAC, so its alu
    # roof is the measured int8 rate of the instruction it issues / 49:
    # tcgen05.mma M=128 N=16 (k_mac_tc, B >= 128) or mma.sync (k_mac_imma);
    # HE_MAC=imad runs the IMAD kernel, whose roof is U1 "modmac".
    mac_tc_used = (B >= 128 and os.environ.get("HE_MAC_TC", "2") != "0") or \
        os.environ.get("HE_MAC_TC") == "1"
    if os.environ.get("HE_MAC", "")[:1] == "i":
        mac_roof, mac_roof_src = u1["modmac"]["per_s"], "U1 modmac (IMAD)"
    elif mac_tc_used:
        mac_roof, mac_roof_src = u1["tc_i8_m128n16"]["per_s"] / 49, \
            "U1 tcgen05.mma kind::i8 M=128 N=16 int8 MAC/s / 49"
    else:
        mac_roof, mac_roof_src = u1["imma_u8"]["per_s"] / 49, \
            "U1 mma.sync m16n8k32 int8 MAC/s / 49"
    kern = {
        "ntt_fwd": (st["ntt_fwd"], W_ntt_bfly, ct_roof, "Gbutterfly/s", W_ntt_bytes),
        "mac_fold": (st["mac_fold"], W_macs, mac_roof, "Gmodmac/s", W_mac_bytes),
        "intt_scatter": (st["intt_scatter"], W_intt_bfly, gs_roof, "Gbutterfly/s",
                         W_intt_bytes),
    }
    rl = {}
    for name, (ms, ops, alu_peak, unit, byts) in kern.items():
        t = ms * 1e-3
        if t <= 0:
            continue
        t_alu, t_hbm = ops / alu_peak, byts / (hbm_gbs * 1e9)
        bound = "alu" if t_alu >= t_hbm else "hbm"
        if bound == "alu":
            rl[name] = {"bound": "alu", "achieved": ops / t / 1e9,
                        "peak": alu_peak / 1e9, "unit": unit,
                        "frac": (ops / t) / alu_peak, "traffic": None,
                        "share_of_step": ms / ms_seq,
                        "hbm_frac": byts / t / 1e9 / hbm_gbs}
        else:
            rl[name] = {"bound": "hbm", "achieved": byts / t / 1e9,
                        "peak": hbm_gbs, "unit": "GB/s",
                        "frac": byts / t / 1e9 / hbm_gbs, "traffic": None,
                        "share_of_step": ms / ms_seq,
                        "alu_frac": (ops / t) / alu_peak}
    for name in ("ntt_fwd", "intt_scatter"):          # FP64 kernels: DFMA-pipe view
        if name in rl:
            ms, ops = kern[name][0], kern[name][1]
            rl[name]["dfma_pipe_frac"] = ops / (ms * 1e-3) * DP_OPS_PER_BFLY / u1["dfma"]["per_s"]
    if "mac_fold" in rl:
        rl["mac_fold"]["alu_peak_source"] = mac_roof_src
    # DRAM traffic per launch from an ncu pass of THIS workload (profiles/
    # traffic_<workload>.json, written by scripts/traffic_summary.py from the
    # same bench command), beside the algorithmic bytes per launch (traffic
    # well above it = re-reads).  A file of another workload is never used.
    tr_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                           f"traffic_{args.workload}.json")
    tr = json.load(open(tr_path)) if os.path.exists(tr_path) else {}
    if tr and tr.get("workload") not in (None, args.workload):
        tr = {}
    for name, (ms, ops, alu_peak, unit, byts) in kern.items():
        if name not in rl:
            continue
        rl[name]["algorithmic_bytes_per_launch"] = byts / len(layers)
        if name in tr:
            rl[name]["traffic"] = tr[name]["mean_dram_bytes_per_launch"]
            rl[name]["traffic_source"] = f"profiles/traffic_{args.workload}.json (ncu " + \
                "dram__bytes_read.sum + dram__bytes_write.sum, " + \
                str(tr[name]["launches"]) + " launches, " + str(tr.get("code", "?")) + ")"
    dom = max(kern, key=lambda k: kern[k][0])
    roofline = dict(rl[dom])
    roofline["kernel"] = dom
    roofline["peak_source"] = ("U1 register-resident microbenchmark on this GPU"
                               if roofline["bound"] == "alu" else hbm_src)
    roofline["timed_in"] = ("sequential analysis pass (streams=1) of the same step, "
                            "CUDA events around each kernel (he_conv_ex)")

    # ---- NTT limbs/s at every ring size of BASELINE's configs (N = 1024,
    # 8192, 16384, 32768; he_ntt_forward / he_ntt_inverse alone, >= 256 MB of
    # limbs per launch so the data is larger than L2), each against the FP64
    # roofs: U1's measured butterfly sequence and the DFMA pipe at the
    # algorithmic 8 FP64 operations per butterfly (dp_mulmod's 6 + add/sub)
    ntt_sweep = []
    if not args.profile:
        for (vN, vprimes) in [(1024, synth.PRIMES_CFG1), (8192, synth.PRIMES_N8192[:2]),
                              (16384, synth.PRIMES_N16384[:2]),
                              (32768, synth.PRIMES_N32768[:2])]:
            vctx = he.Context(list(vprimes), vN.bit_length() - 1, cfg.t, local)
            vL = len(vprimes)
            nlv = max(vL, (256 << 20) // (8 * vN) // vL * vL)
            vbuf = torch.from_numpy(synth.uniform_residues(
                (nlv // vL, vL, vN), list(vprimes), 7, "misc", vN).view(np.int64)).to(dev)
            res = {"N": vN, "limbs_per_launch": nlv}
            lg = vN.bit_length() - 1
            for nm, fn, roof in (("forward", vctx.ntt_forward, ct_roof),
                                 ("inverse", vctx.ntt_inverse, gs_roof)):
                for _ in range(3):
                    fn(vbuf)
                a0, a1 = mk(), mk()
                a0.record()
                for _ in range(5):
                    fn(vbuf)
                a1.record()
                torch.cuda.synchronize()
                tt = a0.elapsed_time(a1) / 5 * 1e-3
                lps = nlv / tt
                bfly = vN // 2 * lg
                res[nm] = {"limbs_per_s": lps,
                           "frac_u1_fp64_roof": lps * bfly / roof,
                           "frac_dfma_pipe": lps * bfly * DP_OPS_PER_BFLY / u1["dfma"]["per_s"],
                           "hbm_frac": lps * 16 * vN / (hbm_gbs * 1e9)}
            ntt_sweep.append(res)
            del vbuf, vctx
    # ---- NTT limbs/s (he_ntt_forward alone, 1024 limbs > L2)
    nl = 1024 // L * L
    buf = torch.from_numpy(synth.uniform_residues(
        (nl // L, L, N), cfg.primes, 7, "misc").view(np.int64)).to(dev)
    for _ in range(3):
        ctx.ntt_forward(buf)
    a, b = mk(), mk()
    a.record()
    for _ in range(10):
        ctx.ntt_forward(buf)
    b.record()
    torch.cuda.synchronize()
    t_ntt = a.elapsed_time(b) / 10 * 1e-3
    logN = N.bit_length() - 1
    ntt = {"N": N, "limbs_per_launch": nl, "limbs_per_s": nl / t_ntt,
           "alu_roof_limbs_per_s": ct_roof / (N // 2 * logN),
           "hbm_roof_limbs_per_s": hbm_gbs * 1e9 / (16 * N)}
    ntt["roof_limbs_per_s"] = min(ntt["alu_roof_limbs_per_s"], ntt["hbm_roof_limbs_per_s"])
    ntt["frac"] = ntt["limbs_per_s"] / ntt["roof_limbs_per_s"]
    # inverse transform (he_ntt_inverse), same batch
    for _ in range(3):
        ctx.ntt_inverse(buf)
    a.record()
    for _ in range(10):
        ctx.ntt_inverse(buf)
    b.record()
    torch.cuda.synchronize()
    t_inv = a.elapsed_time(b) / 10 * 1e-3
    ntt["inverse_limbs_per_s"] = nl / t_inv
    inv_roof = min(gs_roof / (N // 2 * logN), ntt["hbm_roof_limbs_per_s"])
    ntt["inverse_frac"] = ntt["inverse_limbs_per_s"] / inv_roof
    ntt["sizes"] = ntt_sweep
    del buf

    # ---- e2e: the server loop through the public API with host buffers.
    # c0 arrives in the 50-bit wire format (he_residues_unpack50), the
    # server draws its mask phi1 on the device (he_phi1_generate), and the
    # valid-slot payload leaves in the wire format (he_residues_pack50).
    # Copies overlap compute: layer i+1's upload (H2D stream) and layer
    # i-1's download (D2H stream) run while layer i computes.
    e2e = None
    if not args.no_e2e and not args.profile:
        c0_pk_h, c0_pk_d, comp_pk_d, comp_pk_h = [], [], [], []
        for i in range(len(layers)):
            pk = ctx.pack50(c0_d[i])
            c0_pk_d.append(pk)
            c0_pk_h.append(pk.cpu().pin_memory())
            comp_pk_d.append(torch.empty(ctx.packed_bytes(comps[i].numel()),
                                         dtype=torch.uint8, device=dev))
            comp_pk_h.append(torch.empty(comp_pk_d[-1].shape, dtype=torch.uint8).pin_memory())
        if fc:
            fc["c0_pk_d"] = ctx.pack50(fc["c0_d"])
            fc["c0_pk_h"] = fc["c0_pk_d"].cpu().pin_memory()
            fc["out_pk_d"] = torch.empty(ctx.packed_bytes(fc["out"].numel()),
                                         dtype=torch.uint8, device=dev)
            fc["out_pk_h"] = torch.empty(fc["out_pk_d"].shape, dtype=torch.uint8).pin_memory()
        torch.cuda.synchronize()
        h2d = sum(t.numel() for t in c0_pk_h) + (fc["c0_pk_h"].numel() if fc else 0)
        d2h = sum(t.numel() for t in comp_pk_h) + (fc["out_pk_h"].numel() if fc else 0)
        h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        nl = len(layers) + (1 if fc else 0)
        up_done = [torch.cuda.Event() for _ in range(nl)]
        comp_done = [torch.cuda.Event() for _ in range(nl)]
        for e in comp_done:
            e.record(stream)
        mask_seed = [0]
        # variant: the payload switched to one limb (R28) before the wire
        sw = [ctx.empty_u64(*c.shape[:2], 1, c.shape[-1]) for c in comps]
        sw_pk_d = [torch.empty(ctx.packed_bytes(t.numel()), dtype=torch.uint8, device=dev)
                   for t in sw]
        sw_pk_h = [torch.empty(t.shape, dtype=torch.uint8).pin_memory() for t in sw_pk_d]

        # variant: sparse c0 upload (only the k_u columns the conv reads)
        sp = [lw.p.k_u < lw.p.s for lw in layers]
        c0c_d = [ctx.c0_compact(lw.p, c0_d[i]) if sp[i] else None for i, lw in enumerate(layers)]
        c0c_pk_d = [ctx.pack50(t) if t is not None else None for t in c0c_d]
        c0c_pk_h = [t.cpu().pin_memory() if t is not None else None for t in c0c_pk_d]
        torch.cuda.synchronize()

        def e2e_step(ms_keep=0, sparse=False):
            mask_seed[0] += 1
            for i, lw in enumerate(layers):
                spi = sparse and sp[i]
                with torch.cuda.stream(h2d_s):
                    h2d_s.wait_event(comp_done[i])          # WAR vs previous step
                    if spi:
                        c0c_pk_d[i].copy_(c0c_pk_h[i], non_blocking=True)
                    else:
                        c0_pk_d[i].copy_(c0_pk_h[i], non_blocking=True)
                    up_done[i].record(h2d_s)
                stream.wait_event(up_done[i])
                if spi:
                    ctx.unpack50(c0c_pk_d[i], c0c_d[i])
                    ctx.c0_expand(lw.p, c0c_d[i], out=c0_d[i])
                else:
                    ctx.unpack50(c0_pk_d[i], c0_d[i])
                ctx.phi1_generate((mask_seed[0] << 8) + i, phi_d[i])
                ctx.conv(lw.p, c0_d[i], fspecs[i], phi_d[i], outs[i], ws, compact=comps[i])
                if ms_keep:
                    ctx.mod_switch(comps[i], ms_keep, out=sw[i])
                    ctx.pack50(sw[i], sw_pk_d[i])
                else:
                    ctx.pack50(comps[i], comp_pk_d[i])
                comp_done[i].record(stream)
                with torch.cuda.stream(d2h_s):
                    d2h_s.wait_event(comp_done[i])
                    if ms_keep:
                        sw_pk_h[i].copy_(sw_pk_d[i], non_blocking=True)
                    else:
                        comp_pk_h[i].copy_(comp_pk_d[i], non_blocking=True)
            if fc:
                i = len(layers)
                with torch.cuda.stream(h2d_s):
                    h2d_s.wait_event(comp_done[i])
                    fc["c0_pk_d"].copy_(fc["c0_pk_h"], non_blocking=True)
                    up_done[i].record(h2d_s)
                stream.wait_event(up_done[i])
                ctx.unpack50(fc["c0_pk_d"], fc["c0_d"])
                ctx.phi1_generate((mask_seed[0] << 8) + i, fc["ph_d"])
                ctx.fc(fc["n_i"], fc["n_o"], fc["c0_d"], fc["wspec"], fc["benc"],
                       fc["ph_d"], fc["out"], fc["ws"])
                ctx.pack50(fc["out"], fc["out_pk_d"])
                comp_done[i].record(stream)
                with torch.cuda.stream(d2h_s):
                    d2h_s.wait_event(comp_done[i])
                    fc["out_pk_h"].copy_(fc["out_pk_d"], non_blocking=True)
            # the step ends when its last payload is on the host
            stream.wait_stream(d2h_s)

        for _ in range(2):
            e2e_step()
        barrier()
        x0, x1 = mk(), mk()
        x0.record()
        for _ in range(args.steps):
            e2e_step()
        x1.record()
        barrier()
        ms_e2e = max_over_ranks(x0.elapsed_time(x1) / args.steps)
        e2e = {"value": evals_all / (ms_e2e * 1e-3), "unit": "ct×pt evals/s",
               "ms_per_step": ms_e2e, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h,
               "wire": "50-bit packed residues (he_residues_pack50/unpack50); "
                       "phi1 drawn on device (he_phi1_generate)"}
        # PCIe roof of the end-to-end step: the same H2D bytes copied alone
        # (pinned -> device, one stream), and H2D + D2H concurrently
        big_h = torch.empty(h2d, dtype=torch.uint8).pin_memory()
        big_d = torch.empty(h2d, dtype=torch.uint8, device=dev)
        out_h = torch.empty(d2h, dtype=torch.uint8).pin_memory()
        out_d = torch.empty(d2h, dtype=torch.uint8, device=dev)
        for _ in range(2):
            big_d.copy_(big_h, non_blocking=True)
        torch.cuda.synchronize()
        x0.record()
        for _ in range(args.steps):
            big_d.copy_(big_h, non_blocking=True)
        x1.record()
        torch.cuda.synchronize()
        ms_h2d = x0.elapsed_time(x1) / args.steps
        x0.record()
        for _ in range(args.steps):
            with torch.cuda.stream(h2d_s):
                big_d.copy_(big_h, non_blocking=True)
            with torch.cuda.stream(d2h_s):
                out_h.copy_(out_d, non_blocking=True)
            stream.wait_stream(h2d_s)
            stream.wait_stream(d2h_s)
        x1.record()
        torch.cuda.synchronize()
        ms_both = x0.elapsed_time(x1) / args.steps
        e2e["pcie"] = {"h2d_gbs": h2d / (ms_h2d * 1e-3) / 1e9,
                       "h2d_only_ms": ms_h2d, "h2d_plus_d2h_ms": ms_both,
                       "frac": ms_h2d / ms_e2e,
                       "note": "copy-only times of the step's own wire bytes; frac = the "
                               "H2D-only copy time / the e2e step time (1.0 = the step "
                               "runs at the PCIe H2D roof)"}
        del big_h, big_d, out_h, out_d
        # same loop with the conv payloads modulus-switched to one limb
        for _ in range(2):
            e2e_step(1)
        barrier()
        x0.record()
        for _ in range(args.steps):
            e2e_step(1)
        x1.record()
        barrier()
        ms_sw = max_over_ranks(x0.elapsed_time(x1) / args.steps)
        # the switch kernel alone, every conv payload of the step
        m0, m1 = mk(), mk()
        m0.record()
        for i in range(len(layers)):
            ctx.mod_switch(comps[i], 1, out=sw[i])
        m1.record()
        torch.cuda.synchronize()
        sw_ms = m0.elapsed_time(m1)
        sw_bytes = sum(8 * c.numel() + 8 * t.numel() for c, t in zip(comps, sw))
        # both extensions: sparse c0 upload + payload switched to one limb
        for _ in range(2):
            e2e_step(1, True)
        barrier()
        x0.record()
        for _ in range(args.steps):
            e2e_step(1, True)
        x1.record()
        barrier()
        ms_ext = max_over_ranks(x0.elapsed_time(x1) / args.steps)
        e2e["sparse_upload_modswitch"] = {
            "ms_per_step": ms_ext, "value": evals_all / (ms_ext * 1e-3),
            "h2d_bytes_per_step": sum(c0c_pk_h[i].numel() if sp[i] else c0_pk_h[i].numel()
                                      for i in range(len(layers))) +
            (fc["c0_pk_h"].numel() if fc else 0),
            "d2h_bytes_per_step": sum(t.numel() for t in sw_pk_h) +
            (fc["out_pk_h"].numel() if fc else 0),
            "what": "protocol extensions: the client sends only the k_u columns of c0 "
                    "the conv reads (he_c0_compact / he_c0_expand), the payload is "
                    "modulus-switched to one limb"}
        e2e["modswitch"] = {
            "L_keep": 1, "ms_per_step": ms_sw,
            "value": evals_all / (ms_sw * 1e-3),
            "d2h_bytes_per_step": sum(t.numel() for t in sw_pk_h) +
            (fc["out_pk_h"].numel() if fc else 0),
            "kernel_ms_per_step": sw_ms,
            "kernel_hbm_frac": sw_bytes / (sw_ms * 1e-3) / 1e9 / peaks()[0]}

    # ---- multi-GPU: the one exchange of the path -- every
    # rank's compact payload assembled on all ranks (NCCL all_gather over
    # NVLink, by image or by output block as partitioned), timed alone and
    # as part of the step (the step followed by the gather, same clocks)
    gather = None
    if world > 1 and not args.profile:
        from paper_2409_05205_b200.dist import gather_blocks, gather_payload

        def assemble():
            hx = (lambda t: t.cpu()) if gloo_check else (lambda t: t)
            for i, c in enumerate(comps):
                if axis == "out_block":
                    gather_blocks(hx(c), ob_span[i][2])
                else:
                    gather_payload(hx(c), B_global)
            if fc and axis != "out_block":
                gather_payload(hx(fc["out"]), B_global)

        for _ in range(2):
            assemble()
        barrier()
        g0, g1 = mk(), mk()
        g0.record()
        for _ in range(args.steps):
            assemble()
        g1.record()
        barrier()
        ms_g = max_over_ranks(g0.elapsed_time(g1) / args.steps)
        gbytes = sum(c.numel() * 8 for c in comps) * world
        for _ in range(2):
            run_step()
            assemble()
        barrier()
        g0.record()
        for _ in range(args.steps):
            run_step()
            assemble()
        g1.record()
        barrier()
        ms_sg = max_over_ranks(g0.elapsed_time(g1) / args.steps)
        gather = {"ms_per_step": ms_g, "bytes_per_step_all_ranks": gbytes,
                  "GBps": gbytes / (ms_g * 1e-3) / 1e9, "axis": axis,
                  "with_gather": {"ms_per_step": ms_sg,
                                  "value": evals_all / (ms_sg * 1e-3),
                                  "what": "the headline step followed by the NCCL all_gather "
                                          "of every layer's compact payload (and the FC "
                                          "output), K steps timed together"}}

    # ---- client mirror path: the client's per-layer work
    # of Alg. 1 Lines 21-24 + Eq. (2) -- c1^r = valid slots of
    # sum_beta (v_beta s) p_beta^{(n)} through he_conv on the spectra of
    # he_pack_client_p, then he_decrypt_round on the compact payloads -- and
    # the server's offline p = fhat a + e_f (he_server_init_p), timed once.
    # v_beta s stand-ins are the resident uniform residues c0_d (the kernels'
    # cost does not depend on the values).
    extras = not (args.no_client or args.no_extras or args.profile or world > 1 or
                  axis == "out_block")
    client = None
    if extras:
        a_d = d(synth.uniform_residues((L, N), cfg.primes, cfg.seed, "a"))
        i0, i1 = mk(), mk()
        i0.record()
        pps = [ctx.server_init_p(lw.p, d(synth.weights(cfg, lw.idx)), a_d) for lw in layers]
        i1.record()
        torch.cuda.synchronize()
        p_init_ms = i0.elapsed_time(i1)
        pspecs = [ctx.pack_client_p(lw.p, pp) for lw, pp in zip(layers, pps)]
        del pps
        c1s = [torch.empty_like(c) for c in comps]
        msgs = [torch.empty(c.shape[:2] + (c.shape[-1],), dtype=torch.int32, device=dev)
                for c in comps]
        cl_ev = [[mk() for _ in range(3)] for _ in layers]

        def client_step(E=None):
            for i, lw in enumerate(layers):
                if E:
                    E[i][0].record()
                ctx.conv(ctx.dense_plan(lw.p), c0_d[i], pspecs[i], None, None, ws, compact=c1s[i],
                         full=False)
                if E:
                    E[i][1].record()
                ctx.decrypt_round(comps[i], c1s[i], out=msgs[i])
                if E:
                    E[i][2].record()

        for _ in range(2):
            client_step()
        barrier()
        y0, y1 = mk(), mk()
        y0.record()
        for _ in range(args.steps):
            client_step()
        y1.record()
        barrier()
        ms_client = max_over_ranks(y0.elapsed_time(y1) / args.steps)
        client_step(cl_ev)
        torch.cuda.synchronize()
        c1_ms = sum(E[0].elapsed_time(E[1]) for E in cl_ev)
        dec_ms = sum(E[1].elapsed_time(E[2]) for E in cl_ev)
        client = {"ms_per_step": ms_client,
                  "evals_per_s": sum(lw.evals for lw in layers) * world / (ms_client * 1e-3),
                  "c1r_ms": c1_ms, "decrypt_ms": dec_ms,
                  "server_init_p_ms": p_init_ms,
                  "what": "per step: c1^r (he_conv on he_pack_client_p spectra, compact) "
                          "+ he_decrypt_round over every conv layer's payload; "
                          "server_init_p_ms: Alg. 1 Line 5 for all layers, once"}
        del pspecs, c1s, msgs

    # ---- ablation: the unfolded path (full N-point products and inverse per
    # output channel, Alg. 1 Lines 14-17 literally) on the same conv layers,
    # one launch sequence, to show what the fold + incomplete transform save
    ablation = None
    if extras:
        import ctypes
        wsp = torch.empty(max(int(he._lib.he_conv_plain_workspace_bytes(
            ctx._h, ctypes.byref(lw.p), B)) for lw in layers), dtype=torch.uint8, device=dev)
        fpl = [ctx.pack_filters_plain(lw.p, d(synth.weights(cfg, lw.idx))) for lw in layers]
        for i, lw in enumerate(layers):
            ctx.conv_plain(lw.p, c0_d[i], fpl[i], phi_d[i], outs[i], wsp)
        torch.cuda.synchronize()
        a0, a1 = mk(), mk()
        a0.record()
        for i, lw in enumerate(layers):
            ctx.conv_plain(lw.p, c0_d[i], fpl[i], phi_d[i], outs[i], wsp)
        a1.record()
        torch.cuda.synchronize()
        ms_plain = a0.elapsed_time(a1)
        conv_seq = st["ntt_fwd"] + st["mac_fold"] + st["intt_scatter"] + st["gaps"]
        ablation = {"unfolded_conv_ms_per_step": ms_plain,
                    "folded_conv_ms_per_step_sequential": conv_seq,
                    "fold_speedup": ms_plain / conv_seq,
                    "what": "he_conv_plain (full N-point products + N-point inverse per "
                            "(b, n, l), then extraction) vs he_conv, both one launch "
                            "sequence, all 19 conv layers"}
        del fpl, wsp

    # ---- FC packing variants (§8(f)): sub-matrix tiling for n_i n_o > N
    # (R27) on this ring, and the FC at N = 32768 (config 5's ring)
    fc_var = None
    if extras:
        fc_var = []
        for (vn, vprimes, vlog, n_i, n_o, vB) in [
                ("fc512x1000_tiled", cfg.primes, cfg.log2N, 512, 1000, B),
                ("fc64x100_N32768", synth.CONFIGS[5].primes, synth.CONFIGS[5].log2N, 64, 100, B)]:
            vctx = he.Context(vprimes, vlog, cfg.t, local)
            n_it, n_ib, n_ot, n_t = vctx.fc_plan(n_i, n_o)
            rs = np.random.default_rng(5)
            Wv = d(rs.integers(-8, 8, (n_o, n_i)).astype(np.int32))
            bv = d(rs.integers(-8, 8, n_o).astype(np.int32))
            wsp, ben = vctx.fc_pack_weights(Wv, bv)
            c0v = d(synth.uniform_residues((vB, n_ib, len(vprimes), 1 << vlog), vprimes,
                                           cfg.seed, "c0", 98))
            phv = d(synth.phi1((vB, n_o), cfg.t, cfg.seed, 98))
            outv = vctx.empty_u64(vB, len(vprimes), n_o)
            wsv = vctx.fc_workspace(n_i, n_o, vB)
            for _ in range(3):
                vctx.fc(n_i, n_o, c0v, wsp, ben, phv, outv, wsv)
            f0, f1 = mk(), mk()
            f0.record()
            for _ in range(args.steps):
                vctx.fc(n_i, n_o, c0v, wsp, ben, phv, outv, wsv)
            f1.record()
            torch.cuda.synchronize()
            ms = f0.elapsed_time(f1) / args.steps
            fc_var.append({"name": vn, "N": 1 << vlog, "L": len(vprimes), "B": vB,
                           "n_i": n_i, "n_o": n_o, "n_it": n_it, "n_ib": n_ib, "n_ot": n_ot,
                           "n_t": n_t, "ms": ms,
                           "evals_per_s": vB * n_ib * n_t / (ms * 1e-3)})
            del vctx, wsp, ben, c0v, phv, outv, wsv

    # ---- multi-image packing (§8(f) row 4b, R31): the same images and layer,
    # P images per ciphertext at the paper's s = c_i (he_pack_input_multi
    # layout; he_conv unchanged; he_mask_extract_multi payload), against the
    # one-image-per-ciphertext step above: time, ciphertexts and bytes per image
    multi = None
    if (extras or (args.no_extras and not args.profile and world == 1)) and \
            cfg.idx in (3, 5) and axis == "batch":
        Ly = cfg.conv[0]
        so = Ly.c_i if Ly.c_i & (Ly.c_i - 1) == 0 else 0
        pm = ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride, Ly.pad, so)
        Dm, Pm = ctx.multi_image_spacing(pm)
        Bc = -(-B // Pm)
        fm = ctx.pack_filters(pm, d(synth.weights(cfg, 0)))
        c0m = torch.from_numpy(synth.uniform_residues((Bc, pm.n_ib, L, N), cfg.primes, seed_r,
                                                      "c0", 77).view(np.int64)).to(dev)
        phm = d(synth.phi1((Bc, pm.n_ob, N), cfg.t, seed_r, 77))
        outm = ctx.empty_u64(Bc, pm.n_ob, L, N)
        compm = ctx.empty_u64(Bc, pm.n_ob, L, Pm * pm.n_valid)
        wsm = ctx.conv_workspace(pm, Bc)

        def mstep():
            ctx.conv(pm, c0m, fm, phm, outm, wsm)
            ctx.mask_extract_multi(pm, outm, Pm, Dm, compact=compm)

        for _ in range(3):
            mstep()
        barrier()
        m0, m1 = mk(), mk()
        m0.record()
        for _ in range(args.steps):
            mstep()
        m1.record()
        barrier()
        ms_m = m0.elapsed_time(m1) / args.steps
        p1 = layers[0].p
        multi = {"s": pm.s, "images_per_ciphertext": Pm, "spacing_D": Dm,
                 "ciphertexts": Bc, "images": B, "ms_per_step": ms_m,
                 "images_per_s": B / (ms_m * 1e-3),
                 "one_image_per_ct": {"s": p1.s, "ms_per_step": ms_step,
                                      "images_per_s": B / (ms_step * 1e-3)},
                 "c0_bytes_per_image": 8 * pm.n_ib * L * N * Bc / B,
                 "c0_bytes_per_image_one_per_ct": 8 * p1.n_ib * L * N,
                 "out_bytes_per_image": 8 * pm.n_ob * L * N * Bc / B,
                 "out_bytes_per_image_one_per_ct": 8 * p1.n_ob * L * N,
                 "what": "he_conv (full c0^r) + he_mask_extract_multi on ceil(B/P) "
                         "multi-image ciphertexts (reading R31) vs the headline step"}
        del c0m, phm, outm, compm, wsm, fm

    # ---- chained pipeline (§8(f) row 3): the whole encrypted network, layer
    # to layer -- client encryption, server Conv/FC, client share,
    # decryption, R29 stub -- on the same 19 conv layers + FC, B images
    chain = None
    if extras and cfg.fc is not None:
        from paper_2409_05205_b200.chain import Chain
        rs = np.random.default_rng(cfg.seed)
        sk = synth.secret_key(N, cfg.h, cfg.seed)
        a_h = synth.uniform_residues((L, N), cfg.primes, cfg.seed, "a")
        b_h = synth.uniform_residues((L, N), cfg.primes, cfg.seed, "misc", 3)  # pk stand-in
        efs = [d(rs.integers(-8, 9, (lw.Ly.c_o, lw.p.n_ib, N)).astype(np.int32)) for lw in layers]
        ch = Chain(ctx, [lw.Ly for lw in layers],
                   [d(synth.weights(cfg, lw.idx)) for lw in layers],
                   d(synth.fc_weights(cfg)), d(synth.fc_bias(cfg)),
                   d(sk.astype(np.int32)), d(a_h), d(b_h), efs)
        vv = [d(rs.integers(-1, 2, (B, lw.p.n_ib, N)).astype(np.int32)) for lw in layers]
        ee = [d(rs.integers(-8, 9, (B, lw.p.n_ib, N)).astype(np.int32)) for lw in layers]
        v_fc = d(rs.integers(-1, 2, (B, 1, N)).astype(np.int32))
        e_fc = d(rs.integers(-8, 9, (B, 1, N)).astype(np.int32))
        img0 = d(synth.images(cfg, 0))
        for _ in range(2):
            ch.run(img0, vv, ee, 1, 8, 255, v_fc, e_fc)
        barrier()
        h0, h1 = mk(), mk()
        h0.record()
        for k in range(args.steps):
            ch.run(img0, vv, ee, 2 + k, 8, 255, v_fc, e_fc)
        h1.record()
        barrier()
        ms_chain = max_over_ranks(h0.elapsed_time(h1) / args.steps)
        chain = {"ms_per_step": ms_chain, "ms_per_image": ms_chain / B,
                 "images_per_s": B * world / (ms_chain * 1e-3),
                 "what": "plain-20 encrypted end to end on the device: per layer client "
                         "encryption (he_pk_mask, he_pack_input), server conv + mask, "
                         "client c1^r + decryption + R29 stub; avgpool + FC; inputs "
                         "resident, fresh randomness tensors reused across steps"}
        del ch

    # ---- CPU baseline: the oracle as it stands, rank 0, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        from oracle import ref as R
        ring = R.Ring(N, cfg.primes, cfg.t)
        nimg = min(B, 32) if cfg.idx == 4 else 1
        c0n = [t[:nimg].numpy().view(np.uint64) for t in c0_h]
        phn = [t[:nimg].numpy().view(np.uint32) for t in phi_h]
        oplans = [R.plan_conv(lw.Ly, N) for lw in layers]
        Ws = [synth.weights(cfg, i) for i in range(len(layers))]
        t0 = time.perf_counter()
        reps = 0
        while True:                      # ~10 s of oracle work (at most 8 passes)
            for i in range(len(layers)):
                R.compact(R.conv_server(c0n[i], Ws[i], oplans[i], ring, phn[i]), oplans[i])
            if fc:
                R.fc_server(fc["c0_h"][:nimg].numpy().view(np.uint64), synth.fc_weights(cfg),
                            synth.fc_bias(cfg), ring, fc["ph_h"][:nimg].numpy().view(np.uint32))
            reps += 1
            if time.perf_counter() - t0 > 10.0 or reps >= 8:
                break
        dt = time.perf_counter() - t0
        ev = reps * nimg * (sum(lw.evals // B for lw in layers) + (1 if fc else 0))
        cpu = {"value": ev / dt, "unit": "ct×pt evals/s", "cores": os.cpu_count(),
               "kind": "oracle",
               "sample": f"{reps} pass(es) x {nimg} image(s) x all {len(layers)} conv"
                         f"{' + FC' if fc else ''} layers ({dt:.1f} s wall)",
               "cpu_model": cpu_model()}
        # the CPU textbook-NTT path (oracle/cpu_baseline.py:
        # NTT-domain products, pinned to the oracle), same images and layers,
        # all cores; filter spectra prepared outside the timing
        try:
            from oracle import cpu_baseline as CB
            fsp = [CB.prepare_filters(Ws[i], oplans[i], ring) for i in range(len(layers))]
            t0, reps = time.perf_counter(), 0
            while True:
                for i in range(len(layers)):
                    R.compact(CB.conv_server(c0n[i], fsp[i], oplans[i], ring, phn[i]), oplans[i])
                reps += 1
                if time.perf_counter() - t0 > 10.0 or reps >= 8:
                    break
            dtn = time.perf_counter() - t0
            evn = reps * nimg * sum(lw.evals // B for lw in layers)
            cpu["ntt_path"] = {"value": evn / dtn, "unit": "ct×pt evals/s",
                               "cores": os.cpu_count(), "kind": "cpu textbook NTT",
                               "sample": f"{reps} pass(es) x {nimg} image(s) x all "
                                         f"{len(layers)} conv layers ({dtn:.1f} s wall)"}
            del fsp
        except Exception as exc:                      # reported, not fatal
            cpu["ntt_path"] = {"error": repr(exc)[:200]}
        # the same oracle on one host thread (the paper's own numbers are
        # single-thread): a child process with OMP_NUM_THREADS=1
        # times one image through the same layers
        try:
            r1 = subprocess.run(
                [sys.executable, "-c",
                 "import sys; sys.path.insert(0, %r); import bench; "
                 "bench.oracle_single_thread(%d)" % (ROOT, cfg.idx)],
                env=dict(os.environ, OMP_NUM_THREADS="1", CUDA_VISIBLE_DEVICES=""),
                capture_output=True, text=True, timeout=300)
            cpu["single_thread"] = json.loads(r1.stdout.strip().splitlines()[-1])
        except Exception as exc:                      # reported, not fatal
            cpu["single_thread"] = {"error": repr(exc)[:200]}

    clocks = sampler.summary() if not args.profile else None
    if rank == 0:
        value = evals_all / (ms_step * 1e-3)
        line = {
            "metric": "Conv+FC layer ct×pt evals/sec", "value": value,
            "unit": "ct×pt evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"cfg{cfg.idx} {cfg.name}: "
                                   f"{len(layers)} conv{' + FC' if fc else ''}, "
                                   f"N={N}, L={L}, "
                                   + (f"B={B}/GPU" if scaling == "weak" else
                                      f"B={cfg.B} global"),
                       "global_batch": B_global, "N": N, "L": L,
                       "parallelism": (f"dp{world} (batch-sharded, no data-path collective)"
                                       if axis == "batch" else
                                       f"ob{world} (output-channel blocks, no data-path "
                                       f"collective)"),
                       "partition_axis": axis,
                       "streams": nstr, "overlap": args.overlap,
                       "schedule": (args.schedule if nstr > 1 and args.overlap == "layers"
                                    else None),
                       "job_streams": ({str(j): k for j, k in job_stream.items()}
                                       if nstr > 1 and args.overlap == "layers" else None),
                       "cuda_graph": graph is not None,
                       "mac": ("tcgen05.mma kind::i8, TMEM accumulators (k_mac_tc)"
                               if (B >= 128 and os.environ.get("HE_MAC_TC", "2") != "0")
                               or os.environ.get("HE_MAC_TC") == "1"
                               else "mma.sync int8 byte planes (k_mac_imma)"),
                       "l2": "inputs larger than L2 (>1 GB touched per step)"},
            "ms_per_plain20_image": ms_step / B_global if cfg.idx == 4 else None,
            "sequential_ms_per_step": ms_seq,
            "ntt": ntt, "stages_ms_per_step": st, "per_layer": per_layer,
            "roofline": roofline,
            "roofline_all": rl, "u1": u1, "init_ms": init_ms,
            "cpu_baseline": cpu, "e2e": e2e, "payload_only": payload_only, "gather": gather,
            "multi_image": multi, "ablation": ablation, "client": client, "chain": chain, "fc_variants": fc_var, "clocks": clocks,
            "gpu_launches": launches_step * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass

    def summary(self):
        return None


if __name__ == "__main__":
    main()
