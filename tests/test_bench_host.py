"""Host logic of bench.py (not gpu): argument defaults the driver relies on
and the algorithmic work counts behind the roofline."""
import sys
import types

import pytest

sys.argv = sys.argv[:1]
import bench  # noqa: E402
import synth  # noqa: E402
from oracle import ref as R  # noqa: E402


def _plan(Ly, N):
    o = R.plan_conv(Ly, N)
    return types.SimpleNamespace(s=o.s, n_ib=o.n_ib, n_ob=o.n_ob, c_ob=o.c_ob,
                                 n_valid=o.n_valid, k_u=min(o.s, (o.c_ib + 3) & ~3))


def test_defaults(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert (a.gpus, a.impl, a.workload) == (1, "ours", "plain20")
    assert a.warmup >= 3 and a.steps >= 1


def test_layer_work_counts_config4():
    cfg = synth.CONFIGS[4]
    N, L, B = cfg.N, cfg.L, cfg.B
    tot_evals = tot_macs = 0
    for i, Ly in enumerate(cfg.conv):
        p = _plan(Ly, N)
        w = bench.LayerWork(i, Ly, p, N, L, B)
        M = N // p.s
        assert w.evals == B * Ly.c_o * p.n_ib
        # modMACs: every fold group, image, channel and used column
        assert w.macs == L * M * p.n_ib * p.k_u * B * Ly.c_o
        # incomplete forward transform on the k_u used columns
        assert w.ntt_bfly == B * p.n_ib * L * p.k_u * (M // 2) * (M.bit_length() - 1)
        # folded inverse: (N/s)-point transforms per (b, n, l)
        assert w.intt_bfly == B * p.n_ob * p.c_ob * L * (M // 2) * (M.bit_length() - 1)
        tot_evals += w.evals
        tot_macs += w.macs
    assert tot_evals == sum(B * Ly.c_o * _plan(Ly, N).n_ib for Ly in cfg.conv)
    # k_u halves the s = 128 layers' MAC: c_i = 64 of s = 128 columns
    p14 = _plan(cfg.conv[14], N)
    assert (p14.s, p14.k_u) == (128, 64)
