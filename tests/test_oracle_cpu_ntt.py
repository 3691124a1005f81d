"""The CPU textbook-NTT baseline (bench.py cpu_baseline)
computes exactly the oracle's server definition (not gpu)."""
import numpy as np
import pytest

import synth
from oracle import cpu_baseline as CB
from oracle import ref as R

CASES = [
    (synth.CONFIGS[1].conv[0], 1024, synth.PRIMES_CFG1, 2),
    (synth.ConvLayer(5, 7, 6, 5), 1024, None, 3),
    (synth.ConvLayer(40, 70, 4, 4), 1024, None, 2),       # n_ib = 3, n_ob = 5
    (synth.CONFIGS[2].conv[0], 8192, synth.PRIMES_N8192[:2], 1),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-N{c[1]}")
def test_cpu_ntt_baseline_equals_oracle(case):
    Ly, N, primes, B = case
    primes = list(primes) if primes else R.find_primes(N, 50, 2)
    ring = R.Ring(N, primes, 65537)
    plan = R.plan_conv(Ly, N)
    rng = np.random.default_rng(N + B)
    W = rng.integers(-8, 8, (Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h))
    c0 = synth.uniform_residues((B, plan.n_ib, ring.L, N), primes, 3, "c0", B)
    phi = synth.phi1((B, plan.n_ob, N), 65537, 3, B)
    f = CB.prepare_filters(W, plan, ring)
    assert np.array_equal(CB.conv_server(c0, f, plan, ring, phi),
                          R.conv_server(c0, W, plan, ring, phi))
