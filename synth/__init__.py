"""Seeded synthetic workloads shared by the oracle tests, smoke() and bench.py.

This module holds ONLY shapes, ring parameters (as data) and seeded random
draws.  It contains none of the method's arithmetic (no packing, encoding,
NTT or modular products): both the CUDA path and the oracle consume what it
returns, and neither imports the other.

Workloads follow BASELINE.json "configs" (the five plain-20-shaped cases);
the recipe is restated in DESIGN.md ("Input recipe").  CIFAR images and
trained plain-20 weights are not available, and the server computation is
value-independent, so uniform integers of the stated ranges stand in for
them ("Synthetic inputs").

Random numbers the method draws (secret key, v, e0, a, flooding noise,
mask phi1) are drawn here and passed in as inputs (task rule ③).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Tuple

import numpy as np

# --------------------------------------------------------------------------
# Ring parameters (data).  R8 reading: the largest primes below
# 2^50 (config 1: below 2^30) with q = 1 mod 2N, in descending order.  Both
# the oracle (oracle/ref.py:find_primes) and the product context
# (he_ctx_create) re-check primality and q = 1 mod 2N independently; a
# not-gpu test re-derives this table from the oracle's own search.
# --------------------------------------------------------------------------
PRIMES_CFG1 = [1073707009]
PRIMES_N8192 = [1125899906826241, 1125899906629633, 1125899905744897,
                1125899905351681]
PRIMES_N16384 = [1125899904679937, 1125899903991809, 1125899903827969,
                 1125899903795201, 1125899903500289, 1125899903107073]
PRIMES_N32768 = [1125899904679937, 1125899903827969, 1125899903500289,
                 1125899903107073, 1125899902124033, 1125899901665281,
                 1125899899174913, 1125899896160257, 1125899887312897,
                 1125899886395393, 1125899885740033, 1125899885412353]

T_PLAIN = 65537  # plaintext modulus t (BASELINE.json configs[0]; R21)


@dataclasses.dataclass(frozen=True)
class ConvLayer:
    """One Conv layer in the paper's notation (§II-B).

    w_i = number of image rows, h_i = row length (the paper's i^{(m)} uses
    X^{(k-f_w)h_i+l}: k < w_i indexes rows, h_i is the row pitch);
    f_w = filter rows, f_h = filter columns.  pad = 1 means "same" padding
    (client zero-pads (f-1)/2 on each side, R10), pad = 0 means valid.
    """
    c_i: int
    c_o: int
    w_i: int
    h_i: int
    f_w: int = 3
    f_h: int = 3
    stride: int = 1
    pad: int = 1


@dataclasses.dataclass(frozen=True)
class FcLayer:
    """FC layer with n_i inputs and n_o outputs."""
    n_i: int
    n_o: int


@dataclasses.dataclass(frozen=True)
class Config:
    idx: int
    name: str
    N: int
    primes: Tuple[int, ...]
    t: int
    B: int
    conv: Tuple[ConvLayer, ...]
    fc: Optional[FcLayer]
    img_lo: int
    img_hi: int       # inclusive
    w_lo: int
    w_hi: int         # inclusive
    sigma: float = 3.2
    h: int = 64       # secret-key Hamming weight (R4)
    seed: int = 0

    @property
    def L(self) -> int:
        return len(self.primes)

    @property
    def log2N(self) -> int:
        return self.N.bit_length() - 1


def _plain20_layers() -> Tuple[ConvLayer, ...]:
    """plain-20 (f3-d20-w1): 19 3x3 convs, no residuals."""
    L = [ConvLayer(3, 16, 32, 32)]
    L += [ConvLayer(16, 16, 32, 32) for _ in range(6)]
    L += [ConvLayer(16, 32, 32, 32, stride=2)]
    L += [ConvLayer(32, 32, 16, 16) for _ in range(5)]
    L += [ConvLayer(32, 64, 16, 16, stride=2)]
    L += [ConvLayer(64, 64, 8, 8) for _ in range(5)]
    assert len(L) == 19
    return tuple(L)


CONFIGS = {
    1: Config(1, "tiny_conv", 1024, tuple(PRIMES_CFG1), T_PLAIN, 1,
              (ConvLayer(1, 2, 8, 8),), None, 0, 15, -4, 3, seed=101),
    2: Config(2, "cifar_conv1", 8192, tuple(PRIMES_N8192[:3]), T_PLAIN, 1,
              (ConvLayer(3, 16, 32, 32),), None, 0, 255, -8, 7, seed=202),
    3: Config(3, "plain20_mid", 8192, tuple(PRIMES_N8192[:4]), T_PLAIN, 64,
              (ConvLayer(32, 32, 16, 16),), None, 0, 255, -8, 7, seed=303),
    4: Config(4, "plain20_stack", 16384, tuple(PRIMES_N16384), T_PLAIN, 32,
              _plain20_layers(), FcLayer(64, 100), 0, 255, -8, 7, seed=404),
    5: Config(5, "plain20_s3_sweep", 32768, tuple(PRIMES_N32768), T_PLAIN,
              256, (ConvLayer(64, 64, 8, 8),), None, 0, 255, -8, 7,
              seed=505),
}


# --------------------------------------------------------------------------
# Seeded streams (R26): one base seed per config, one sub-stream per tensor
# identified by a fixed tag and integer indices.
# --------------------------------------------------------------------------
_TAGS = {"img": 1, "w": 2, "c0": 3, "phi1": 4, "sk": 5, "v": 6, "e0": 7,
         "a": 8, "ef": 9, "fc_w": 10, "fc_b": 11, "fc_in": 12, "ve": 13,
         "misc": 99}


def rng(seed: int, tag: str, *idx: int) -> np.random.Generator:
    return np.random.Generator(
        np.random.PCG64(np.random.SeedSequence([seed, _TAGS[tag], *idx])))


def images(cfg: Config, layer: int, B: Optional[int] = None,
           shard: int = 0) -> np.ndarray:
    """int32 [B][c_i][w_i][h_i], uniform in [img_lo, img_hi]."""
    Ly = cfg.conv[layer]
    B = cfg.B if B is None else B
    g = rng(cfg.seed, "img", layer, shard)
    return g.integers(cfg.img_lo, cfg.img_hi + 1,
                      size=(B, Ly.c_i, Ly.w_i, Ly.h_i), dtype=np.int32)


def weights(cfg: Config, layer: int) -> np.ndarray:
    """int32 [c_o][c_i][f_w][f_h], uniform in [w_lo, w_hi]."""
    Ly = cfg.conv[layer]
    g = rng(cfg.seed, "w", layer)
    return g.integers(cfg.w_lo, cfg.w_hi + 1,
                      size=(Ly.c_o, Ly.c_i, Ly.f_w, Ly.f_h), dtype=np.int32)


def uniform_residues(shape, primes, seed: int, tag: str = "c0",
                     *idx: int) -> np.ndarray:
    """uint64 [..., L, N]: independent uniform residues in [0, q_j) per limb.

    `shape` is the full shape including the L axis at position -2.  Used
    for synthetic c0 (R23: RLWE c0 is pseudorandom and the server function
    does not inspect values) and for the public polynomial a (R7).
    """
    shape = tuple(shape)
    L = len(primes)
    assert shape[-2] == L
    g = rng(seed, tag, *idx)
    out = np.empty(shape, dtype=np.uint64)
    for j, q in enumerate(primes):
        out[..., j, :] = g.integers(0, q, size=shape[:-2] + shape[-1:],
                                    dtype=np.uint64)
    return out


def phi1(shape, t: int, seed: int, *idx: int) -> np.ndarray:
    """uint32 mask values uniform in [0, t) (R15)."""
    g = rng(seed, "phi1", *idx)
    return g.integers(0, t, size=tuple(shape), dtype=np.uint32)


def fc_weights(cfg: Config) -> np.ndarray:
    """int32 [n_o][n_i] in [w_lo, w_hi] (W is n_o x n_i)."""
    g = rng(cfg.seed, "fc_w")
    return g.integers(cfg.w_lo, cfg.w_hi + 1, size=(cfg.fc.n_o, cfg.fc.n_i),
                      dtype=np.int32)


def fc_bias(cfg: Config) -> np.ndarray:
    """int32 [n_o] in [w_lo, w_hi] (R18)."""
    g = rng(cfg.seed, "fc_b")
    return g.integers(cfg.w_lo, cfg.w_hi + 1, size=(cfg.fc.n_o,),
                      dtype=np.int32)


def fc_inputs(cfg: Config, B: Optional[int] = None) -> np.ndarray:
    """int32 [B][n_i] in [img_lo, img_hi] (R22)."""
    B = cfg.B if B is None else B
    g = rng(cfg.seed, "fc_in")
    return g.integers(cfg.img_lo, cfg.img_hi + 1, size=(B, cfg.fc.n_i),
                      dtype=np.int32)


# ---- client-side randomness (oracle protocol tests only) -----------------
def secret_key(N: int, h: int, seed: int) -> np.ndarray:
    """int64 [N] sparse ternary, Hamming weight h, uniform positions/signs
    (R4)."""
    g = rng(seed, "sk")
    s = np.zeros(N, dtype=np.int64)
    pos = g.choice(N, size=h, replace=False)
    s[pos] = g.choice(np.array([-1, 1], dtype=np.int64), size=h)
    return s


def v_poly(N: int, seed: int, *idx: int) -> np.ndarray:
    """int64 [N], P(0)=1/2, P(+-1)=1/4."""
    g = rng(seed, "v", *idx)
    u = g.integers(0, 4, size=N)
    return np.where(u < 2, 0, np.where(u == 2, 1, -1)).astype(np.int64)


def gauss_poly(N: int, sigma: float, seed: int, tag: str,
               *idx: int) -> np.ndarray:
    """int64 [N], round(N(0, sigma^2)) (R5; no tail cut)."""
    g = rng(seed, tag, *idx)
    return np.rint(g.normal(0.0, sigma, size=N)).astype(np.int64)


def conv_layers(cfg: Config) -> List[ConvLayer]:
    return list(cfg.conv)
