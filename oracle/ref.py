"""Plain CPU oracle for the rotation-free HE Conv/FC path (arXiv 2409.05205).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module.
It shares no code with the CUDA path (paper_2409_05205_b200/) and the CUDA
path never imports it.  Inputs come from synth/ (seeded draws only).

Everything here is the plain definition of what the method computes, in the
paper's order and notation, with Python integers (exact) or the companion C
library he_oracle.c (unsigned __int128) for the heavy sums.  Citations are
PAPER.md line numbers with the section / equation / algorithm; readings
R1..R26 are listed in DESIGN.md.

Pins (tests/test_oracle_*.py, -m "not gpu"), function by function -- each
function below is checked against something other than itself:
  is_prime / find_primes / min_psi   test_oracle_ring: SURVEY App. A prime
        values; q = 1 mod 2N; psi^N = -1 and psi of order exactly 2N.
  encode / encode_bigint             test_oracle_ring: C encoding == literal
        big-integer round(Q m / t); centred-remainder identity.
  schoolbook_py / negacyclic_at / sparse_mul (+ reduce_exp, to_residues)
        test_oracle_ring: three independent product paths agree;
        X^{N-1} X = -1 (golden SPEC.md:61).
  ntt_def / intt_def / ntt_def_py    test_oracle_ring: INTT(NTT(a)) = a;
        NTT(delta_0) = 1; convolution theorem vs schoolbook.
  incomplete_ntt_def (+ reduce_mod_binomial)  test_oracle_ring: the reduction
        mod X^s - zeta_g by long division; fold identity.
  plan_conv / pack_input_int / filter_poly_int (+ pad_image, filter_terms)
        test_oracle_packing: integer-mode product equals the brute-force
        Eq. (3)/(4) conv (conv2d_ref) on 8 shapes; golden SPEC.md:266/284/285.
  conv2d_ref                         test_oracle_packing: golden SPEC.md:648.
  output_positions / conv_server / compact   test_oracle_protocol:
        decryption - phi1 == brute-force conv mod t (configs 1-2).
  fc_input_int / fc_weight_terms / fc_weight_eq10_literal / fc_server
        test_oracle_packing: Theorem 1 exhaustive; golden SPEC.md:416/430;
        protocol decrypts to W I + B.
  plan_fc / fc_input_blocks / fc_server_tiled (+ fc_submatrix)
        test_oracle_protocol: trivial-key decryption == W I + B.
  keygen / encrypt_c0 / crt_decode / conv_protocol_decrypt /
  fc_protocol_decrypt / centered_mod_t / server_p / client_c1r /
  decrypt_round                      test_oracle_protocol / test_oracle_ring:
        full protocol recovers the brute-force conv / FC mod t; CRT by
        exact big integers.
  splitmix64_py / phi1_stream        test_oracle_ring: Vigna's published
        SplitMix64 reference value.
  mod_switch                         test_oracle_protocol: exact rationals.
  multi_image_spacing / shift_negacyclic / pack_input_multi_int /
  output_positions_multi / compact_multi   test_oracle_multi: integer-mode
        products equal every image's brute-force conv at its shifted slots
        (and one row less of spacing breaks it); a trivially encrypted
        multi-image ciphertext through conv_server decrypts to every
        image's conv mod t.
  relu_requant / avgpool             test_oracle_stub: hand-computed golden
        values (tests/golden/r29_stub.json); ReLU == PAPER.md:86's
        (X + sign(X) X) / 2.
  plain_chain                        test_oracle_protocol: the encrypted
        protocol chain equals it layer by layer.
No oracle function is unpinned.  GPU ciphertext residues are pinned through
these identities; no ciphertext value is printed in the paper.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "he_oracle.c")


# ---------------------------------------------------------------------------
# C helper library (built with gcc; plain C, OpenMP).
# ---------------------------------------------------------------------------
def build_lib(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared",
                               "-o", _LIB_PATH, _SRC])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_lib()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i32, i64, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        L.orc_negacyclic_at.argtypes = [P, P, i32, u64, P, i32, P]
        L.orc_sparse_mul.argtypes = [P, i32, u64, P, P, i32, P]
        L.orc_encode.argtypes = [P, i64, u64, u64, u64, u64, P]
        L.orc_conv_server.argtypes = [P, i32, i32, i32, i32, P, i32, i32, i32,
                                      i32, P, P, P, P, P, P, u64, u64, P]
        L.orc_fc_server.argtypes = [P, i32, i32, i32, P, i32, P, P, i32, P, P,
                                    P, u64, u64, P]
        L.orc_ntt_def.argtypes = [P, i32, u64, u64, P, i32, P]
        L.orc_intt_def.argtypes = [P, i32, u64, u64, P]
        L.orc_powmod.argtypes = [u64, u64, u64]
        L.orc_powmod.restype = u64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


# ---------------------------------------------------------------------------
# Number theory for the RNS ring (§II-A: R_Q = Z_Q[X]/(X^N+1);
# PAPER.md:28 §I: CRT / NTT).  Readings R8, R9.
# ---------------------------------------------------------------------------
def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin (bases up to 37: exact below 3.3e24)."""
    if n < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37]
    for p in small:
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def find_primes(N: int, bits: int, count: int) -> List[int]:
    """R8: the `count` largest primes q < 2^bits with q = 1 (mod 2N)."""
    out = []
    q = ((2 ** bits - 1) // (2 * N)) * (2 * N) + 1
    while q >= 2 ** bits:
        q -= 2 * N
    while len(out) < count:
        if is_prime(q):
            out.append(q)
        q -= 2 * N
    return out


def min_psi(q: int, N: int) -> int:
    """R9: the smallest primitive 2N-th root of unity mod q.

    Any x with x^N = -1 has order exactly 2N (N a power of two).  Find one
    from a generator candidate, then take the minimum over its N odd powers
    (all primitive 2N-th roots)."""
    assert (q - 1) % (2 * N) == 0
    g = 2
    while True:
        x = pow(g, (q - 1) // (2 * N), q)
        if pow(x, N, q) == q - 1:
            break
        g += 1
    best, x2, cur = x, x * x % q, x
    for _ in range(N - 1):
        cur = cur * x2 % q
        best = min(best, cur)
    return best


@dataclasses.dataclass
class Ring:
    N: int
    primes: Tuple[int, ...]
    t: int

    def __post_init__(self):
        self.Q = 1
        for q in self.primes:
            self.Q *= q
        self.delta = self.Q // self.t            # Delta_t = floor(Q/t)  (R2)
        self.r_t = self.Q % self.t               # r_t = Q mod t          (R2)
        self.delta_mod_q = np.array([self.delta % q for q in self.primes],
                                    dtype=np.uint64)
        self.q_arr = np.array(self.primes, dtype=np.uint64)

    @property
    def L(self):
        return len(self.primes)


def encode_bigint(m: Sequence[int], ring: Ring) -> np.ndarray:
    """Literal R2 definition, big integers: enc_j(m) = round(Q*(m mod t)/t)
    mod q_j.  No ties since t is odd.  Returns uint64 [L][len(m)]."""
    out = np.zeros((ring.L, len(m)), dtype=np.uint64)
    for i, mv in enumerate(m):
        mt = int(mv) % ring.t
        v = (2 * ring.Q * mt + ring.t) // (2 * ring.t)   # round(Q*mt/t)
        for j, q in enumerate(ring.primes):
            out[j, i] = v % q
    return out


def encode(m: np.ndarray, ring: Ring) -> np.ndarray:
    """R2 via he_oracle.c orc_encode (checked against encode_bigint).
    m: uint32 [...]; returns uint64 [L][...]."""
    m = np.ascontiguousarray(m, dtype=np.uint32)
    out = np.empty((ring.L,) + m.shape, dtype=np.uint64)
    for j, q in enumerate(ring.primes):
        o = np.empty(m.shape, dtype=np.uint64)
        lib().orc_encode(_p(m), m.size, q, int(ring.delta_mod_q[j]), ring.r_t,
                         ring.t, _p(o))
        out[j] = o
    return out


# ---------------------------------------------------------------------------
# Negacyclic products (§II-A).
# ---------------------------------------------------------------------------
def schoolbook_py(a: Sequence[int], b: Sequence[int], N: int,
                  q: Optional[int] = None) -> List[int]:
    """c_k = sum_{i+j=k} a_i b_j - sum_{i+j=k+N} a_i b_j (exact Python ints,
    optionally reduced mod q).  Small N only."""
    c = [0] * N
    for i in range(N):
        ai = int(a[i])
        if ai == 0:
            continue
        for j in range(N):
            k = i + j
            if k < N:
                c[k] += ai * int(b[j])
            else:
                c[k - N] -= ai * int(b[j])
    if q is not None:
        c = [x % q for x in c]
    return c


def negacyclic_at(a: np.ndarray, b: np.ndarray, q: int,
                  pos: Optional[np.ndarray] = None) -> np.ndarray:
    """Coefficients `pos` of a*b mod (X^N+1, q) by the definition (C)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    N = a.shape[-1]
    if pos is None:
        out = np.empty(N, dtype=np.uint64)
        lib().orc_negacyclic_at(_p(a), _p(b), N, q, None, 0, _p(out))
    else:
        pos = np.ascontiguousarray(pos, dtype=np.int32)
        out = np.empty(pos.size, dtype=np.uint64)
        lib().orc_negacyclic_at(_p(a), _p(b), N, q, _p(pos), pos.size,
                                _p(out))
    return out


def sparse_mul(a: np.ndarray, terms: Sequence[Tuple[int, int]], q: int
               ) -> np.ndarray:
    """a * (sum w X^e) mod (X^N+1, q), terms reduced to 0 <= e < N."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    N = a.shape[-1]
    e = np.array([t[0] for t in terms], dtype=np.int32)
    w = np.array([t[1] for t in terms], dtype=np.int64)
    out = np.empty(N, dtype=np.uint64)
    lib().orc_sparse_mul(_p(a), N, q, _p(e), _p(w), len(terms), _p(out))
    return out


def reduce_exp(e: int, N: int) -> Tuple[int, int]:
    """X^e in Z[X]/(X^N+1): returns (e', sign) with 0 <= e' < N.
    X^N = -1."""
    sign = 1
    while e < 0:
        e += N
        sign = -sign
    while e >= N:
        e -= N
        sign = -sign
    return e, sign


def to_residues(c: Sequence[int], q: int) -> np.ndarray:
    return np.array([int(x) % q for x in c], dtype=np.uint64)


# ---------------------------------------------------------------------------
# Definitional negacyclic NTT (R9): A[k] = a(psi^{2k+1}), natural order k.
# ---------------------------------------------------------------------------
def ntt_def(a: np.ndarray, q: int, psi: int,
            ks: Optional[np.ndarray] = None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    N = a.shape[-1]
    ks = np.arange(N, dtype=np.int32) if ks is None else \
        np.ascontiguousarray(ks, dtype=np.int32)
    out = np.empty(ks.size, dtype=np.uint64)
    lib().orc_ntt_def(_p(a), N, q, psi, _p(ks), ks.size, _p(out))
    return out


def intt_def(A: np.ndarray, q: int, psi: int) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.uint64)
    N = A.shape[-1]
    out = np.empty(N, dtype=np.uint64)
    lib().orc_intt_def(_p(A), N, q, psi, _p(out))
    return out


def ntt_def_py(a: Sequence[int], q: int, psi: int) -> List[int]:
    """Pure-Python definition, tiny N (pins the C routine)."""
    N = len(a)
    return [sum(int(a[i]) * pow(psi, (2 * k + 1) * i, q) for i in range(N)) % q
            for k in range(N)]


# ---------------------------------------------------------------------------
# Conv layer: plan (R11), packing (Eq. 5, 6, 7), brute force (Eq. 3, 4).
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class ConvPlan:
    c_i: int
    c_o: int
    w_i: int
    h_i: int
    f_w: int
    f_h: int
    stride: int
    pad: int
    N: int
    s: int
    c_ib: int
    n_ib: int
    c_ob: int
    n_ob: int
    w_p: int
    h_p: int
    w_o: int
    h_o: int

    @property
    def step(self) -> int:          # offset spacing of t_n (R11)
        return self.s // self.c_ob

    def t_n(self, n: int) -> int:   # Eq. (7) shift n*c_i/c_o, generalised
        return (n % self.c_ob) * self.step

    @property
    def n_valid(self) -> int:       # compact entries per output block (a8)
        return self.c_ob * self.w_o * self.h_o


def plan_conv(layer, N: int, s_override: int = 0) -> ConvPlan:
    """R11: s = largest power of two with s*w_p*h_p <= N (paper: s = c_i,
    PAPER.md:121 "N = max(w_i h_i s, f_w f_h s)", s >= c_i); input / output
    channel blocks c_ib = min(c_i, s), c_ob = min(c_o, s).
    Output size: w_o = floor((w_p - f_w + 1)/stride)."""
    padw = (layer.f_w - 1) // 2 if layer.pad else 0
    padh = (layer.f_h - 1) // 2 if layer.pad else 0
    w_p, h_p = layer.w_i + 2 * padw, layer.h_i + 2 * padh
    if w_p * h_p > N:
        raise ValueError("image does not fit the ring")
    if s_override:
        s = s_override
        if s & (s - 1) or s * w_p * h_p > N:
            raise ValueError("illegal s_override")
    else:
        s = 1
        while 2 * s * w_p * h_p <= N:
            s *= 2
    c_ib, c_ob = min(layer.c_i, s), min(layer.c_o, s)
    w_o = (w_p - layer.f_w + 1) // layer.stride
    h_o = (h_p - layer.f_h + 1) // layer.stride
    return ConvPlan(layer.c_i, layer.c_o, layer.w_i, layer.h_i, layer.f_w,
                    layer.f_h, layer.stride, layer.pad, N, s, c_ib,
                    -(-layer.c_i // c_ib), c_ob, -(-layer.c_o // c_ob),
                    w_p, h_p, w_o, h_o)


def pad_image(img: np.ndarray, plan: ConvPlan) -> np.ndarray:
    """R10 "same" padding: zeros around each channel.  img [c][w_i][h_i]."""
    pw, ph = (plan.w_p - plan.w_i) // 2, (plan.h_p - plan.h_i) // 2
    out = np.zeros((img.shape[0], plan.w_p, plan.h_p), dtype=np.int64)
    out[:, pw:pw + plan.w_i, ph:ph + plan.h_i] = img
    return out


def conv2d_ref(img: np.ndarray, W: np.ndarray, plan: ConvPlan) -> np.ndarray:
    """Eq. (3)/(4) by direct loops on the padded image:
    out[n][k][l] = sum_m sum_{k',l'} F^{(m,n)}_{k',l'} I^{(m)}_{sk+k', sl+l'}.
    img [c_i][w_i][h_i], W [c_o][c_i][f_w][f_h] -> int64 [c_o][w_o][h_o]."""
    Ip = pad_image(img, plan)
    out = np.zeros((plan.c_o, plan.w_o, plan.h_o), dtype=np.int64)
    S = plan.stride
    for n in range(plan.c_o):
        for k in range(plan.w_o):
            for l in range(plan.h_o):
                acc = 0
                for m in range(plan.c_i):
                    for kk in range(plan.f_w):
                        for ll in range(plan.f_h):
                            acc += int(W[n, m, kk, ll]) * \
                                int(Ip[m, S * k + kk, S * l + ll])
                out[n, k, l] = acc
    return out


def pack_input_int(img: np.ndarray, plan: ConvPlan) -> np.ndarray:
    """Eq. (5) with the s-embedding, padded row pitch h_p
    and input-channel blocks (R10, R11, R13):
      i_beta(X) = sum_{m<c_ib} sum_{k<w_p, l<h_p} Ip^{(beta c_ib+m)}_{k,l}
                  X^{s((k-f_w)h_p + l) + m}        (mod X^N + 1)
    Returns int64 [n_ib][N] (exact integers, negacyclic signs applied)."""
    Ip = pad_image(img, plan)
    N, s = plan.N, plan.s
    out = np.zeros((plan.n_ib, N), dtype=np.int64)
    for beta in range(plan.n_ib):
        for m in range(plan.c_ib):
            ch = beta * plan.c_ib + m
            if ch >= plan.c_i:
                break
            for k in range(plan.w_p):
                for l in range(plan.h_p):
                    v = int(Ip[ch, k, l])
                    if v == 0:
                        continue
                    e, sg = reduce_exp(s * ((k - plan.f_w) * plan.h_p + l) + m,
                                       N)
                    out[beta, e] += sg * v
    return out


def filter_terms(W: np.ndarray, plan: ConvPlan, n: int, beta: int,
                 shifted: bool = True) -> List[Tuple[int, int]]:
    """Eq. (6) with the s-embedding and blocks, and Eq. (7)
     shift X^{t_n} when `shifted`:
      fhat_beta^{(n)}(X) = X^{t_n} sum_{m<c_ib} sum_{k<f_w,l<f_h}
                 F^{(beta c_ib+m, n)}_{k,l} X^{s(h_p f_w - (k h_p + l)) - m}
    Returns the sparse polynomial as [(exponent in [0,N), signed weight)]
    with like exponents merged."""
    N, s = plan.N, plan.s
    acc: Dict[int, int] = {}
    tn = plan.t_n(n) if shifted else 0
    for m in range(plan.c_ib):
        ch = beta * plan.c_ib + m
        if ch >= plan.c_i:
            break
        for k in range(plan.f_w):
            for l in range(plan.f_h):
                w = int(W[n, ch, k, l])
                if w == 0:
                    continue
                e, sg = reduce_exp(s * (plan.h_p * plan.f_w - (k * plan.h_p + l))
                                   - m + tn, N)
                acc[e] = acc.get(e, 0) + sg * w
    return sorted((e, w) for e, w in acc.items() if w != 0)


def filter_poly_int(W, plan, n, beta, shifted=True) -> np.ndarray:
    out = np.zeros(plan.N, dtype=np.int64)
    for e, w in filter_terms(W, plan, n, beta, shifted):
        out[e] += w
    return out


def output_positions(plan: ConvPlan) -> np.ndarray:
    """Valid-slot positions of one output block, in increasing order (R16):
    i = s*(stride*K*h_p + stride*L) + t_n, K < w_o, L < h_o, n in block
    ("valid coefficients ... locate in slots k c_i + n c_i/c_o").
    int64 [c_ob * w_o * h_o], ordered (K, L, n)."""
    s, S = plan.s, plan.stride
    pos = []
    for K in range(plan.w_o):
        for L in range(plan.h_o):
            base = s * (S * K * plan.h_p + S * L)
            for nl in range(plan.c_ob):
                pos.append(base + nl * plan.step)
    return np.array(pos, dtype=np.int64)


# ---------------------------------------------------------------------------
# Server side (the path under test).
# ---------------------------------------------------------------------------
def _conv_terms(W: np.ndarray, plan: ConvPlan):
    offs, tb, te, tw = [0], [], [], []
    for n in range(plan.c_o):
        for beta in range(plan.n_ib):
            for e, w in filter_terms(W, plan, n, beta, shifted=True):
                tb.append(beta)
                te.append(e)
                tw.append(w)
        offs.append(len(te))
    return (np.array(offs, np.int32), np.array(tb, np.int32),
            np.array(te, np.int32), np.array(tw, np.int64))


def conv_server(c0: np.ndarray, W: np.ndarray, plan: ConvPlan, ring: Ring,
                phi1: Optional[np.ndarray] = None) -> np.ndarray:
    """Algorithm 1 server side + mask.

    c0: uint64 [B][n_ib][L][N] canonical residues; W: int [c_o][c_i][f_w][f_h]
    phi1: uint32 [B][n_ob][N] in [0,t) or None.
    Returns the full c0^r: uint64 [B][n_ob][L][N] (R14: positions s*j + t_n
    for all j, 0 elsewhere, then + enc(phi1) everywhere)."""
    c0 = np.ascontiguousarray(c0, dtype=np.uint64)
    B = c0.shape[0]
    assert c0.shape == (B, plan.n_ib, ring.L, plan.N)
    offs, tb, te, tw = _conv_terms(W, plan)
    out = np.empty((B, plan.n_ob, ring.L, plan.N), dtype=np.uint64)
    ph = None if phi1 is None else np.ascontiguousarray(phi1, dtype=np.uint32)
    if ph is not None:
        assert ph.shape == (B, plan.n_ob, plan.N)
    lib().orc_conv_server(_p(c0), B, plan.n_ib, ring.L, plan.N, _p(ring.q_arr),
                          plan.s, plan.c_o, plan.c_ob, plan.n_ob, _p(offs),
                          _p(tb), _p(te), _p(tw), _p(ph),
                          _p(ring.delta_mod_q), ring.r_t, ring.t, _p(out))
    return out


def compact(out_full: np.ndarray, plan: ConvPlan) -> np.ndarray:
    """a8: gather the valid slots ("do not need to be sent").
    [B][n_ob][L][N] -> [B][n_ob][L][n_valid]."""
    return np.ascontiguousarray(out_full[..., output_positions(plan)])


# ---------------------------------------------------------------------------
# Multi-image packing (reading R31 -- a protocol
# extension beyond the paper, which keeps one image per ciphertext,
# PAPER.md:304).  P images share one input ciphertext at offsets p*D:
#   c(X) = sum_{p<P} X^{p D} i_p(X)   (mod X^N + 1),
# with i_p the Eq. (5) packing of image p.  The server's product with the
# unchanged Eq. (6)/(7) filters is linear, so image p's conv outputs appear
# at p*D + (the single-image valid slots) provided no other image's product
# reaches them.  Counting only the image's nonzero (unpadded) pixels, the
# product i_p f (with the Eq. (7) shift t_n < s) has exponents in [lo, hi],
# and image p's valid slots lie in [0, v_hi].  The spacing
#   D = the least multiple of s with D > hi and D + lo > v_hi,  P = floor(N/D)
# makes the neighbour below end before p*D and the one above start after the
# valid slots, and (P*D <= N) the lowest image's negative exponents wrap
# (negacyclic) above the top image's slots, so every slot is exactly image
# p's.  D is a multiple of s because the server computes slots s*j + t_n.
# ---------------------------------------------------------------------------
def multi_image_spacing(plan: ConvPlan) -> Tuple[int, int]:
    """(D, P): image spacing and images per ciphertext (R31)."""
    s, hp = plan.s, plan.h_p
    pw, ph = (plan.w_p - plan.w_i) // 2, (plan.h_p - plan.h_i) // 2
    # Eq. (5) exponents of the nonzero pixels, Eq. (6) exponents (+ t_n < s)
    in_lo = s * ((pw - plan.f_w) * hp + ph)
    in_hi = s * ((pw + plan.w_i - 1 - plan.f_w) * hp + ph + plan.h_i - 1) + plan.c_ib - 1
    f_lo = s * (hp - plan.f_h + 1) - (plan.c_ib - 1)
    f_hi = s * hp * plan.f_w + (s - 1)
    lo, hi = in_lo + f_lo, in_hi + f_hi
    S = plan.stride
    v_hi = s * (S * (plan.w_o - 1) * hp + S * (plan.h_o - 1)) + s - 1
    D = max(hi + 1, v_hi - lo + 1)
    D = -(-D // s) * s
    return D, plan.N // D


def shift_negacyclic(a: np.ndarray, k: int) -> np.ndarray:
    """X^k a(X) mod X^N + 1 for integer coefficient vectors (last axis)."""
    N = a.shape[-1]
    out = np.zeros_like(a)
    for e in range(N):
        f, sg = reduce_exp(e + k, N)
        out[..., f] += sg * a[..., e]
    return out


def pack_input_multi_int(imgs: np.ndarray, plan: ConvPlan, D: int) -> np.ndarray:
    """imgs [P][c_i][w_i][h_i] -> int64 [n_ib][N] = sum_p X^{p D} i_p(X)."""
    out = np.zeros((plan.n_ib, plan.N), dtype=np.int64)
    for p in range(imgs.shape[0]):
        out += shift_negacyclic(pack_input_int(imgs[p], plan), p * D)
    return out


def output_positions_multi(plan: ConvPlan, P: int, D: int) -> np.ndarray:
    """Valid slots of P images sharing a ciphertext: image p's single-image
    slots shifted by p*D (all below N for P*D <= N), image-major order."""
    pos = output_positions(plan)
    allp = np.concatenate([p * D + pos for p in range(P)])
    assert allp.max() < plan.N
    return allp


def compact_multi(out_full: np.ndarray, plan: ConvPlan, P: int, D: int) -> np.ndarray:
    """a8 for multi-image ciphertexts: [B][n_ob][L][N] -> [B][n_ob][L][P n_valid]."""
    return np.ascontiguousarray(out_full[..., output_positions_multi(plan, P, D)])


# ---------------------------------------------------------------------------
# FC layer: Eq. (9), Eq. (10) / R17, Theorem 1, Algorithm 2.
# ---------------------------------------------------------------------------
def fc_input_int(I: np.ndarray, n_o: int, N: int) -> np.ndarray:
    """Eq. (9): i(X) = sum_l I_l X^{l n_o}.  int64 [N]."""
    n_i = I.shape[0]
    assert n_i * n_o <= N
    out = np.zeros(N, dtype=np.int64)
    for l in range(n_i):
        out[l * n_o] = int(I[l])
    return out


def fc_weight_terms(W: np.ndarray, N: int) -> List[Tuple[int, int]]:
    """R17 generalisation of Eq. (10) valid for N >= n_i n_o:
      w(X) = sum_k W_{k,0} X^k - sum_{l>=1} sum_k W_{k,l} X^{N - l n_o + k}.
    At N = n_i n_o this is exactly Eq. (10) (substitute l -> n_i - l)."""
    n_o, n_i = W.shape
    assert n_i * n_o <= N
    terms = []
    for k in range(n_o):
        if W[k, 0]:
            terms.append((k, int(W[k, 0])))
    for l in range(1, n_i):
        for k in range(n_o):
            if W[k, l]:
                terms.append((N - l * n_o + k, -int(W[k, l])))
    return sorted(terms)


def fc_weight_eq10_literal(W: np.ndarray) -> np.ndarray:
    """Eq. (10) exactly as printed (N = n_i n_o):
      w(X) = sum_k W_{k,0} X^k - sum_k sum_{l=1}^{n_i-1} W_{k,n_i-l} X^{l n_o+k}."""
    n_o, n_i = W.shape
    N = n_i * n_o
    out = np.zeros(N, dtype=np.int64)
    for k in range(n_o):
        out[k] += int(W[k, 0])
        for l in range(1, n_i):
            out[l * n_o + k] -= int(W[k, n_i - l])
    return out


def fc_server(c0: np.ndarray, W: np.ndarray, bias: Optional[np.ndarray],
              ring: Ring, phi1: Optional[np.ndarray] = None) -> np.ndarray:
    """Algorithm 2 Line 13: c0^r = c0*w + b, first n_o
    coefficients only, plus enc(phi1).
    c0 uint64 [B][L][N]; returns uint64 [B][L][n_o]."""
    c0 = np.ascontiguousarray(c0, dtype=np.uint64)
    B, L, N = c0.shape
    n_o = W.shape[0]
    terms = fc_weight_terms(W, N)
    te = np.array([t[0] for t in terms], np.int32)
    tw = np.array([t[1] for t in terms], np.int64)
    bm = None if bias is None else \
        np.ascontiguousarray(np.asarray(bias, np.int64) % ring.t, np.uint32)
    ph = None if phi1 is None else np.ascontiguousarray(phi1, np.uint32)
    out = np.empty((B, L, n_o), dtype=np.uint64)
    lib().orc_fc_server(_p(c0), B, L, N, _p(ring.q_arr), n_o, _p(te), _p(tw),
                        len(terms), _p(bm), _p(ph), _p(ring.delta_mod_q),
                        ring.r_t, ring.t, _p(out))
    return out


# ---------------------------------------------------------------------------
# Client side of Algorithms 1 and 2 (oracle only; used to pin the server
# output by decryption).  Eq. (1), Eq. (2) in the BFV reading (R1).
# ---------------------------------------------------------------------------
def signed_to_residues(x: np.ndarray, ring: Ring) -> np.ndarray:
    """int64 [..., N] -> uint64 [..., L, N] (x mod q_j)."""
    x = np.asarray(x, dtype=np.int64)
    out = np.empty(x.shape[:-1] + (ring.L, x.shape[-1]), dtype=np.uint64)
    for j, q in enumerate(ring.primes):
        out[..., j, :] = np.mod(x, q).astype(np.uint64)
    return out


def keygen(ring: Ring, s_key: np.ndarray, a: np.ndarray, e: np.ndarray):
    """pk = (b, a), b = -a s + e mod Q.  a [L][N] uniform."""
    s_res = signed_to_residues(s_key, ring)
    e_res = signed_to_residues(e, ring)
    b = np.empty_like(a)
    for j, q in enumerate(ring.primes):
        as_ = negacyclic_at(a[j], s_res[j], q)
        b[j] = (np.asarray(e_res[j], dtype=object) - np.asarray(as_, object)) % q
    return b.astype(np.uint64)


def encrypt_c0(ring: Ring, m_int: np.ndarray, b: np.ndarray, v: np.ndarray,
               e0: np.ndarray) -> np.ndarray:
    """Eq. (1) first component only (Alg. 1 Line 9):
    c0 = v*b + round(Delta m) + e0 mod Q, with the BFV encoding R2.
    m_int int64 [N] (any sign), returns uint64 [L][N]."""
    N = ring.N
    m_t = np.mod(m_int, ring.t).astype(np.uint32)
    enc = encode(m_t, ring)
    v_res = signed_to_residues(v, ring)
    e_res = signed_to_residues(e0, ring)
    out = np.empty((ring.L, N), dtype=np.uint64)
    for j, q in enumerate(ring.primes):
        vb = negacyclic_at(v_res[j], b[j], q)
        out[j] = ((vb.astype(object) + enc[j].astype(object)
                   + e_res[j].astype(object)) % q).astype(np.uint64)
    return out


def crt_decode(res: List[np.ndarray], ring: Ring) -> List[int]:
    """Eq. (2) in the BFV reading: centered CRT lift r of the residues, then
    round(t r / Q) mod t."""
    Q = ring.Q
    out = []
    n = len(res[0])
    coeffs = []
    for j, q in enumerate(ring.primes):
        Qj = Q // q
        coeffs.append((Qj * pow(Qj, -1, q)) % Q)
    for i in range(n):
        r = 0
        for j in range(ring.L):
            r += int(res[j][i]) * coeffs[j]
        r %= Q
        if r > Q // 2:
            r -= Q
        m = (2 * ring.t * r + Q) // (2 * Q)        # round(t r / Q)
        out.append(m % ring.t)
    return out


def conv_protocol_decrypt(ring: Ring, plan: ConvPlan, W: np.ndarray,
                          out_full_b: np.ndarray, s_key: np.ndarray,
                          a: np.ndarray, v_list: List[np.ndarray],
                          ef_list: Dict[Tuple[int, int], np.ndarray],
                          phi1_b: Optional[np.ndarray]) -> np.ndarray:
    """Client side of Algorithm 1 for one image:
      p_beta^{(n)} = fhat_beta^{(n)} a + e_f      (Line 5)
      c1^{(n)} = sum_beta v_beta s p_beta^{(n)}   (Line 21, R13)
      c1^r gathered at the same slots (Lines 22-24); r = c0^r + c1^r;
      decrypt (Eq. 2), subtract phi1.
    out_full_b: uint64 [n_ob][L][N] (server output for this image).
    Returns int64 [c_o][w_o][h_o] = decrypted conv mod t (centered)."""
    s_res = signed_to_residues(s_key, ring)
    res = np.zeros((plan.c_o, plan.w_o, plan.h_o), dtype=np.int64)
    pos_block = output_positions(plan)
    vs = {}                                            # v_beta * s per limb
    for beta in range(plan.n_ib):
        v_res = signed_to_residues(v_list[beta], ring)
        for j, q in enumerate(ring.primes):
            vs[(beta, j)] = negacyclic_at(v_res[j], s_res[j], q)
    for ob in range(plan.n_ob):
        for nl in range(plan.c_ob):
            n = ob * plan.c_ob + nl
            if n >= plan.c_o:
                break
            pos = pos_block[nl::plan.c_ob]            # this channel's slots
            c1 = [np.zeros(len(pos), dtype=object) for _ in ring.primes]
            for beta in range(plan.n_ib):
                terms = filter_terms(W, plan, n, beta, shifted=True)
                ef = signed_to_residues(ef_list[(n, beta)], ring)
                for j, q in enumerate(ring.primes):
                    p = (sparse_mul(a[j], terms, q).astype(object)
                         + ef[j].astype(object)) % q
                    c1[j] = (c1[j] + negacyclic_at(
                        vs[(beta, j)], p.astype(np.uint64), q, pos
                    ).astype(object)) % q
            r = [(out_full_b[ob, j, pos].astype(object) + c1[j]) % q
                 for j, q in enumerate(ring.primes)]
            m = np.array(crt_decode(r, ring), dtype=np.int64)
            if phi1_b is not None:
                m = (m - phi1_b[ob, pos].astype(np.int64)) % ring.t
            m = np.where(m > ring.t // 2, m - ring.t, m)
            res[n] = m.reshape(plan.w_o, plan.h_o)
    return res


def centered_mod_t(x: np.ndarray, t: int) -> np.ndarray:
    """R24: compare conv sums mod t, centered in (-t/2, t/2]."""
    m = np.mod(x, t)
    return np.where(m > t // 2, m - t, m)


def fc_protocol_decrypt(ring: Ring, W: np.ndarray, out_b: np.ndarray,
                        s_key: np.ndarray, a: np.ndarray, v: np.ndarray,
                        ef: np.ndarray, phi1_b: Optional[np.ndarray]
                        ) -> np.ndarray:
    """Client side of Algorithm 2 for one input:
      p = w a + e_f (Line 6); c1^r = v s p (first n_o coefficients);
      r = c0^r + c1^r; decrypt (Eq. 2); subtract phi1.
    out_b: uint64 [L][n_o].  Returns int64 [n_o], centered mod t."""
    n_o = W.shape[0]
    terms = fc_weight_terms(W, ring.N)
    s_res = signed_to_residues(s_key, ring)
    v_res = signed_to_residues(v, ring)
    ef_res = signed_to_residues(ef, ring)
    pos = np.arange(n_o)
    r = []
    for j, q in enumerate(ring.primes):
        p = (sparse_mul(a[j], terms, q).astype(object)
             + ef_res[j].astype(object)) % q
        vs = negacyclic_at(v_res[j], s_res[j], q)
        c1 = negacyclic_at(vs, p.astype(np.uint64), q, pos).astype(object)
        r.append((out_b[j].astype(object) + c1) % q)
    m = np.array(crt_decode(r, ring), dtype=np.int64)
    if phi1_b is not None:
        m = (m - phi1_b.astype(np.int64)) % ring.t
    return np.where(m > ring.t // 2, m - ring.t, m)


# ---------------------------------------------------------------------------
# Server mask stream (R15): phi1[i] = SplitMix64(seed, i) mod t.
# ---------------------------------------------------------------------------
_SM_G = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


def splitmix64_py(seed: int, i: int) -> int:
    """Definition with Python integers (Vigna's SplitMix64 finaliser applied
    to the counter state seed + (i+1) * gamma)."""
    z = (seed + (i + 1) * _SM_G) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def phi1_stream(seed: int, n: int, t: int) -> np.ndarray:
    """Vectorised SplitMix64 (uint64 wrap-around arithmetic) mod t."""
    with np.errstate(over="ignore"):
        i = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed & _M64) + i * np.uint64(_SM_G)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z % np.uint64(t)).astype(np.uint32)


# ---------------------------------------------------------------------------
# Client mirror path of Algorithm 1 as separate steps (pinned through
# conv_protocol_decrypt's decryption test and tests/test_oracle_protocol.py).
# ---------------------------------------------------------------------------
def server_p(W: np.ndarray, plan: ConvPlan, ring: Ring, a: np.ndarray,
             ef: Dict[Tuple[int, int], np.ndarray]) -> np.ndarray:
    """Alg. 1 Line 5: p_beta^{(n)} = fhat_beta^{(n)} a + e_f
    (fhat with the Eq. (7) shift).  a [L][N]; ef[(n, beta)] int64 [N].
    Returns uint64 [c_o][n_ib][L][N]."""
    out = np.empty((plan.c_o, plan.n_ib, ring.L, ring.N), np.uint64)
    for n in range(plan.c_o):
        for beta in range(plan.n_ib):
            terms = filter_terms(W, plan, n, beta, shifted=True)
            e = signed_to_residues(ef[(n, beta)], ring)
            for j, q in enumerate(ring.primes):
                out[n, beta, j] = ((sparse_mul(a[j], terms, q).astype(object)
                                    + e[j].astype(object)) % q).astype(np.uint64)
    return out


def client_c1r(vs: np.ndarray, p: np.ndarray, plan: ConvPlan, ring: Ring
               ) -> np.ndarray:
    """Alg. 1 Lines 21-24: c1^{(n)} = sum_beta
    (v_beta s) p_beta^{(n)} at the slots s j + t_n, all j, 0 elsewhere --
    the layout of conv_server's full c0^r (R13, R14); Lines 22-24's payload
    is compact() of it (the valid slots).
    vs uint64 [B][n_ib][L][N] (residues of v_beta s); p from server_p.
    Returns uint64 [B][n_ob][L][N]."""
    B = vs.shape[0]
    N = ring.N
    out = np.zeros((B, plan.n_ob, ring.L, N), np.uint64)
    for b in range(B):
        for ob in range(plan.n_ob):
            for nl in range(plan.c_ob):
                n = ob * plan.c_ob + nl
                if n >= plan.c_o:
                    break
                pos = np.arange(plan.t_n(n), N, plan.s)
                for j, q in enumerate(ring.primes):
                    acc = np.zeros(pos.size, dtype=object)
                    for beta in range(plan.n_ib):
                        acc = (acc + negacyclic_at(vs[b, beta, j], p[n, beta, j], q,
                                                   pos).astype(object)) % q
                    out[b, ob, j, pos] = acc.astype(np.uint64)
    return out


def decrypt_round(r: np.ndarray, ring: Ring) -> np.ndarray:
    """Eq. (2) in the BFV reading: m = round(t CRT(r) / Q) mod t, per
    coefficient of r [..][L][len] (exact big integers).  uint32 [..][len]."""
    r = np.asarray(r)
    lead, ln = r.shape[:-2], r.shape[-1]
    flat = r.reshape((-1, ring.L, ln))
    out = np.empty((flat.shape[0], ln), np.uint32)
    for i in range(flat.shape[0]):
        out[i] = np.array(crt_decode([flat[i, j] for j in range(ring.L)], ring),
                          dtype=np.uint32)
    return out.reshape(lead + (ln,))


def reduce_mod_binomial(a: np.ndarray, s: int, zeta: int, q: int) -> np.ndarray:
    """a(X) mod (X^s - zeta) over Z_q by definition: X^{j s + u} =
    zeta^j X^u, so coefficient u is sum_j a[j s + u] zeta^j (DESIGN.md §4,
    the incomplete transform behind the fold).  Returns uint64 [s]."""
    a = [int(x) for x in a]
    N = len(a)
    out = [0] * s
    zj = 1
    for j in range(N // s):
        for u in range(s):
            out[u] = (out[u] + a[j * s + u] * zj) % q
        zj = zj * zeta % q
    return np.array(out, dtype=np.uint64)


def incomplete_ntt_def(a: np.ndarray, q: int, psi: int, s: int) -> np.ndarray:
    """The transform the conv fold runs on c0 and f: block g
    (g < N/s) of s outputs = a mod (X^s - zeta_g), zeta_g =
    psi^{s (2 brv_{log2(N/s)}(g) + 1)}, the N/s roots of Y^{N/s} = -1 (Y = X^s)
    in the bit-reversed order of the full NTT (s = 1: ntt_def in bit-reversed
    order).  Returns uint64 [N]."""
    N = len(a)
    T = (N // s).bit_length() - 1
    out = np.empty(N, np.uint64)
    for g in range(N // s):
        b = int(format(g, f"0{T}b")[::-1], 2) if T else 0
        out[g * s:(g + 1) * s] = reduce_mod_binomial(a, s, pow(psi, s * (2 * b + 1), q), q)
    return out


# ---------------------------------------------------------------------------
# FC for n_i n_o > N (§8(f) packing variant).  PAPER.md:205: "If n_i n_o > N,
# then the weight matrix can be decomposed into sub-matrices whose sizes are
# smaller or equal to N, and our proposed packing scheme still applies to
# the decomposed matrices."  Reading R27: sub-matrices of n_ot rows x n_it
# columns, n_it = min(n_i, N), n_ot = min(n_o, floor(N / n_it)) (Table III's
# ceil(n_o / floor(N / n_i)) polynomials when n_i <= N); input block beta is
# its own ciphertext (Eq. (9) with stride n_ot), output tile t sums the
# products over the input blocks, bias and mask added once.
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class FcPlan:
    n_i: int
    n_o: int
    N: int
    n_it: int
    n_ib: int
    n_ot: int
    n_t: int


def plan_fc(n_i: int, n_o: int, N: int) -> FcPlan:
    n_it = min(n_i, N)
    n_ot = min(n_o, N // n_it)
    return FcPlan(n_i, n_o, N, n_it, -(-n_i // n_it), n_ot, -(-n_o // n_ot))


def fc_input_blocks(I: np.ndarray, fp: FcPlan) -> np.ndarray:
    """Eq. (9) per input block: int64 [n_ib][N]."""
    return np.stack([fc_input_int(np.asarray(I)[b * fp.n_it:(b + 1) * fp.n_it], fp.n_ot, fp.N)
                     for b in range(fp.n_ib)])


def fc_submatrix(W: np.ndarray, fp: FcPlan, beta: int, t: int) -> np.ndarray:
    """Rows t n_ot .. +n_ot, columns beta n_it .. +n_it of W, zero-padded to
    n_ot x n_it (the packing stride of every tile is n_ot)."""
    sub = np.zeros((fp.n_ot, fp.n_it), dtype=np.int64)
    blk = np.asarray(W, np.int64)[t * fp.n_ot:(t + 1) * fp.n_ot,
                                   beta * fp.n_it:(beta + 1) * fp.n_it]
    sub[:blk.shape[0], :blk.shape[1]] = blk
    return sub


def fc_server_tiled(c0: np.ndarray, W: np.ndarray, bias: Optional[np.ndarray],
                    ring: Ring, phi1: Optional[np.ndarray] = None) -> np.ndarray:
    """Algorithm 2 Line 13 per sub-matrix: tile t = sum_beta c0_beta w_{beta,t}
    (first n_ot coefficients), + enc(B) + enc(phi1).
    c0 uint64 [B][n_ib][L][N]; phi1 uint32 [B][n_o]; returns uint64
    [B][L][n_o]."""
    n_o, n_i = np.asarray(W).shape
    B = c0.shape[0]
    fp = plan_fc(n_i, n_o, ring.N)
    assert c0.shape == (B, fp.n_ib, ring.L, ring.N)
    qo = np.array(ring.primes, dtype=object)[None, :, None]
    out = np.empty((B, ring.L, n_o), dtype=np.uint64)
    for t in range(fp.n_t):
        k0, k1 = t * fp.n_ot, min(n_o, (t + 1) * fp.n_ot)
        acc = np.zeros((B, ring.L, fp.n_ot), dtype=object)
        for beta in range(fp.n_ib):
            part = fc_server(c0[:, beta], fc_submatrix(W, fp, beta, t), None, ring, None)
            acc = (acc + part.astype(object)) % qo
        acc = acc[:, :, :k1 - k0]
        if bias is not None:
            acc = (acc + encode(np.mod(np.asarray(bias, np.int64)[k0:k1], ring.t).astype(np.uint32),
                                ring).astype(object)[None]) % qo
        if phi1 is not None:
            for b in range(B):
                acc[b] = (acc[b] + encode(np.asarray(phi1)[b, k0:k1].astype(np.uint32),
                                          ring).astype(object)) % qo[0]
        out[:, :, k0:k1] = acc.astype(np.uint64)
    return out


# ---------------------------------------------------------------------------
# Modulus switching before the wire (§8(f); the BFV counterpart of the
# paper's Q -> Q' rescale, PAPER.md:300 and Table II's log Q' factor).
# Reading R28: Q' = q_0 ... q_{L'-1} (the first L' limbs), each share is
# switched on its own: x' = round(Q' x / Q) mod Q' with x the canonical
# CRT value in [0, Q); no ties since Q / Q' is odd.
# ---------------------------------------------------------------------------
def mod_switch(r: np.ndarray, ring: Ring, L_keep: int) -> np.ndarray:
    """r uint64 [..][L][len] -> uint64 [..][L_keep][len], exact big ints."""
    r = np.asarray(r)
    lead, ln = r.shape[:-2], r.shape[-1]
    flat = r.reshape((-1, ring.L, ln))
    P = 1
    for q in ring.primes[L_keep:]:
        P *= q
    out = np.empty((flat.shape[0], L_keep, ln), np.uint64)
    for i in range(flat.shape[0]):
        for k in range(ln):
            x = 0
            for j, q in enumerate(ring.primes):          # CRT by definition
                Qj = ring.Q // q
                x += int(flat[i, j, k]) * Qj * pow(Qj, -1, q)
            x %= ring.Q
            y = (2 * x + P) // (2 * P)                    # round(x / P)
            for j in range(L_keep):
                out[i, j, k] = y % ring.primes[j]
    return out.reshape(lead + (L_keep, ln))


# ---------------------------------------------------------------------------
# Chained pipeline (§8(f), Fig. 5): after each layer the
# client decrypts, the garbled-circuit stage removes phi1 and applies ReLU,
# and the client re-packs the activations for the next layer.  The GC is a
# trusted stub here (reading R29, phi2 = 0): x = centered((m - phi1) mod t),
# y = min(qmax, max(x, 0) >> shift); the network's global average pooling
# before the FC (plain-20) is floor(mean) per channel, also in the stub.
# ---------------------------------------------------------------------------
def relu_requant(x: np.ndarray, t: int, shift: int, qmax: int) -> np.ndarray:
    """R29 stub on conv outputs (any integers): centered mod t, ReLU,
    arithmetic shift, clamp."""
    c = centered_mod_t(np.asarray(x, np.int64), t)
    return np.minimum(qmax, np.maximum(c, 0) >> shift).astype(np.int64)


def avgpool(x: np.ndarray) -> np.ndarray:
    """[C][H][W] -> [C]: floor(sum / (H W))."""
    x = np.asarray(x, np.int64)
    return x.reshape(x.shape[0], -1).sum(1) // (x.shape[1] * x.shape[2])


def plain_chain(img: np.ndarray, Ws, layers, N: int, t: int, shift: int, qmax: int,
                fcW: Optional[np.ndarray] = None, fcB: Optional[np.ndarray] = None):
    """Plaintext reference of the chained pipeline for one image: per layer
    conv2d_ref (Eq. (3)/(4)) -> relu_requant; then avgpool -> FC (W I + B),
    centered mod t.  Returns (activations per layer, logits or None)."""
    acts = []
    x = np.asarray(img, np.int64)
    for W, Ly in zip(Ws, layers):
        x = relu_requant(conv2d_ref(x, W, plan_conv(Ly, N)), t, shift, qmax)
        acts.append(x)
    logits = None
    if fcW is not None:
        v = avgpool(x)
        logits = centered_mod_t(np.asarray(fcW, np.int64) @ v +
                                (0 if fcB is None else np.asarray(fcB, np.int64)), t)
    return acts, logits
