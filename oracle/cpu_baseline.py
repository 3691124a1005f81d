"""CPU textbook-NTT baseline -- TEST / BENCHMARK
INFRASTRUCTURE ONLY: bench.py's cpu_baseline leg times it as the "fairer
CPU baseline" beside the sparse-direct oracle; tests/test_oracle_cpu_ntt.py
pins it against the oracle's definition (ref.conv_server).  It is not a
parity reference for the GPU and shares no code with the CUDA path.
C source: oracle/cpu_ntt_baseline.c (gcc, OpenMP)."""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

from oracle import ref as R

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cpu_ntt_baseline.c")
_LIB_PATH = os.path.join(_HERE, "libcpu_ntt.so")
_lib = None


def build_lib(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O3", "-march=native", "-fopenmp", "-fPIC", "-shared",
                               "-o", _LIB_PATH, _SRC])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build_lib()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i32, i64, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        L.cpu_ntt_forward.argtypes = [P, i64, i32, i32, P, P]
        L.cpu_ntt_conv_server.argtypes = [P, i32, i32, i32, i32, P, P, i32, i32, i32, i32,
                                          P, P, P, P, u64, u64, P]
        L.cpu_ntt_companions.argtypes = [P, P, i64, i32, i32, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def prepare_filters(W: np.ndarray, plan: R.ConvPlan, ring: R.Ring):
    """Spectra of the Eq. (6)-(7) filter polynomials, [c_o][n_ib][L][N], and
    their Shoup companions (server initialisation; not part of the timed unit)."""
    f = np.stack([np.stack([R.signed_to_residues(R.filter_poly_int(W, plan, n, beta), ring)
                            for beta in range(plan.n_ib)]) for n in range(plan.c_o)])
    f = np.ascontiguousarray(f, dtype=np.uint64)
    psi = np.array([R.min_psi(q, plan.N) for q in ring.primes], dtype=np.uint64)
    lib().cpu_ntt_forward(_p(f), plan.c_o * plan.n_ib, ring.L, plan.N, _p(ring.q_arr), _p(psi))
    fp = np.empty_like(f)
    lib().cpu_ntt_companions(_p(f), _p(fp), plan.c_o * plan.n_ib, ring.L, plan.N, _p(ring.q_arr))
    return f, fp


def conv_server(c0: np.ndarray, fspec, plan: R.ConvPlan, ring: R.Ring,
                phi1: Optional[np.ndarray] = None) -> np.ndarray:
    """The server work unit of ref.conv_server, computed with NTT-domain
    products: uint64 [B][n_ob][L][N]."""
    c0 = np.ascontiguousarray(c0, dtype=np.uint64)
    B = c0.shape[0]
    out = np.empty((B, plan.n_ob, ring.L, plan.N), dtype=np.uint64)
    psi = np.array([R.min_psi(q, plan.N) for q in ring.primes], dtype=np.uint64)
    ph = None if phi1 is None else np.ascontiguousarray(phi1, dtype=np.uint32)
    lib().cpu_ntt_conv_server(_p(c0), B, plan.n_ib, ring.L, plan.N, _p(ring.q_arr), _p(psi),
                              plan.s, plan.c_o, plan.c_ob, plan.n_ob, _p(fspec[0]),
                              _p(fspec[1]), _p(ph),
                              _p(ring.delta_mod_q), ring.r_t, ring.t, _p(out))
    return out
