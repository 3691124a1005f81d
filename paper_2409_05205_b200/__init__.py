"""Thin Python binding of libhe_rotfree.so (include/he_rotfree.h).

Argument marshalling only: every step of the path runs in the library's
sm_100a kernels.  Torch is used for device memory and streams; residue
tensors are torch.int64 (bit patterns of the uint64 residues), masks and
integer data torch.int32.  There is no CPU fallback: importing this module
raises if the CUDA library is missing, and every call checks that its
tensors live on the context's CUDA device.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhe_rotfree.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import "
        f"__graft_entry__ as g; g.build()'` (nvcc, sm_100a). There is no CPU "
        f"fallback.")

_lib = ctypes.CDLL(LIB_PATH)

HE_OK, HE_EINVAL, HE_ESHAPE, HE_EPARAM, HE_ECUDA, HE_ENOMEM = range(6)


class HeError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        msg = f"{what}: {_lib.he_status_str(status).decode()}"
        if status == HE_ECUDA:
            msg += f" ({_lib.he_last_cuda_error().decode()})"
        super().__init__(msg)


class RingDesc(ctypes.Structure):
    _fields_ = [("log2N", ctypes.c_uint32), ("L", ctypes.c_uint32),
                ("q", ctypes.POINTER(ctypes.c_uint64)), ("t", ctypes.c_uint64)]


class ConvDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("c_i", "c_o", "w_i", "h_i", "f_w", "f_h", "stride", "pad")]


class ConvPlan(ctypes.Structure):
    _fields_ = [("d", ConvDesc)] + [(n, ctypes.c_int32) for n in
                                     ("s", "c_ib", "n_ib", "c_ob", "n_ob", "w_p",
                                      "h_p", "w_o", "h_o", "n_valid", "k_u")]

    def __repr__(self):
        return (f"ConvPlan(s={self.s}, c_ib={self.c_ib}, n_ib={self.n_ib}, "
                f"c_ob={self.c_ob}, n_ob={self.n_ob}, w_o={self.w_o}, "
                f"h_o={self.h_o}, n_valid={self.n_valid})")


class FcDesc(ctypes.Structure):
    _fields_ = [("n_i", ctypes.c_int32), ("n_o", ctypes.c_int32)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_SZ = ctypes.c_size_t


def _sig(name, args, res=ctypes.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_lib.he_status_str.argtypes = [ctypes.c_int]
_lib.he_status_str.restype = ctypes.c_char_p
_lib.he_last_cuda_error.argtypes = []
_lib.he_last_cuda_error.restype = ctypes.c_char_p
_sig("he_ctx_create", [ctypes.POINTER(RingDesc), _I, ctypes.POINTER(_P)])
_sig("he_ctx_destroy", [_P], None)
_sig("he_ctx_psi", [_P, ctypes.c_uint32], ctypes.c_uint64)
_sig("he_conv_plan_make", [_P, ctypes.POINTER(ConvDesc), _I,
                           ctypes.POINTER(ConvPlan)])
_sig("he_conv_plan_dense", [ctypes.POINTER(ConvPlan), ctypes.POINTER(ConvPlan)])
_sig("he_pack_input", [_P, ctypes.POINTER(ConvPlan), _P, _I, _P, _P, _P])
_sig("he_filter_bytes", [_P, ctypes.POINTER(ConvPlan)], _SZ)
_sig("he_pack_filters_workspace_bytes", [_P, ctypes.POINTER(ConvPlan)], _SZ)
_sig("he_pack_filters", [_P, ctypes.POINTER(ConvPlan), _P, _P, _P, _SZ, _P])
_sig("he_conv_workspace_bytes", [_P, ctypes.POINTER(ConvPlan), _I], _SZ)
_sig("he_conv", [_P, ctypes.POINTER(ConvPlan), _P, _I, _P, _P, _P, _P, _SZ,
                 _P])
_sig("he_conv_ex", [_P, ctypes.POINTER(ConvPlan), _P, _I, _P, _P, _P, _P, _P,
                    _SZ, _P, _P])
_sig("he_fc_ex", [_P, ctypes.POINTER(FcDesc), _P, _I, _P, _P, _P, _P, _P, _SZ,
                  _P, _P])
_sig("he_mask_extract", [_P, ctypes.POINTER(ConvPlan), _P, _I, _P, _P, _P])
_sig("he_pack_fc_input", [_P, ctypes.POINTER(FcDesc), _P, _I, _P, _P, _P])
_sig("he_fc_wspec_bytes", [_P, ctypes.POINTER(FcDesc)], _SZ)
_sig("he_fc_workspace_bytes", [_P, ctypes.POINTER(FcDesc), _I], _SZ)
_sig("he_pack_fc_weights", [_P, ctypes.POINTER(FcDesc), _P, _P, _P, _P, _P,
                            _SZ, _P])
_sig("he_fc", [_P, ctypes.POINTER(FcDesc), _P, _I, _P, _P, _P, _P, _P, _SZ,
               _P])
_sig("he_residues_pack50", [_P, _SZ, _P, _P])
_sig("he_residues_unpack50", [_P, _SZ, _P, _P])
_sig("he_phi1_generate", [_P, ctypes.c_uint64, _SZ, _P, _P])
_sig("he_ntt_forward", [_P, _P, _I, _P])
_sig("he_ntt_inverse", [_P, _P, _I, _P])
_sig("he_ntt_forward_partial", [_P, _P, _I, _I, _P])
_sig("he_server_p_workspace_bytes", [_P, ctypes.POINTER(ConvPlan)], _SZ)
_sig("he_server_init_p", [_P, ctypes.POINTER(ConvPlan), _P, _P, _P, _P, _P,
                          _SZ, _P])
_sig("he_pack_client_p", [_P, ctypes.POINTER(ConvPlan), _P, _P, _P, _SZ, _P])
_sig("he_residues_from_int", [_P, _P, ctypes.c_long, _P, _P])
_sig("he_poly_mul", [_P, _P, _P, _I, _I, _P, _P, _SZ, _P])
_sig("he_decrypt_round", [_P, _P, _P, ctypes.c_long, ctypes.c_long, _P, _P])
_sig("he_mod_switch", [_P, _P, ctypes.c_long, ctypes.c_long, _I, _P, _P])
_sig("he_pk_mask", [_P, _P, _P, ctypes.c_long, _P, _P, _P, _SZ, _P])
_sig("he_pk_mask_vs", [_P, _P, _P, ctypes.c_long, _P, _P, _P, _P, _P, _SZ, _P])
_sig("he_relu_requant", [_P, ctypes.POINTER(ConvPlan), _P, _I, _P, _I, _I, _P, _P])
_sig("he_avgpool", [_P, ctypes.c_long, _I, _P, _P])
_sig("he_multi_image_spacing", [_P, ctypes.POINTER(ConvPlan), _P, _P])
_sig("he_pack_input_multi", [_P, ctypes.POINTER(ConvPlan), _P, _I, _I, _I, _P, _P, _P])
_sig("he_mask_extract_multi", [_P, ctypes.POINTER(ConvPlan), _P, _I, _I, _I, _P, _P, _P])
_sig("he_unmask", [_P, _P, _P, ctypes.c_long, _P, _P])
_sig("he_c0_compact", [_P, ctypes.POINTER(ConvPlan), _P, _I, _P, _P])
_sig("he_filter_coeffs", [_P, ctypes.POINTER(ConvPlan), _P, _I, _P, _P, _SZ, _P])
_sig("he_conv_plain_workspace_bytes", [_P, ctypes.POINTER(ConvPlan), _I], _SZ)
_sig("he_pack_filters_plain", [_P, ctypes.POINTER(ConvPlan), _P, _P, _P])
_sig("he_conv_plain", [_P, ctypes.POINTER(ConvPlan), _P, _I, _P, _P, _P, _P, _SZ, _P])
_sig("he_c0_expand", [_P, ctypes.POINTER(ConvPlan), _P, _I, _P, _P])
_sig("he_fc_server_p_workspace_bytes", [_P, ctypes.POINTER(FcDesc)], _SZ)
_sig("he_fc_server_init_p", [_P, ctypes.POINTER(FcDesc), _P, _P, _P, _P, _P, _SZ, _P])
_sig("he_pack_fc_client_p", [_P, ctypes.POINTER(FcDesc), _P, _P, _P, _SZ, _P])

EXPORTED = ["he_status_str", "he_last_cuda_error", "he_multi_image_spacing",
            "he_pack_input_multi", "he_mask_extract_multi", "he_ctx_create", "he_ctx_destroy", "he_ctx_psi",
            "he_conv_plan_make", "he_conv_plan_dense", "he_pack_input", "he_filter_bytes",
            "he_pack_filters_workspace_bytes", "he_pack_filters",
            "he_conv_workspace_bytes", "he_conv", "he_conv_ex", "he_mask_extract",
            "he_pack_fc_input", "he_fc_wspec_bytes", "he_fc_workspace_bytes",
            "he_pack_fc_weights", "he_fc", "he_fc_ex", "he_residues_pack50",
            "he_residues_unpack50", "he_phi1_generate", "he_ntt_forward",
            "he_ntt_inverse", "he_ntt_forward_partial", "he_server_p_workspace_bytes", "he_server_init_p",
            "he_pack_client_p", "he_residues_from_int", "he_poly_mul",
            "he_decrypt_round", "he_mod_switch", "he_pk_mask", "he_pk_mask_vs",
            "he_relu_requant",
            "he_avgpool", "he_unmask", "he_c0_compact", "he_c0_expand", "he_filter_coeffs",
            "he_conv_plain_workspace_bytes", "he_pack_filters_plain", "he_conv_plain", "he_fc_server_p_workspace_bytes", "he_fc_server_init_p",
            "he_pack_fc_client_p"]


def _events(events):
    """list of torch.cuda.Event -> void*[] of cudaEvent_t (or None)."""
    if events is None:
        return None
    arr = (ctypes.c_void_p * len(events))(*[e.cuda_event for e in events])
    return arr


def _check(st: int, what: str):
    if st != HE_OK:
        raise HeError(st, what)


def _stream(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def conv_plan_make(ctx: Optional["Context"], c_i, c_o, w_i, h_i, f_w=3, f_h=3,
                   stride=1, pad=1, s_override=0) -> ConvPlan:
    d = ConvDesc(c_i, c_o, w_i, h_i, f_w, f_h, stride, pad)
    p = ConvPlan()
    _check(_lib.he_conv_plan_make(ctx._h, ctypes.byref(d), s_override,
                                  ctypes.byref(p)), "he_conv_plan_make")
    return p


class Context:
    """he_ctx: immutable ring context on one CUDA device."""

    def __init__(self, primes: Sequence[int], log2N: int, t: int = 65537,
                 device: int = 0):
        self.primes = [int(q) for q in primes]
        self.L = len(self.primes)
        self.log2N = log2N
        self.N = 1 << log2N
        self.t = t
        self.device = torch.device("cuda", device)
        arr = (ctypes.c_uint64 * self.L)(*self.primes)
        self._q = arr
        r = RingDesc(log2N, self.L, ctypes.cast(arr, ctypes.POINTER(
            ctypes.c_uint64)), t)
        h = ctypes.c_void_p()
        _check(_lib.he_ctx_create(ctypes.byref(r), device, ctypes.byref(h)),
               "he_ctx_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.he_ctx_destroy(h)
        self._h = None

    def psi(self, j: int) -> int:
        return int(_lib.he_ctx_psi(self._h, j))

    # -------------------------------------------------------------- helpers
    def _dev(self, *ts):
        for t in ts:
            if t is not None and (not t.is_cuda or t.device != self.device
                                  or not t.is_contiguous()):
                raise ValueError("tensors must be contiguous on " +
                                 str(self.device))

    def empty_u64(self, *shape) -> torch.Tensor:
        return torch.empty(shape, dtype=torch.int64, device=self.device)

    @staticmethod
    def _ptr(t: Optional[torch.Tensor]):
        return ctypes.c_void_p(t.data_ptr()) if t is not None else None

    # ---------------------------------------------------------------- conv
    def plan(self, c_i, c_o, w_i, h_i, f_w=3, f_h=3, stride=1, pad=1,
             s_override=0) -> ConvPlan:
        return conv_plan_make(self, c_i, c_o, w_i, h_i, f_w, f_h, stride, pad,
                              s_override)

    def pack_input(self, p: ConvPlan, img: torch.Tensor,
                   ve: Optional[torch.Tensor] = None,
                   out: Optional[torch.Tensor] = None, stream=None):
        B = img.shape[0]
        if out is None:
            out = self.empty_u64(B, p.n_ib, self.L, self.N)
        self._dev(img, ve, out)
        _check(_lib.he_pack_input(self._h, ctypes.byref(p), self._ptr(img), B,
                                  self._ptr(ve), self._ptr(out),
                                  _stream(stream)), "he_pack_input")
        return out

    def pack_filters(self, p: ConvPlan, W: torch.Tensor, stream=None):
        nb = _lib.he_filter_bytes(self._h, ctypes.byref(p))
        fspec = self.empty_u64(nb // 8)
        wsb = _lib.he_pack_filters_workspace_bytes(self._h, ctypes.byref(p))
        ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        self._dev(W)
        _check(_lib.he_pack_filters(self._h, ctypes.byref(p), self._ptr(W),
                                    self._ptr(fspec), self._ptr(ws), wsb,
                                    _stream(stream)), "he_pack_filters")
        return fspec

    def conv_workspace(self, p: ConvPlan, B: int) -> torch.Tensor:
        nb = _lib.he_conv_workspace_bytes(self._h, ctypes.byref(p), B)
        return torch.empty(nb, dtype=torch.uint8, device=self.device)

    def conv(self, p: ConvPlan, c0: torch.Tensor, fspec: torch.Tensor,
             phi1: Optional[torch.Tensor] = None,
             out: Optional[torch.Tensor] = None,
             ws: Optional[torch.Tensor] = None, stream=None, events=None,
             compact: Optional[torch.Tensor] = None, full: bool = True):
        """he_conv; he_conv_ex when `compact` (fused payload) or `events`
        (4 torch.cuda.Event with enable_timing, recorded at the K1/K3/K4
        stage boundaries) is given.  full=False skips the full output."""
        B = c0.shape[0]
        if out is None and full:
            out = self.empty_u64(B, p.n_ob, self.L, self.N)
        if ws is None:
            ws = self.conv_workspace(p, B)
        self._dev(c0, fspec, phi1, out, ws, compact)
        if events is None and compact is None:
            _check(_lib.he_conv(self._h, ctypes.byref(p), self._ptr(c0), B,
                                self._ptr(fspec), self._ptr(phi1),
                                self._ptr(out), self._ptr(ws),
                                ws.numel() * ws.element_size(),
                                _stream(stream)), "he_conv")
        else:
            _check(_lib.he_conv_ex(self._h, ctypes.byref(p), self._ptr(c0), B,
                                   self._ptr(fspec), self._ptr(phi1),
                                   self._ptr(out), self._ptr(compact),
                                   self._ptr(ws),
                                   ws.numel() * ws.element_size(),
                                   _stream(stream), _events(events)),
                   "he_conv_ex")
        return out if full else compact

    def mask_extract(self, p: ConvPlan, out_full: torch.Tensor,
                     phi1: Optional[torch.Tensor] = None,
                     compact: Optional[torch.Tensor] = None, stream=None):
        B = out_full.shape[0]
        if compact is None:
            compact = self.empty_u64(B, p.n_ob, self.L, p.n_valid)
        self._dev(out_full, phi1, compact)
        _check(_lib.he_mask_extract(self._h, ctypes.byref(p),
                                    self._ptr(out_full), B, self._ptr(phi1),
                                    self._ptr(compact), _stream(stream)),
               "he_mask_extract")
        return compact

    # ------------------------------------------------ multi-image packing
    def multi_image_spacing(self, p: ConvPlan):
        """(D, P) of he_multi_image_spacing (R31)."""
        D, P = ctypes.c_int32(), ctypes.c_int32()
        _check(_lib.he_multi_image_spacing(self._h, ctypes.byref(p), ctypes.byref(D),
                                           ctypes.byref(P)), "he_multi_image_spacing")
        return D.value, P.value

    def pack_input_multi(self, p: ConvPlan, img: torch.Tensor, P: int, D: int,
                         ve: Optional[torch.Tensor] = None,
                         out: Optional[torch.Tensor] = None, stream=None):
        B = img.shape[0]
        Bc = -(-B // P)
        if out is None:
            out = self.empty_u64(Bc, p.n_ib, self.L, self.N)
        self._dev(img, ve, out)
        _check(_lib.he_pack_input_multi(self._h, ctypes.byref(p), self._ptr(img), B, P, D,
                                        self._ptr(ve), self._ptr(out), _stream(stream)),
               "he_pack_input_multi")
        return out

    def mask_extract_multi(self, p: ConvPlan, out_full: torch.Tensor, P: int, D: int,
                           phi1: Optional[torch.Tensor] = None,
                           compact: Optional[torch.Tensor] = None, stream=None):
        Bc = out_full.shape[0]
        if compact is None:
            compact = self.empty_u64(Bc, p.n_ob, self.L, P * p.n_valid)
        self._dev(out_full, phi1, compact)
        _check(_lib.he_mask_extract_multi(self._h, ctypes.byref(p), self._ptr(out_full), Bc,
                                          P, D, self._ptr(phi1), self._ptr(compact),
                                          _stream(stream)), "he_mask_extract_multi")
        return compact

    # ------------------------------------------------------------------ FC
    def fc_plan(self, n_i, n_o):
        """(n_it, n_ib, n_ot, n_t) of the sub-matrix tiling (he_rotfree.h)."""
        n_it = min(n_i, self.N)
        n_ot = min(n_o, self.N // n_it)
        return n_it, -(-n_i // n_it), n_ot, -(-n_o // n_ot)

    def fc_pack_input(self, n_i, n_o, inp: torch.Tensor,
                      ve: Optional[torch.Tensor] = None,
                      out: Optional[torch.Tensor] = None, stream=None):
        """-> [B][n_ib][L][N] (one ciphertext per input block)."""
        f = FcDesc(n_i, n_o)
        B = inp.shape[0]
        if out is None:
            out = self.empty_u64(B, self.fc_plan(n_i, n_o)[1], self.L, self.N)
        self._dev(inp, ve, out)
        _check(_lib.he_pack_fc_input(self._h, ctypes.byref(f), self._ptr(inp),
                                     B, self._ptr(ve), self._ptr(out),
                                     _stream(stream)), "he_pack_fc_input")
        return out

    def fc_pack_weights(self, W: torch.Tensor,
                        bias: Optional[torch.Tensor] = None, stream=None):
        n_o, n_i = W.shape
        f = FcDesc(n_i, n_o)
        wspec = self.empty_u64(_lib.he_fc_wspec_bytes(self._h,
                                                      ctypes.byref(f)) // 8)
        benc = self.empty_u64(self.L, n_o)
        wsb = _lib.he_fc_workspace_bytes(self._h, ctypes.byref(f), 1)
        ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        self._dev(W, bias)
        _check(_lib.he_pack_fc_weights(self._h, ctypes.byref(f), self._ptr(W),
                                       self._ptr(bias), self._ptr(wspec),
                                       self._ptr(benc), self._ptr(ws), wsb,
                                       _stream(stream)), "he_pack_fc_weights")
        return wspec, benc

    def fc_workspace(self, n_i, n_o, B) -> torch.Tensor:
        f = FcDesc(n_i, n_o)
        nb = _lib.he_fc_workspace_bytes(self._h, ctypes.byref(f), B)
        return torch.empty(nb, dtype=torch.uint8, device=self.device)

    def fc(self, n_i, n_o, c0: torch.Tensor, wspec: torch.Tensor,
           bias_enc: torch.Tensor, phi1: Optional[torch.Tensor] = None,
           out: Optional[torch.Tensor] = None,
           ws: Optional[torch.Tensor] = None, stream=None, events=None):
        f = FcDesc(n_i, n_o)
        B = c0.shape[0]
        if out is None:
            out = self.empty_u64(B, self.L, n_o)
        if ws is None:
            ws = self.fc_workspace(n_i, n_o, B)
        self._dev(c0, wspec, bias_enc, phi1, out, ws)
        args = (self._h, ctypes.byref(f), self._ptr(c0), B, self._ptr(wspec),
                self._ptr(bias_enc), self._ptr(phi1), self._ptr(out),
                self._ptr(ws), ws.numel() * ws.element_size(), _stream(stream))
        if events is None:
            _check(_lib.he_fc(*args), "he_fc")
        else:
            _check(_lib.he_fc_ex(*args, _events(events)), "he_fc_ex")
        return out

    # --------------------------------------------------------- wire format
    @staticmethod
    def packed_bytes(n: int) -> int:
        return n * 50 // 8

    def pack50(self, x: torch.Tensor, out: Optional[torch.Tensor] = None,
               stream=None) -> torch.Tensor:
        """Residues (any shape, int64 view of u64 < 2^50) -> uint8 wire bytes."""
        n = x.numel()
        if out is None:
            out = torch.empty(self.packed_bytes(n), dtype=torch.uint8,
                              device=self.device)
        self._dev(x, out)
        _check(_lib.he_residues_pack50(self._ptr(x), n, self._ptr(out),
                                       _stream(stream)), "he_residues_pack50")
        return out

    def unpack50(self, packed: torch.Tensor, out: torch.Tensor,
                 stream=None) -> torch.Tensor:
        self._dev(packed, out)
        _check(_lib.he_residues_unpack50(self._ptr(packed), out.numel(),
                                         self._ptr(out), _stream(stream)),
               "he_residues_unpack50")
        return out

    def phi1_generate(self, seed: int, out: torch.Tensor, stream=None):
        """out (int32 view of uint32) <- SplitMix64(seed, i) mod t."""
        self._dev(out)
        _check(_lib.he_phi1_generate(self._h, seed & (2 ** 64 - 1), out.numel(),
                                     self._ptr(out), _stream(stream)),
               "he_phi1_generate")
        return out

    # ---------------------------------------------------------- transforms
    def ntt_forward(self, data: torch.Tensor, stream=None):
        self._dev(data)
        batch = data.numel() // (self.L * self.N)
        _check(_lib.he_ntt_forward(self._h, self._ptr(data), batch,
                                   _stream(stream)), "he_ntt_forward")
        return data

    def ntt_forward_partial(self, data: torch.Tensor, skip: int, stream=None):
        self._dev(data)
        batch = data.numel() // (self.L * self.N)
        _check(_lib.he_ntt_forward_partial(self._h, self._ptr(data), batch, skip,
                                           _stream(stream)), "he_ntt_forward_partial")
        return data

    def ntt_inverse(self, data: torch.Tensor, stream=None):
        self._dev(data)
        batch = data.numel() // (self.L * self.N)
        _check(_lib.he_ntt_inverse(self._h, self._ptr(data), batch,
                                   _stream(stream)), "he_ntt_inverse")
        return data

    # ------------------------------------------- client mirror path (§8 f)
    def server_init_p(self, p: ConvPlan, W: torch.Tensor, a: torch.Tensor,
                      ef: Optional[torch.Tensor] = None, stream=None):
        """Alg. 1 Line 5: p_beta^{(n)} = fhat_beta^{(n)} a + e_f
        -> int64 view [c_o][n_ib][L][N]."""
        out = self.empty_u64(p.d.c_o, p.n_ib, self.L, self.N)
        wsb = _lib.he_server_p_workspace_bytes(self._h, ctypes.byref(p))
        ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        self._dev(W, a, ef)
        _check(_lib.he_server_init_p(self._h, ctypes.byref(p), self._ptr(W),
                                     self._ptr(a), self._ptr(ef),
                                     self._ptr(out), self._ptr(ws), wsb,
                                     _stream(stream)), "he_server_init_p")
        return out

    def dense_plan(self, p: ConvPlan) -> ConvPlan:
        """The plan with k_u = s (he_conv_plan_dense): for the client's conv
        on he_pack_client_p spectra."""
        out = ConvPlan()
        _check(_lib.he_conv_plan_dense(ctypes.byref(p), ctypes.byref(out)),
               "he_conv_plan_dense")
        return out

    def pack_client_p(self, p: ConvPlan, pp: torch.Tensor, stream=None):
        """Spectra of X^{-t_n} p in he_pack_filters' layout, for
        conv(dense_plan(p), vs, pspec).  p may be the normal plan."""
        p = self.dense_plan(p)
        nb = _lib.he_filter_bytes(self._h, ctypes.byref(p))
        pspec = self.empty_u64(nb // 8)
        wsb = _lib.he_pack_filters_workspace_bytes(self._h, ctypes.byref(p))
        ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        self._dev(pp)
        _check(_lib.he_pack_client_p(self._h, ctypes.byref(p), self._ptr(pp),
                                     self._ptr(pspec), self._ptr(ws), wsb,
                                     _stream(stream)), "he_pack_client_p")
        return pspec

    def residues_from_int(self, x: torch.Tensor, stream=None):
        """int32 [..][N] -> int64 view [..][L][N] of x mod q_j."""
        n = x.numel() // self.N
        out = self.empty_u64(*x.shape[:-1], self.L, self.N)
        self._dev(x)
        _check(_lib.he_residues_from_int(self._h, self._ptr(x), n,
                                         self._ptr(out), _stream(stream)),
               "he_residues_from_int")
        return out

    def poly_mul(self, x: torch.Tensor, y: torch.Tensor,
                 out: Optional[torch.Tensor] = None, stream=None):
        """Negacyclic products x[b] * y[b or 0] over [B][L][N]."""
        B = x.numel() // (self.L * self.N)
        yb = y.numel() // (self.L * self.N)
        if out is None:
            out = torch.empty_like(x)
        wsb = 8 * yb * self.L * self.N
        ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        self._dev(x, y, out)
        _check(_lib.he_poly_mul(self._h, self._ptr(x), self._ptr(y), B, yb,
                                self._ptr(out), self._ptr(ws), wsb,
                                _stream(stream)), "he_poly_mul")
        return out

    def decrypt_round(self, c0r: torch.Tensor,
                      c1r: Optional[torch.Tensor] = None,
                      out: Optional[torch.Tensor] = None, stream=None):
        """m = round(t CRT(c0r + c1r) / Q) mod t over [..][L][len]
        -> int32 view (uint32 values) [..][len]."""
        ln = c0r.shape[-1]
        n = c0r.numel() // (self.L * ln)
        m = out if out is not None else torch.empty(
            *c0r.shape[:-2], ln, dtype=torch.int32, device=self.device)
        self._dev(c0r, c1r)
        _check(_lib.he_decrypt_round(self._h, self._ptr(c0r), self._ptr(c1r),
                                     n, ln, self._ptr(m), _stream(stream)),
               "he_decrypt_round")
        return m

    def mod_switch(self, x: torch.Tensor, L_keep: int,
                   out: Optional[torch.Tensor] = None, stream=None):
        """[..][L][len] -> [..][L_keep][len]: round(Q' x / Q) mod q_j."""
        ln = x.shape[-1]
        n = x.numel() // (self.L * ln)
        if out is None:
            out = self.empty_u64(*x.shape[:-2], L_keep, ln)
        self._dev(x, out)
        _check(_lib.he_mod_switch(self._h, self._ptr(x), n, ln, L_keep,
                                  self._ptr(out), _stream(stream)), "he_mod_switch")
        return out

    # ------------------------------------------ chained pipeline (§8(f))
    def pk_mask(self, v: torch.Tensor, e: Optional[torch.Tensor], b: torch.Tensor,
                out: Optional[torch.Tensor] = None, stream=None):
        """ve = v b + e (Eq. (1)) for int32 v, e [..][N] -> [..][L][N]."""
        n = v.numel() // self.N
        if out is None:
            out = self.empty_u64(*v.shape[:-1], self.L, self.N)
        ws = torch.empty(8 * self.L * self.N, dtype=torch.uint8, device=self.device)
        self._dev(v, e, b, out)
        _check(_lib.he_pk_mask(self._h, self._ptr(v), self._ptr(e), n, self._ptr(b),
                               self._ptr(out), self._ptr(ws), ws.numel(),
                               _stream(stream)), "he_pk_mask")
        return out

    def relu_requant(self, p: ConvPlan, m: torch.Tensor, phi1: Optional[torch.Tensor],
                     shift: int, qmax: int, out: Optional[torch.Tensor] = None,
                     stream=None):
        B = m.shape[0]
        if out is None:
            out = torch.empty(B, p.d.c_o, p.w_o, p.h_o, dtype=torch.int32,
                              device=self.device)
        self._dev(m, phi1, out)
        _check(_lib.he_relu_requant(self._h, ctypes.byref(p), self._ptr(m), B,
                                    self._ptr(phi1), shift, qmax, self._ptr(out),
                                    _stream(stream)), "he_relu_requant")
        return out

    def avgpool(self, x: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None):
        """int32 [B][C][H][W] -> [B][C] floor means."""
        rows, hw = x.shape[0] * x.shape[1], x.shape[2] * x.shape[3]
        if out is None:
            out = torch.empty(x.shape[0], x.shape[1], dtype=torch.int32, device=self.device)
        self._dev(x, out)
        _check(_lib.he_avgpool(self._ptr(x), rows, hw, self._ptr(out), _stream(stream)),
               "he_avgpool")
        return out

    def fc_server_init_p(self, W: torch.Tensor, a: torch.Tensor,
                         e: Optional[torch.Tensor] = None, stream=None):
        n_o, n_i = W.shape
        f = FcDesc(n_i, n_o)
        n_it, n_ib, n_ot, n_t = self.fc_plan(n_i, n_o)
        out = self.empty_u64(n_ib, n_t, self.L, self.N)
        wsb = _lib.he_fc_server_p_workspace_bytes(self._h, ctypes.byref(f))
        ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        self._dev(W, a, e)
        _check(_lib.he_fc_server_init_p(self._h, ctypes.byref(f), self._ptr(W), self._ptr(a),
                                        self._ptr(e), self._ptr(out), self._ptr(ws), wsb,
                                        _stream(stream)), "he_fc_server_init_p")
        return out

    def pack_fc_client_p(self, n_i, n_o, pp: torch.Tensor, stream=None):
        f = FcDesc(n_i, n_o)
        pspec = self.empty_u64(_lib.he_fc_wspec_bytes(self._h, ctypes.byref(f)) // 8)
        ws = torch.empty(8 * pp.numel(), dtype=torch.uint8, device=self.device)
        self._dev(pp)
        _check(_lib.he_pack_fc_client_p(self._h, ctypes.byref(f), self._ptr(pp),
                                        self._ptr(pspec), self._ptr(ws), ws.numel(),
                                        _stream(stream)), "he_pack_fc_client_p")
        return pspec

    def unmask(self, m: torch.Tensor, phi1: Optional[torch.Tensor] = None,
               out: Optional[torch.Tensor] = None, stream=None):
        if out is None:
            out = torch.empty(m.shape, dtype=torch.int32, device=self.device)
        self._dev(m, phi1, out)
        _check(_lib.he_unmask(self._h, self._ptr(m), self._ptr(phi1), m.numel(),
                              self._ptr(out), _stream(stream)), "he_unmask")
        return out

    # --------------------------------- sparse c0 upload (protocol extension)
    def c0_compact(self, p: ConvPlan, c0: torch.Tensor,
                   out: Optional[torch.Tensor] = None, stream=None):
        """[B][n_ib][L][N] -> [B][n_ib][L][M k_u]: the columns the conv reads."""
        B = c0.shape[0]
        if out is None:
            out = self.empty_u64(B, p.n_ib, self.L, (self.N // p.s) * p.k_u)
        self._dev(c0, out)
        _check(_lib.he_c0_compact(self._h, ctypes.byref(p), self._ptr(c0), B,
                                  self._ptr(out), _stream(stream)), "he_c0_compact")
        return out

    def c0_expand(self, p: ConvPlan, c0c: torch.Tensor,
                  out: Optional[torch.Tensor] = None, stream=None):
        B = c0c.shape[0]
        if out is None:
            out = self.empty_u64(B, p.n_ib, self.L, self.N)
        self._dev(c0c, out)
        _check(_lib.he_c0_expand(self._h, ctypes.byref(p), self._ptr(c0c), B,
                                 self._ptr(out), _stream(stream)), "he_c0_expand")
        return out

    def filter_coeffs(self, p: ConvPlan, W: torch.Tensor, shifted: bool = True,
                      stream=None):
        """a2 debug export: [c_o][n_ib][L][N] coefficient-domain f or fhat."""
        out = self.empty_u64(p.d.c_o, p.n_ib, self.L, self.N)
        ws = torch.empty(out.numel() * 8 if shifted else 8, dtype=torch.uint8,
                         device=self.device)
        self._dev(W, out)
        _check(_lib.he_filter_coeffs(self._h, ctypes.byref(p), self._ptr(W), int(shifted),
                                     self._ptr(out), self._ptr(ws), ws.numel(),
                                     _stream(stream)), "he_filter_coeffs")
        return out

    # ------------------------------------- unfolded reference path (ablation)
    def pack_filters_plain(self, p: ConvPlan, W: torch.Tensor, stream=None):
        out = self.empty_u64(p.d.c_o, p.n_ib, self.L, self.N)
        self._dev(W, out)
        _check(_lib.he_pack_filters_plain(self._h, ctypes.byref(p), self._ptr(W),
                                          self._ptr(out), _stream(stream)),
               "he_pack_filters_plain")
        return out

    def conv_plain(self, p: ConvPlan, c0: torch.Tensor, fplain: torch.Tensor,
                   phi1: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                   ws: Optional[torch.Tensor] = None, stream=None):
        B = c0.shape[0]
        if out is None:
            out = self.empty_u64(B, p.n_ob, self.L, self.N)
        if ws is None:
            ws = torch.empty(_lib.he_conv_plain_workspace_bytes(self._h, ctypes.byref(p), B),
                             dtype=torch.uint8, device=self.device)
        self._dev(c0, fplain, phi1, out, ws)
        _check(_lib.he_conv_plain(self._h, ctypes.byref(p), self._ptr(c0), B,
                                  self._ptr(fplain), self._ptr(phi1), self._ptr(out),
                                  self._ptr(ws), ws.numel(), _stream(stream)), "he_conv_plain")
        return out

    def pk_mask_vs(self, v: torch.Tensor, e: Optional[torch.Tensor], b: torch.Tensor,
                   s_res: torch.Tensor, stream=None):
        """(v b + e, v s) for int32 v, e [..][N] -> two [..][L][N] tensors."""
        n = v.numel() // self.N
        ve = self.empty_u64(*v.shape[:-1], self.L, self.N)
        vs = self.empty_u64(*v.shape[:-1], self.L, self.N)
        ws = torch.empty(16 * self.L * self.N, dtype=torch.uint8, device=self.device)
        self._dev(v, e, b, s_res, ve, vs)
        _check(_lib.he_pk_mask_vs(self._h, self._ptr(v), self._ptr(e), n, self._ptr(b),
                                  self._ptr(s_res), self._ptr(ve), self._ptr(vs),
                                  self._ptr(ws), ws.numel(), _stream(stream)), "he_pk_mask_vs")
        return ve, vs
