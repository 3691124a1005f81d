"""Chained pipeline (Fig. 5):
layer after layer, the client encrypts (c0 only, Eq. (1)), the server runs
the rotation-free Conv (Alg. 1) or FC (Alg. 2) with its mask phi1, the
client computes its share c1^r and decrypts, and the trusted GC stub (R29)
unmasks, applies ReLU + requantisation and re-packs the activations for the
next layer.  Orchestration only: every step is a call into
libhe_rotfree.so (he_pk_mask_vs, he_pack_input, he_phi1_generate, he_conv,
he_decrypt_round, he_relu_requant, he_avgpool, he_fc,
he_unmask).  Randomness (v, e0, the server's e_f) is supplied by the caller
as device tensors, so runs are reproducible and comparable with the oracle.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch


class Chain:
    """Server and client state of one network on one context.

    layers: synth.ConvLayer list; Ws: int32 device tensors [c_o][c_i][3][3];
    fcW int32 [n_o][n_i] / fcB int32 [n_o] device tensors or None;
    s_key int32 [N], a / b_pk uint64 (int64 view) [L][N] device tensors;
    ef: per layer int32 [c_o][n_ib][N] (server noise of p), ef_fc int32
    [n_ib][n_t][N] or None."""

    def __init__(self, ctx, layers, Ws, fcW, fcB, s_key, a, b_pk, ef, ef_fc=None):
        self.ctx = ctx
        self.layers = list(layers)
        self.plans = [ctx.plan(Ly.c_i, Ly.c_o, Ly.w_i, Ly.h_i, Ly.f_w, Ly.f_h, Ly.stride,
                               Ly.pad) for Ly in self.layers]
        self.b_pk = b_pk
        # server initialisation: filter spectra (Alg. 1 Line 4) and p (Line 5)
        self.fspecs = [ctx.pack_filters(p, W) for p, W in zip(self.plans, Ws)]
        self.dplans = [ctx.dense_plan(p) for p in self.plans]   # client operand is dense
        self.pspecs = [ctx.pack_client_p(p, ctx.server_init_p(p, W, a, e))
                       for p, W, e in zip(self.plans, Ws, ef)]
        self.s_res = ctx.residues_from_int(s_key.reshape(1, -1)).reshape(ctx.L, ctx.N)
        self.fc = None
        if fcW is not None:
            n_o, n_i = fcW.shape
            wspec, benc = ctx.fc_pack_weights(fcW, fcB)
            pspec = ctx.pack_fc_client_p(n_i, n_o, ctx.fc_server_init_p(fcW, a, ef_fc))
            self.fc = dict(n_i=n_i, n_o=n_o, wspec=wspec, benc=benc, pspec=pspec,
                           zero=torch.zeros(ctx.L, n_o, dtype=torch.int64,
                                            device=ctx.device))

    def run(self, img: torch.Tensor, v: Sequence[torch.Tensor], e0: Sequence[torch.Tensor],
            phi_seed: int, shift: int, qmax: int, v_fc: Optional[torch.Tensor] = None,
            e0_fc: Optional[torch.Tensor] = None, keep: bool = False):
        """img int32 [B][c_i][w][h]; v[l], e0[l] int32 [B][n_ib][N] per layer.
        Returns (activations per layer if keep else [last], logits or None)."""
        ctx = self.ctx
        B = img.shape[0]
        acts: List[torch.Tensor] = []
        x = img
        for li, p in enumerate(self.plans):
            # client: c0-only encryption of the packed activations
            ve, vs = ctx.pk_mask_vs(v[li], e0[li], self.b_pk, self.s_res)
            c0 = ctx.pack_input(p, x, ve)
            # server: conv + mask, compact payload only
            phi = torch.empty(B, p.n_ob, ctx.N, dtype=torch.int32, device=ctx.device)
            ctx.phi1_generate(phi_seed * 1000 + li, phi)
            comp0 = ctx.empty_u64(B, p.n_ob, ctx.L, p.n_valid)
            ctx.conv(p, c0, self.fspecs[li], phi, compact=comp0, full=False)
            # client: share c1^r, decryption, GC stub
            comp1 = ctx.empty_u64(B, p.n_ob, ctx.L, p.n_valid)
            ctx.conv(self.dplans[li], vs, self.pspecs[li], None, compact=comp1, full=False)
            m = ctx.decrypt_round(comp0, comp1)
            x = ctx.relu_requant(p, m, phi, shift, qmax)
            if keep or li == len(self.plans) - 1:
                acts.append(x)
        logits = None
        if self.fc is not None:
            f = self.fc
            xin = ctx.avgpool(x)
            ve, vs = ctx.pk_mask_vs(v_fc, e0_fc, self.b_pk, self.s_res)
            c0 = ctx.fc_pack_input(f["n_i"], f["n_o"], xin, ve)
            phi = torch.empty(B, f["n_o"], dtype=torch.int32, device=ctx.device)
            ctx.phi1_generate(phi_seed * 1000 + 999, phi)
            out0 = ctx.fc(f["n_i"], f["n_o"], c0, f["wspec"], f["benc"], phi)
            out1 = ctx.fc(f["n_i"], f["n_o"], vs, f["pspec"], f["zero"], None)
            logits = ctx.unmask(ctx.decrypt_round(out0, out1), phi)
        return acts, logits
