"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the SPEC-only ``preprocessing`` module (
PAPER.md Alg. 3 "P(o, u, v)" lines 480-530 and Alg. 4): the
mask-bank protocol that moves every HE evaluation of a linear operator to an
offline phase, and the HE-free online training of linear layers.

Operator ids (Alg. 4): for each linear layer
  FWD     u o v      = W  o X           u = W       (MO), v = <X>_1   (DO)
  BWDX    u o_x v    = W  o_x gY        u = W       (MO), v = <gY>_1  (DO)
  GRADW   u (.) v    = gY (.) X         u = <gY>_0  (MO), v = <X>_1   (DO)
  GRADWR  u (.)rev v = v (.) u          u = <X>_0   (MO), v = <gY>_1  (DO)
with FC (W (n_o,n_i), X (n_i,B), gY (n_o,B)) and Conv2d (W (c_o,c_i,s,s),
X (B,c_i,H,W), gY (B,c_o,oh,ow)) shapes.

Bank (Alg. 3 P_prep): MO masks u'_i (i < m), DO masks v'_j, MO masks s_ij;
the HE evaluation u'_i o Enc(v'_j) - s_ij (the same he_eval as Alg. 1/2) is
decrypted by the DO into D_ij = u'_i o v'_j - s_ij.
Online (Alg. 3 steps 7-10): MO draws k_i, sends u~ = u - sum k_i u'_i; DO
draws l_j, sends v~ = v - sum l_j v'_j;
  <u o v>_0 = u o v~ + sum_j l_j sum_i k_i s_ij
  <u o v>_1 = sum_j l_j (u~ o v'_j + sum_i k_i D_ij)
Random streams: prep_stream(layer, op, purpose), the bank is keyed by the
bank seed; k / l by the step seed (Ctx.seed) like every online stream.
"""

from __future__ import annotations

import numpy as np

from . import convops as CO
from . import kernels as OK
from . import packing as PK
from . import protocols as PR
from .ring import RingParams, SeededRng

FWD, BWDX, GRADW, GRADWR = range(4)
OP_NAMES = ("fwd", "bwdx", "gradw", "gradw_rev")
# prep purposes
U_MASK, V_MASK, S_MASK, ENC = range(4)
# online op codes (stream_id(layer, 20 + op, purpose)): purpose 0 = MO scalars k, 1 = DO scalars l
OP_ONLINE = 20


def prep_stream(layer: int, op: int, purpose: int) -> int:
    return 2_000_000 + 1000 * layer + 10 * op + purpose


def _m(v, ring):
    return np.asarray(v, dtype=np.uint64) & ring.mask


class Operator:
    """One linear operator of one layer: shapes, plaintext rule, HE rule."""

    def __init__(self, layer_spec, op: int, B: int, in_hw=None):
        self.spec, self.op, self.B = tuple(layer_spec), op, B
        if layer_spec[0] == "fc":
            _, n_i, n_o = layer_spec
            W, X, G = (n_o, n_i), (n_i, B), (n_o, B)
        else:
            _, c_i, c_o, s, p, st = layer_spec
            H, Wd = in_hw
            oh, ow = PK.conv_out_hw(H, Wd, s, p, st)
            W, X, G = (c_o, c_i, s, s), (B, c_i, H, Wd), (B, c_o, oh, ow)
            self.conv = (B, c_i, c_o, H, Wd, s, p, st)
        self.u_shape, self.v_shape, self.out_shape = {
            FWD: (W, X, G), BWDX: (W, G, X), GRADW: (G, X, W), GRADWR: (X, G, W)}[op]

    @property
    def is_fc(self):
        return self.spec[0] == "fc"

    def apply(self, u, v):
        """The plaintext operator over Z_2^64 (masked by the caller)."""
        if self.is_fc:
            if self.op == FWD:
                return OK.matmul_wrap(u, v)
            if self.op == BWDX:
                return OK.matmul_wrap(np.ascontiguousarray(u.T), v)
            if self.op == GRADW:  # u = gY, v = X
                return OK.matmul_wrap(u, np.ascontiguousarray(v.T))
            return OK.matmul_wrap(v, np.ascontiguousarray(u.T))  # u = X, v = gY
        B, c_i, c_o, H, Wd, s, p, st = self.conv
        if self.op == FWD:
            return CO.conv_fwd(v, u, p, st)
        if self.op == BWDX:
            return CO.conv_bwdx(v, u, H, Wd, p, st)
        if self.op == GRADW:
            return CO.conv_gradw(v, u, s, p, st)
        return CO.conv_gradw(u, v, s, p, st)

    def he(self, ctx: PR.Ctx, u, v, s_mask, enc_rng):
        """DO's decryption of u o Enc(v) - s (the Alg. 1/2 evaluator)."""
        n_out = int(np.prod(self.out_shape))
        if self.is_fc:
            if self.op == FWD:
                n_o, n_i = u.shape
                return PR.he_matmul(ctx, v, None, u, None, PK.MatmulGeometry(n_i, n_o, self.B), s_mask, enc_rng)
            if self.op == BWDX:
                n_o, n_i = u.shape
                return PR.he_matmul(ctx, v, None, np.ascontiguousarray(u.T), None, PK.MatmulGeometry(n_o, n_i, self.B),
                                    s_mask, enc_rng)
            if self.op == GRADW:  # gY (n_o,B) (.) X (n_i,B): v = X^T encrypted, W-role = gY plaintext
                n_o = u.shape[0]
                n_i = v.shape[0]
                return PR.he_matmul(ctx, np.ascontiguousarray(v.T), None, u, None, PK.MatmulGeometry(self.B, n_o, n_i),
                                    s_mask, enc_rng)
            n_i = u.shape[0]  # GRADWR: u = X (MO, plaintext input role), v = gY (DO, encrypted weight role)
            n_o = v.shape[0]
            return PR.he_matmul(ctx, None, np.ascontiguousarray(u.T), None, v, PK.MatmulGeometry(self.B, n_o, n_i),
                                s_mask, enc_rng)
        B, c_i, c_o, H, Wd, s, p, st = self.conv
        kind = ("fwd", "bwdx", "gradw", "gradw")[self.op]
        plan = PK.plan_conv_layer(kind, B, c_i, c_o, H, Wd, s, p, st, ctx.p.N)
        if self.op in (FWD, BWDX):
            out = PR.he_eval(ctx, plan, v, None, u, None, s_mask, n_out, enc_rng)
        elif self.op == GRADW:  # u = gY (W-role plaintext), v = X (encrypted input)
            out = PR.he_eval(ctx, plan, v, None, u, None, s_mask, n_out, enc_rng)
        else:  # GRADWR: u = X (plaintext input role), v = gY (encrypted W-role)
            out = PR.he_eval(ctx, plan, None, u, None, v, s_mask, n_out, enc_rng)
        return out.reshape(self.out_shape)


class MaskBank:
    """Role-split bank of one operator."""

    def __init__(self, opd: Operator, m: int):
        self.opd, self.m = opd, m
        self.u = None   # MO: [m] + u_shape
        self.s = None   # MO: [m, m] + out_shape
        self.v = None   # DO: [m] + v_shape
        self.d = None   # DO: [m, m] + out_shape  (u'_i o v'_j - s_ij)
        self.n_used = 0


def prep_operator(ctx: PR.Ctx, layer: int, opd: Operator, m: int, bank_seed: int) -> MaskBank:  # Alg. 3 P_prep
    ring = ctx.ring
    bank = MaskBank(opd, m)
    g = lambda purpose: SeededRng(bank_seed, prep_stream(layer, opd.op, purpose))  # noqa: E731
    bank.u = g(U_MASK).uniform_ring((m, *opd.u_shape), ring)
    bank.v = g(V_MASK).uniform_ring((m, *opd.v_shape), ring)
    bank.s = g(S_MASK).uniform_ring((m, m, *opd.out_shape), ring)
    bank.d = np.zeros_like(bank.s)
    enc = g(ENC)
    for i in range(m):
        for j in range(m):
            bank.d[i, j] = opd.he(ctx, bank.u[i], bank.v[j], bank.s[i, j], enc)
    return bank


def _lincomb(coefs, tensors, ring):
    acc = np.zeros(tensors.shape[1:], dtype=np.uint64)
    for c, t in zip(coefs, tensors):
        acc = acc + np.uint64(c) * t
    return _m(acc, ring)


def _nonzero_scalars(rng: SeededRng, m: int, ring: RingParams):
    k = rng.uniform_ring((m,), ring)
    return np.where(k == 0, np.uint64(1), k)


def online_shared_product(ctx: PR.Ctx, layer: int, bank: MaskBank, u, v):  # Alg. 3 P_online
    """Shares (MO, DO) of u o v; u held by the MO, v by the DO; no HE."""
    ring, opd, m = ctx.ring, bank.opd, bank.m
    k = _nonzero_scalars(ctx.rng(layer, OP_ONLINE + opd.op, 0), m, ring)  # MO
    ell = _nonzero_scalars(ctx.rng(layer, OP_ONLINE + opd.op, 1), m, ring)  # DO
    u_t = _m(u - _lincomb(k, bank.u, ring), ring)  # MO -> DO: u~, k
    v_t = _m(v - _lincomb(ell, bank.v, ring), ring)  # DO -> MO: v~, l
    # MO: <u o v'_j>_0 = sum_i k_i s_ij ;  <u o v>_0 = u o v~ + sum_j l_j <u o v'_j>_0
    mo = _m(opd.apply(u, v_t), ring)
    do = np.zeros(opd.out_shape, dtype=np.uint64)
    for j in range(m):
        mo = _m(mo + np.uint64(ell[j]) * _lincomb(k, bank.s[:, j], ring), ring)
        # DO: <u o v'_j>_1 = u~ o v'_j + sum_i k_i D_ij
        dj = _m(opd.apply(u_t, bank.v[j]) + _lincomb(k, bank.d[:, j], ring), ring)
        do = _m(do + np.uint64(ell[j]) * dj, ring)
    bank.n_used += 1
    return mo, do


# ---------------------------------------------------------------- Alg. 4 ---

class PrepState:
    """The four banks of every linear layer of a model (Alg. 4 preprocessing)."""

    def __init__(self, ctx: PR.Ctx, model, B: int, m: int = 8, bank_seed: int = 1):
        self.m = m
        self.banks = []
        for l, i in enumerate(model.lin):
            spec = model.layers[i]
            hw = model.io[i][0][1:] if spec[0] == "conv" else None
            self.banks.append([prep_operator(ctx, l, Operator(spec, op, B, hw), m, bank_seed) for op in range(4)])


def prep_linear_forward(ctx, layer, banks, W, b, x_mo, x_do, conv=None):
    """Alg. 4 forward: <Y>_0 = <W o X_1>_0 + W o X_0 + b,  <Y>_1 = <W o X_1>_1."""
    ring = ctx.ring
    p0, p1 = online_shared_product(ctx, layer, banks[FWD], W, x_do)
    loc = banks[FWD].opd.apply(W, x_mo)
    bias = b[:, None] if banks[FWD].opd.is_fc else b[None, :, None, None]
    return _m(p0 + loc + bias, ring), p1


def prep_linear_backward_input(ctx, layer, banks, W, gy_mo, gy_do):
    ring = ctx.ring
    p0, p1 = online_shared_product(ctx, layer, banks[BWDX], W, gy_do)
    return _m(p0 + banks[BWDX].opd.apply(W, gy_mo), ring), p1


def prep_grad_weight(ctx, layer, banks, x_mo, x_do, gy_mo, gy_do, e=None):
    """Alg. 4 weight gradient: cross terms by P_online(.) and P_online(.rev), revealed at the MO (2f)."""
    ring = ctx.ring
    a0, a1 = online_shared_product(ctx, layer, banks[GRADW], gy_mo, x_do)  # <gY>_0 (.) <X>_1
    c0, c1 = online_shared_product(ctx, layer, banks[GRADWR], x_mo, gy_do)  # <X>_0 (.)rev <gY>_1
    opd = banks[GRADW].opd
    hat = _m(a1 + c1 + opd.apply(gy_do, x_do), ring)  # DO
    if e is not None:
        hat = _m(hat + e, ring)
    return _m(hat + a0 + c0 + opd.apply(gy_mo, x_mo), ring)  # MO
