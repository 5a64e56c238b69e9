"""Pencil+ preprocessing on the B200: the mask-bank protocol (the SPEC-only
``preprocessing`` module; Alg. 3,
Alg. 4).

Offline (P_prep, once per operator): the MO draws masks u'_i and s_ij, the DO
draws v'_j; the MO evaluates u'_i o Enc(v'_j) - s_ij with the SAME fused
evaluator as Alg. 1/2 (Session.he_matmul / he_eval: encrypt, TMA-pipelined
ct x pt MAC, mask NTT, decrypt-to-share) and the DO keeps the decryptions
D_ij = u'_i o v'_j - s_ij.  m^2 evaluations per operator -- the GPU-heavy,
data-independent part.

Online (P_online, every step): no HE at all --
  MO draws k_i, sends u~ = u - sum_i k_i u'_i        (pb_ring_lincomb)
  DO draws l_j, sends v~ = v - sum_j l_j v'_j        (pb_ring_lincomb)
  <u o v>_0 = u o v~ + sum_ij k_i l_j s_ij           (ring GEMM / conv + lincomb)
  <u o v>_1 = u~ o (v - v~) + sum_ij k_i l_j D_ij    (bilinearity: sum_j l_j u~ o v'_j)
The four operators per linear layer (Alg. 4): FWD u o v = W o <X>_1, BWDX
W o_x <gY>_1, GRADW <gY>_0 (.) <X>_1, GRADWR <X>_0 (.)rev <gY>_1.

Masks, k and l come from the same numpy-identical Philox streams as the
oracle (oracle/preprocessing.py), and the banks' decrypted entries do not
depend on the HE randomness, so banks and online shares are
bit-identical to the oracle's.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .errors import ShapeError
from .linear_protocols import _ring_conv, _ring_matmul, _split
from .poly_encoding import MatmulGeometry, conv_out_hw, plan_conv_layer
from .ring import DO, MO, RingTensor, SeededRng, ShareTensor

FWD, BWDX, GRADW, GRADWR = range(4)
U_MASK, V_MASK, S_MASK, ENC = range(4)
OP_ONLINE = 20   # online scalar streams: stream_id(layer, 20 + op, 0 = MO's k / 1 = DO's l)
OP_PREP = 40     # HE evaluations of the offline phase: stream_id(layer, 40 + op, purpose)
MSG_PREP_CT = 0x40      # DO -> MO Enc(v'_j)             (offline)
MSG_PREP_MASKED = 0x41  # MO -> DO Enc(u'_i o v'_j - s)   (offline)
MSG_ONLINE_U = 0x42     # MO -> DO u~, k                  (online)
MSG_ONLINE_V = 0x43     # DO -> MO v~, l                  (online)


def prep_stream(layer: int, op: int, purpose: int) -> int:
    return 2_000_000 + 1000 * layer + 10 * op + purpose


class Operator:
    """One linear operator of one layer (SPEC:384 OperatorDescriptor)."""

    def __init__(self, layer_spec, op: int, B: int, in_hw=None):
        self.spec, self.op, self.B = tuple(layer_spec), op, B
        if layer_spec[0] == "fc":
            _, n_i, n_o = layer_spec
            W, X, G = (n_o, n_i), (n_i, B), (n_o, B)
            self.fc = (n_i, n_o)
        else:
            _, c_i, c_o, s, p, st = layer_spec
            H, Wd = in_hw
            oh, ow = conv_out_hw(H, Wd, s, p, st)
            W, X, G = (c_o, c_i, s, s), (B, c_i, H, Wd), (B, c_o, oh, ow)
            self.conv = (B, c_i, c_o, H, Wd, s, p, st)
        self.u_shape, self.v_shape, self.out_shape = {
            FWD: (W, X, G), BWDX: (W, G, X), GRADW: (G, X, W), GRADWR: (X, G, W)}[op]

    @property
    def is_fc(self):
        return self.spec[0] == "fc"

    def apply(self, u: torch.Tensor, v: torch.Tensor, ell: int, c: torch.Tensor | None = None) -> torch.Tensor:
        """The plaintext operator on the device, mod 2^ell; ``c``: + c (fused
        into the FC GEMM's epilogue)."""
        if self.is_fc:
            n_i, n_o = self.fc
            B = self.B
            kw = dict(c=c, sign=1) if c is not None else {}
            if self.op == FWD:
                return _ring_matmul(u, v, n_o, n_i, B, ell, **kw)
            if self.op == BWDX:
                return _ring_matmul(u, v, n_i, n_o, B, ell, ta=True, **kw)
            if self.op == GRADW:  # gY (n_o,B) X^T
                return _ring_matmul(u, v, n_o, B, n_i, ell, tb=True, **kw)
            return _ring_matmul(v, u, n_o, B, n_i, ell, tb=True, **kw)  # u = X, v = gY
        B, c_i, c_o, H, Wd, s, p, st = self.conv
        args = (B, c_i, c_o, H, Wd, s, p, st, ell)
        if self.op == FWD:
            out = _ring_conv(_lib.CONV_FWD, v, u, *args, self.out_shape)
        elif self.op == BWDX:
            out = _ring_conv(_lib.CONV_BWDX, v, u, *args, self.out_shape)
        elif self.op == GRADW:
            out = _ring_conv(_lib.CONV_GRADW, v, u, *args, self.out_shape)
        else:
            out = _ring_conv(_lib.CONV_GRADW, u, v, *args, self.out_shape)
        return out if c is None else _add(out, c, ell)

    def he(self, sess, layer: int, u: torch.Tensor, v: torch.Tensor, s_mask: torch.Tensor) -> torch.Tensor:
        """DO's decryption of u o Enc(v) - s through the Alg. 1/2 evaluator."""
        out = _dev.empty_u64(*self.out_shape)
        op = OP_PREP + self.op
        kw = dict(msg_in=MSG_PREP_CT, msg_out=MSG_PREP_MASKED)
        if self.is_fc:
            n_i, n_o = self.fc
            B = self.B
            if self.op == FWD:
                sess.he_matmul(layer, op, MatmulGeometry(n_i, n_o, B), out, s_mask, v_ct=v, w_pt=u, **kw)
            elif self.op == BWDX:
                sess.he_matmul(layer, op, MatmulGeometry(n_o, n_i, B), out, s_mask, v_ct=v, w_pt=u,
                               w_strides=(1, n_i), **kw)
            elif self.op == GRADW:  # v = X read as X^T (B x n_i), W-role = gY
                sess.he_matmul(layer, op, MatmulGeometry(B, n_o, n_i), out, s_mask, v_ct=v, v_strides=(1, B), w_pt=u,
                               **kw)
            else:  # GRADWR: W-role gY encrypted (DO), input-role X^T plaintext (MO)
                sess.he_matmul(layer, op, MatmulGeometry(B, n_o, n_i), out, s_mask, w_ct=v, v_pt=u, v_strides=(1, B),
                               **kw)
            return out
        B, c_i, c_o, H, Wd, s, p, st = self.conv
        kind = ("fwd", "bwdx", "gradw", "gradw")[self.op]
        plan = plan_conv_layer(kind, B, c_i, c_o, H, Wd, s, p, st, sess.p.N)
        if self.op == GRADWR:
            sess.he_eval(layer, op, plan, out, s_mask, w_ct=v, v_pt=u, **kw)
        else:
            sess.he_eval(layer, op, plan, out, s_mask, v_ct=v, w_pt=u, **kw)
        return out


class MaskBank:
    """Role-split bank of one operator: MO holds u'[m], s[m][m];
    the DO holds v'[m], D[m][m] = u'_i o v'_j - s_ij.  Device tensors."""

    def __init__(self, opd: Operator, m: int):
        self.opd, self.m = opd, m
        self.u = self.s = self.v = self.d = None
        self.n_used = 0


def prep_operator(sess, layer: int, opd: Operator, m: int, bank_seed: int) -> MaskBank:  # Alg. 3 P_prep
    ring = sess.ring
    if m < 1 or m > 16:
        raise ShapeError("mask count m must be in [1, 16]")
    bank = MaskBank(opd, m)

    def g(purpose):
        return SeededRng(bank_seed, prep_stream(layer, opd.op, purpose))

    bank.u = g(U_MASK).uniform_ring((m, *opd.u_shape), ring)
    bank.v = g(V_MASK).uniform_ring((m, *opd.v_shape), ring)
    bank.s = g(S_MASK).uniform_ring((m, m, *opd.out_shape), ring)
    bank.d = torch.empty_like(bank.s)
    for i in range(m):
        for j in range(m):
            bank.d[i, j].copy_(opd.he(sess, layer, bank.u[i].contiguous(), bank.v[j].contiguous(),
                                      bank.s[i, j].contiguous()))
    return bank


def _lincomb(out, base, a, b, T, ell, subtract):
    ma = a.numel()
    mb = 1 if b is None else b.numel()
    n = out.numel()
    _lib.call("pb_ring_lincomb", 1 if subtract else 0, _dev.ptr(out), _dev.ptr(base), _dev.ptr(a), ma, _dev.ptr(b), mb,
              _dev.ptr(T), n, ell, _dev.stream())
    return out


def _scalars(sess, layer: int, op: int, m: int):
    """(k, l): the MO's and the DO's nonzero online scalars (streams
    (layer, OP_ONLINE + op, 0 / 1)), one launch."""
    rk, rl = sess.rng(layer, OP_ONLINE + op, 0), sess.rng(layer, OP_ONLINE + op, 1)
    k, lj = _dev.empty_u64(m), _dev.empty_u64(m)
    seed, sptr = rk.np_args()
    rk.reserve(m)
    rl.reserve(m)
    _lib.call("pb_prep_scalars", _dev.ptr(k), _dev.ptr(lj), m, seed, sptr, rk.stream, rl.stream, sess.ring.ell,
              _dev.stream())
    return k, lj


def online_shared_product(sess, layer: int, bank: MaskBank, u: torch.Tensor, v: torch.Tensor):  # Alg. 3 P_online
    """(MO share, DO share) of u o v with u at the MO, v at the DO: no HE.
    The MO's chain (u~, then u o v~ + sum k_i l_j s_ij) runs on the calling
    stream, the DO's (sum_j l_j v'_j, v~ = v - that, then u~ o (v - v~) +
    sum k_i l_j D_ij) on an auxiliary stream; each waits only for the message
    it receives.  The mask-weighted sums are folded into the FC GEMMs'
    epilogues."""
    ring, opd, m = sess.ring, bank.opd, bank.m
    ell = ring.ell
    if tuple(u.shape) != opd.u_shape or tuple(v.shape) != opd.v_shape:
        raise ShapeError(f"bank expects u {opd.u_shape}, v {opd.v_shape}")
    k, lj = _scalars(sess, layer, opd.op, m)
    main = torch.cuda.current_stream()
    # every buffer is allocated on the calling stream before the fork (the aux
    # stream waits for it; the join orders any reuse after the aux work)
    vmask, v_t, u_t = torch.empty_like(v), torch.empty_like(v), torch.empty_like(u)
    t_d, t_s = _dev.empty_u64(*opd.out_shape), _dev.empty_u64(*opd.out_shape)
    with sess.aux() as aux:
        def do_side():  # DO: sum_j l_j v'_j (= v - v~), then v~ = v - it; sum k_i l_j D_ij
            _lincomb(vmask, None, lj, None, bank.v, ell, False)
            _lib.call("pb_ring_binary", _lib.RING_SUB, _dev.ptr(v_t), _dev.ptr(v), _dev.ptr(vmask), v.numel(),
                      v.numel(), ell, _dev.stream())
            _lincomb(t_d, None, k, lj, bank.d, ell, False)
            ev = torch.cuda.Event()
            ev.record()
            return ev
        ev_vt = aux.run(do_side)
        _lincomb(u_t, u, k, None, bank.u, ell, True)  # MO -> DO: u~, k
        sess.channel.send(MO, MSG_ONLINE_U, u_t, 8 * (u_t.numel() + m))
        sess.channel.send(DO, MSG_ONLINE_V, v_t, 8 * (v_t.numel() + m))  # DO -> MO: v~, l
        _lincomb(t_s, None, k, lj, bank.s, ell, False)
        ev_ut = torch.cuda.Event()
        ev_ut.record(main)
        main.wait_event(ev_vt)
        mo = opd.apply(u, v_t, ell, c=t_s)  # MO: u o v~ + sum k_i l_j s_ij
        aux.stream.wait_event(ev_ut)
        do = aux.run(lambda: opd.apply(u_t, vmask, ell, c=t_d))  # DO: u~ o (v - v~) + sum k_i l_j D_ij
    bank.n_used += 1
    return mo, do


# ---------------------------------------------------------------- Alg. 4 ---

class PrepState:
    """The four banks (o, o_x, (.), (.)rev) of every linear layer of a model."""

    def __init__(self, sess, model, B: int, m: int = 8, bank_seed: int = 1):
        self.m = m
        self.banks = []
        for l, i in enumerate(model.lin):
            spec = model.layers[i]
            hw = model.io[i][0][1:] if spec[0] == "conv" else None
            self.banks.append([prep_operator(sess, l, Operator(spec, op, B, hw), m, bank_seed) for op in range(4)])


def _add(a, b, ell):
    out = torch.empty_like(a)
    _lib.call("pb_ring_binary", _lib.RING_ADD, _dev.ptr(out), _dev.ptr(a), _dev.ptr(b), a.numel(), a.numel(), ell,
              _dev.stream())
    return out


def prep_linear_forward(sess, layer: int, banks, W: RingTensor, b: RingTensor, x_a: ShareTensor, x_b: ShareTensor,
                        mo_x_zero: bool = False):
    """Alg. 4 forward: <Y>_0 = <W o X_1>_0 + W o X_0 + b,  <Y>_1 = <W o X_1>_1 (scale 2f).
    ``mo_x_zero``: the MO's input share is zero (the first layer): no W o X_0."""
    x_mo, x_do = _split(x_a, x_b)
    ring = sess.ring
    opd = banks[FWD].opd
    p0, p1 = online_shared_product(sess, layer, banks[FWD], W.values, x_do.value.values)
    from .linear_protocols import _add_bcast

    inner = p0.shape[1] if opd.is_fc else p0.shape[2] * p0.shape[3]
    if not mo_x_zero:
        p0 = opd.apply(W.values, x_mo.value.values, ring.ell, c=p0)  # the add fused into the FC GEMM
    y0 = _add_bcast(p0, b.values, inner, ring.ell)
    return (ShareTensor(MO, RingTensor(y0, 2 * ring.f, ring, _canonical=True)),
            ShareTensor(DO, RingTensor(p1, 2 * ring.f, ring, _canonical=True)))


def prep_linear_backward_input(sess, layer: int, banks, W: RingTensor, gy_a: ShareTensor, gy_b: ShareTensor,
                               mo_gy_zero: bool = False):
    gy_mo, gy_do = _split(gy_a, gy_b)
    ring = sess.ring
    p0, p1 = online_shared_product(sess, layer, banks[BWDX], W.values, gy_do.value.values)
    g0 = p0 if mo_gy_zero else banks[BWDX].opd.apply(W.values, gy_mo.value.values, ring.ell, c=p0)
    return (ShareTensor(MO, RingTensor(g0, 2 * ring.f, ring, _canonical=True)),
            ShareTensor(DO, RingTensor(p1, 2 * ring.f, ring, _canonical=True)))


def prep_grad_weight(sess, layer: int, banks, x_a: ShareTensor, x_b: ShareTensor, gy_a: ShareTensor,
                     gy_b: ShareTensor, e: torch.Tensor | None = None, mo_x_zero: bool = False,
                     mo_gy_zero: bool = False) -> RingTensor:
    """Alg. 4 weight gradient, revealed at the MO (scale 2f).  A cross term with
    a zero MO share (``mo_gy_zero``: <gY>_0 (.) <X>_1 at the last layer,
    ``mo_x_zero``: <X>_0 (.)rev <gY>_1 at the first) is zero and skipped, as is
    the MO's local term then; the adds ride the FC GEMM epilogues."""
    x_mo, x_do = _split(x_a, x_b)
    gy_mo, gy_do = _split(gy_a, gy_b)
    ring = sess.ring
    ell = ring.ell
    opd = banks[GRADW].opd
    terms0, terms1 = [], []
    if not mo_gy_zero:
        a0, a1 = online_shared_product(sess, layer, banks[GRADW], gy_mo.value.values, x_do.value.values)
        terms0.append(a0)
        terms1.append(a1)
    if not mo_x_zero:
        c0, c1 = online_shared_product(sess, layer, banks[GRADWR], x_mo.value.values, gy_do.value.values)
        terms0.append(c0)
        terms1.append(c1)
    acc1 = terms1[0] if len(terms1) == 1 else _add(*terms1, ell) if terms1 else None
    hat = opd.apply(gy_do.value.values, x_do.value.values, ell, c=acc1)  # DO: + local term
    if e is not None:
        hat = _add(hat, e, ell)
    from .linear_protocols import MSG_GRADW

    sess.channel.send(DO, MSG_GRADW, hat, hat.numel() * 8)
    out = hat
    for t in terms0:  # MO: + its shares of the cross terms
        out = _add(out, t, ell)
    if not (mo_x_zero or mo_gy_zero):
        out = opd.apply(gy_mo.value.values, x_mo.value.values, ell, c=out)  # + the MO's local term
    return RingTensor(out, 2 * ring.f, ring, _canonical=True)
