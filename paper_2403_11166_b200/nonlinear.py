"""Non-linear layers with the SPEC's dealer backend ("local
correlated-randomness generator co-resident in test harnesses; fast,
insecure, default for unit tests and benchmarks of non-OT costs").

The OT-based protocols (secure comparison, bit injection) are
outside the hot path this engine accelerates; what the training step needs
from them is their *functionality* on shares, which the dealer provides
exactly: reconstruct, apply, reshare.  The reshare mask comes from the
numpy-identical Philox stream stream_id(layer, op, dealer) on the device,
so every output share matches the CPU oracle bit-for-bit.

    relu_forward     y = DReLU(x) * x, d cached        (SPEC:533-541, 1{x >= 0})
    truncate         faithful: arith_shift(x, bits)
    relu_backward    grad x = d * grad y (no new compare)
    avgpool_forward  local 2x2 window sums, then a 2-bit truncation
    avgpool_backward replicate to the 2x2 window, then a 2-bit truncation
"""

from __future__ import annotations

import torch

from . import _dev, _lib
from .linear_protocols import (OP_POOL_B, OP_POOL_F, OP_RELU, OP_RELU_B, OP_TRUNC_B, OP_TRUNC_F, P_DEALER, Session,
                               _split)
from .ring import DO, MO, RingTensor, ShareTensor


def _dealer(sess: Session, layer: int, op_code: int, kind: int, a: ShareTensor, b: ShareTensor, k: int = 0,
            d_in: torch.Tensor | None = None, want_d: bool = False):
    mo, do = _split(a, b)
    ring = sess.ring
    in_mo, in_do = mo.value.values.contiguous(), do.value.values.contiguous()
    x_mo, x_do = torch.empty_like(in_mo), torch.empty_like(in_do)  # fresh outputs: no input copies
    n = x_mo.numel()
    d_out = torch.empty(x_mo.shape, dtype=torch.uint8, device=x_mo.device) if want_d else None
    rng = sess.rng(layer, op_code, P_DEALER)
    off = rng.reserve(n)
    sd, sp = rng.np_args()
    _lib.call("pb_dealer_op_out", kind, _dev.ptr(in_mo), _dev.ptr(in_do), _dev.ptr(x_mo), _dev.ptr(x_do), n, k,
              _dev.ptr(d_in), _dev.ptr(d_out), sd, sp, rng.stream, off, ring.ell, _dev.stream())
    return x_mo, x_do, d_out


def relu_forward(sess: Session, layer: int, a: ShareTensor, b: ShareTensor):
    x_mo, x_do, d = _dealer(sess, layer, OP_RELU, _lib.DEALER_RELU, a, b, want_d=True)
    s = a.scale
    return (ShareTensor(MO, RingTensor(x_mo, s, sess.ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, sess.ring, _canonical=True)), d)


def truncate(sess: Session, layer: int, a: ShareTensor, b: ShareTensor, bits: int, backward: bool = False):
    op = OP_TRUNC_B if backward else OP_TRUNC_F
    x_mo, x_do, _ = _dealer(sess, layer, op, _lib.DEALER_TRUNC, a, b, k=bits)
    s = a.scale - bits
    return (ShareTensor(MO, RingTensor(x_mo, s, sess.ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, sess.ring, _canonical=True)))


def relu_backward(sess: Session, layer: int, d: torch.Tensor, a: ShareTensor, b: ShareTensor):
    x_mo, x_do, _ = _dealer(sess, layer, OP_RELU_B, _lib.DEALER_SELECT, a, b, d_in=d)
    s = a.scale
    return (ShareTensor(MO, RingTensor(x_mo, s, sess.ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, sess.ring, _canonical=True)))


def _pool_local(op: int, v: torch.Tensor, out_hw, ell: int) -> torch.Tensor:
    B, C, H, W = v.shape
    oh, ow = out_hw
    out = _dev.empty_u64(B, C, oh, ow)
    hh, ww = (H, W) if op == _lib.POOL_SUM else (oh, ow)
    _lib.call("pb_pool2", op, _dev.ptr(v), B * C, hh, ww, ell, _dev.ptr(out), _dev.stream())
    return out


def avgpool_forward(sess: Session, layer: int, a: ShareTensor, b: ShareTensor):
    """AvgPool2 forward: each party sums its 2x2 windows, then
    the sum is truncated by 2 bits (dealer, stream (layer, OP_POOL_F))."""
    mo, do = _split(a, b)
    ring = sess.ring
    B, C, H, W = do.shape
    sm = _pool_local(_lib.POOL_SUM, mo.value.values, (H // 2, W // 2), ring.ell)
    sd = _pool_local(_lib.POOL_SUM, do.value.values, (H // 2, W // 2), ring.ell)
    s = a.scale
    x_mo, x_do, _ = _dealer(sess, layer, OP_POOL_F, _lib.DEALER_TRUNC, ShareTensor(MO, RingTensor(sm, s, ring, _canonical=True)),
                            ShareTensor(DO, RingTensor(sd, s, ring, _canonical=True)), k=2)
    return (ShareTensor(MO, RingTensor(x_mo, s, ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, ring, _canonical=True)))


def avgpool_backward(sess: Session, layer: int, a: ShareTensor, b: ShareTensor):
    """AvgPool2 backward: replicate each gradient to its 2x2 window, then a
    2-bit truncation (dealer, stream (layer, OP_POOL_B))."""
    mo, do = _split(a, b)
    ring = sess.ring
    B, C, h, w = do.shape
    rm = _pool_local(_lib.POOL_REPLICATE, mo.value.values, (2 * h, 2 * w), ring.ell)
    rd = _pool_local(_lib.POOL_REPLICATE, do.value.values, (2 * h, 2 * w), ring.ell)
    s = a.scale
    x_mo, x_do, _ = _dealer(sess, layer, OP_POOL_B, _lib.DEALER_TRUNC, ShareTensor(MO, RingTensor(rm, s, ring, _canonical=True)),
                            ShareTensor(DO, RingTensor(rd, s, ring, _canonical=True)), k=2)
    return (ShareTensor(MO, RingTensor(x_mo, s, ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, ring, _canonical=True)))


def relu_truncate(sess: Session, layer: int, a: ShareTensor, b: ShareTensor, bits: int):
    """ReLU followed by the forward truncation in ONE dealer round: the
    output shares are the truncation's reshare (stream (layer, OP_TRUNC_F)) of
    arith_shift(relu(x), bits) -- exactly the two-step composition's, since the
    ReLU's own reshare is consumed by the truncation and never observed."""
    x_mo, x_do, d = _dealer(sess, layer, OP_TRUNC_F, _lib.DEALER_RELU_TRUNC, a, b, k=bits, want_d=True)
    s = a.scale - bits
    return (ShareTensor(MO, RingTensor(x_mo, s, sess.ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, sess.ring, _canonical=True)), d)


def truncate_relu_backward(sess: Session, layer_relu: int, d: torch.Tensor, a: ShareTensor, b: ShareTensor,
                           bits: int):
    """Backward truncation of grad X followed by ReLU' (cached d) in ONE dealer
    round; output shares = the ReLU-backward reshare (stream (layer_relu,
    OP_RELU_B)) of d * arith_shift(x, bits), as the two-step composition."""
    x_mo, x_do, _ = _dealer(sess, layer_relu, OP_RELU_B, _lib.DEALER_TRUNC_SELECT, a, b, k=bits, d_in=d)
    s = a.scale - bits
    return (ShareTensor(MO, RingTensor(x_mo, s, sess.ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, sess.ring, _canonical=True)))
