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
"""

from __future__ import annotations

import torch

from . import _dev, _lib
from .linear_protocols import OP_RELU, OP_RELU_B, OP_TRUNC_B, OP_TRUNC_F, P_DEALER, Session, _split
from .ring import DO, MO, RingTensor, ShareTensor


def _dealer(sess: Session, layer: int, op_code: int, kind: int, a: ShareTensor, b: ShareTensor, k: int = 0,
            d_in: torch.Tensor | None = None, want_d: bool = False):
    mo, do = _split(a, b)
    ring = sess.ring
    x_mo = mo.value.values.clone()
    x_do = do.value.values.clone()
    n = x_mo.numel()
    d_out = torch.empty(x_mo.shape, dtype=torch.uint8, device=x_mo.device) if want_d else None
    rng = sess.rng(layer, op_code, P_DEALER)
    off = rng.reserve(n)
    sd, sp = rng.np_args()
    _lib.call("pb_dealer_op", kind, _dev.ptr(x_mo), _dev.ptr(x_do), n, k, _dev.ptr(d_in), _dev.ptr(d_out), sd, sp,
              rng.stream, off, ring.ell, _dev.stream())
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
