"""Non-linear layers with two backends, chosen by
``Session.nonlinear``:

* "dealer" (default; "local correlated-randomness generator
  co-resident in test harnesses; fast, insecure, default for unit tests and
  benchmarks of non-OT costs"): reconstruct, apply, reshare -- the reshare
  mask from the numpy-identical Philox stream stream_id(layer, op, dealer);
* "ot": the protocols themselves (csrc/pb_nonlinear.cu) -- secure comparison
  in 4-bit blocks with 1-of-16 leaf OTs and a Beaver-AND tree, DReLU from the
  MSBs + one comparison, bit injection (MUX) with two 1-of-2 OTs, faithful
  truncation by the wrap / low-carry comparisons + B2A -- with SPEC:479's
  dealer OT functionality, all parties' share arithmetic on the device, one
  thread per element; randomness from the stream (layer, op, P_OT).
Both backends reconstruct to the same values, so training steps are
bit-identical to the reference engine either way; every output share
matches the CPU oracle (oracle/protocols.py, oracle/nonlinear.py) bit-for-bit.

    relu_forward     y = DReLU(x) * x, d cached        (SPEC:533-541, 1{x >= 0})
    truncate         faithful: arith_shift(x, bits)
    relu_backward    grad x = d * grad y (no new compare)
    avgpool_forward  local 2x2 window sums, then a 2-bit truncation
    avgpool_backward replicate to the 2x2 window, then a 2-bit truncation
"""

from __future__ import annotations

import torch

from . import _dev, _lib
from .linear_protocols import (OP_POOL_B, OP_POOL_F, OP_RELU, OP_RELU_B, OP_TRUNC_B, OP_TRUNC_F, P_DEALER, P_OT,
                               Session, _split)
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


MSG_NL = 0x60  # SPEC:581 message codes 0x60-0x6F


def _ot_bytes(op: int, ell: int, k: int) -> int:
    """Per-element protocol payload a two-process run sends (census): per
    comparison over n bits, q = ceil(n/4) 1-of-16 OTs of 2-bit messages (16 x 2
    bits from the sender) plus 2 (q - 1) Beaver ANDs opening 2 bits each way;
    per MUX two 1-of-2 OTs of ell-bit messages each way."""
    def cmp(nb):
        q = (nb + 3) // 4
        return 4 * q + (q - 1)
    mux = 2 * 2 * ((ell + 7) // 8)
    trunc = cmp(ell) + cmp(k) + 2 * mux
    return {_lib.NL_DRELU: cmp(ell - 1), _lib.NL_MUX: mux, _lib.NL_TRUNC: trunc,
            _lib.NL_RELU_TRUNC: cmp(ell - 1) + mux + trunc, _lib.NL_TRUNC_MUX: trunc + mux}[op]


def _ot(sess: Session, layer: int, op_code: int, kind: int, a: ShareTensor, b: ShareTensor, k: int = 0,
        d_in: torch.Tensor | None = None, want_d: bool = False):
    """One OT-protocol op over all elements (pb_nl_op): MO = party 0, DO = party 1."""
    mo, do = _split(a, b)
    ring = sess.ring
    in_mo, in_do = mo.value.values.contiguous(), do.value.values.contiguous()
    n = in_mo.numel()
    y_mo = torch.empty_like(in_mo) if kind != _lib.NL_DRELU else None
    y_do = torch.empty_like(in_do) if kind != _lib.NL_DRELU else None
    d_out = torch.empty(in_mo.shape, dtype=torch.uint8, device=in_mo.device) if want_d else None
    rng = sess.rng(layer, op_code, P_OT)
    off = rng.reserve(n * int(_lib.load().pb_nl_words(kind)))
    sd, sp = rng.np_args()
    _lib.call("pb_nl_op", kind, _dev.ptr(in_mo), _dev.ptr(in_do), n, ring.ell, k, _dev.ptr(d_in), _dev.ptr(d_out), sd,
              sp, rng.stream, off, _dev.ptr(y_mo), _dev.ptr(y_do), _dev.stream())
    sess.channel.send(MO, MSG_NL, None, n * _ot_bytes(kind, ring.ell, k))
    return y_mo, y_do, d_out


def _nl(sess: Session, layer: int, op_code: int, dealer_kind: int, ot_kind: int, a, b, k=0, d_in=None,
        want_d=False):
    if sess.nonlinear == "ot":
        return _ot(sess, layer, op_code, ot_kind, a, b, k=k, d_in=d_in, want_d=want_d)
    return _dealer(sess, layer, op_code, dealer_kind, a, b, k=k, d_in=d_in, want_d=want_d)


def relu_forward(sess: Session, layer: int, a: ShareTensor, b: ShareTensor):
    if sess.nonlinear == "ot":  # DReLU, then the MUX on the same stream
        _, _, d = _ot(sess, layer, OP_RELU, _lib.NL_DRELU, a, b, want_d=True)
        x_mo, x_do, _ = _ot(sess, layer, OP_RELU, _lib.NL_MUX, a, b, d_in=d)
        s = a.scale
        return (ShareTensor(MO, RingTensor(x_mo, s, sess.ring, _canonical=True)),
                ShareTensor(DO, RingTensor(x_do, s, sess.ring, _canonical=True)), d)
    x_mo, x_do, d = _dealer(sess, layer, OP_RELU, _lib.DEALER_RELU, a, b, want_d=True)
    s = a.scale
    return (ShareTensor(MO, RingTensor(x_mo, s, sess.ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, sess.ring, _canonical=True)), d)


def truncate(sess: Session, layer: int, a: ShareTensor, b: ShareTensor, bits: int, backward: bool = False):
    op = OP_TRUNC_B if backward else OP_TRUNC_F
    x_mo, x_do, _ = _nl(sess, layer, op, _lib.DEALER_TRUNC, _lib.NL_TRUNC, a, b, k=bits)
    s = a.scale - bits
    return (ShareTensor(MO, RingTensor(x_mo, s, sess.ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, sess.ring, _canonical=True)))


def relu_backward(sess: Session, layer: int, d: torch.Tensor, a: ShareTensor, b: ShareTensor):
    x_mo, x_do, _ = _nl(sess, layer, OP_RELU_B, _lib.DEALER_SELECT, _lib.NL_MUX, a, b, d_in=d)
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
    x_mo, x_do, _ = _nl(sess, layer, OP_POOL_F, _lib.DEALER_TRUNC, _lib.NL_TRUNC,
                        ShareTensor(MO, RingTensor(sm, s, ring, _canonical=True)),
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
    x_mo, x_do, _ = _nl(sess, layer, OP_POOL_B, _lib.DEALER_TRUNC, _lib.NL_TRUNC,
                        ShareTensor(MO, RingTensor(rm, s, ring, _canonical=True)),
                        ShareTensor(DO, RingTensor(rd, s, ring, _canonical=True)), k=2)
    return (ShareTensor(MO, RingTensor(x_mo, s, ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, ring, _canonical=True)))


def relu_truncate(sess: Session, layer: int, a: ShareTensor, b: ShareTensor, bits: int):
    """ReLU followed by the forward truncation in ONE dealer round: the
    output shares are the truncation's reshare (stream (layer, OP_TRUNC_F)) of
    arith_shift(relu(x), bits) -- exactly the two-step composition's, since the
    ReLU's own reshare is consumed by the truncation and never observed."""
    x_mo, x_do, d = _nl(sess, layer, OP_TRUNC_F, _lib.DEALER_RELU_TRUNC, _lib.NL_RELU_TRUNC, a, b, k=bits,
                        want_d=True)
    s = a.scale - bits
    return (ShareTensor(MO, RingTensor(x_mo, s, sess.ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, sess.ring, _canonical=True)), d)


def truncate_relu_backward(sess: Session, layer_relu: int, d: torch.Tensor, a: ShareTensor, b: ShareTensor,
                           bits: int):
    """Backward truncation of grad X followed by ReLU' (cached d) in ONE dealer
    round; output shares = the ReLU-backward reshare (stream (layer_relu,
    OP_RELU_B)) of d * arith_shift(x, bits), as the two-step composition."""
    x_mo, x_do, _ = _nl(sess, layer_relu, OP_RELU_B, _lib.DEALER_TRUNC_SELECT, _lib.NL_TRUNC_MUX, a, b, k=bits,
                        d_in=d)
    s = a.scale - bits
    return (ShareTensor(MO, RingTensor(x_mo, s, sess.ring, _canonical=True)),
            ShareTensor(DO, RingTensor(x_do, s, sess.ring, _canonical=True)))
