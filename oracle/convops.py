"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plaintext Z_2^64 conv-layer operators with padding / stride (the local
terms of the conv protocols and the reference engine's arithmetic), built
from the reference's valid-mode stride-1 ``conv2d_wrap`` (K:260-278,
restated in oracle/kernels.c) plus data-movement-only transforms (zero
padding, stride subsampling, zero-stuffing dilation, kernel flip, channel /
batch transposition) -- SPEC:284, 286.  Index conventions match
oracle/packing.conv_index_maps:

    fwd    Y[b,o,y,x]  = sum_{c,i,j} W[o,c,i,j] Xpad[b,c,y*st+i,x*st+j]
    bwdx   dX          = the adjoint of fwd in X
    gradw  dW[o,c,i,j] = sum_{b,y,x} dY[b,o,y,x] Xpad[b,c,y*st+i,x*st+j]

AvgPool2: forward = local 2x2 window sums (the 2-bit
truncation is a separate protocol step), backward = replicate each gradient
to its 4 positions.
"""

from __future__ import annotations

import numpy as np

from . import kernels as OK
from .packing import conv_out_hw


def _u(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def pad(x, p):
    if p == 0:
        return _u(x)
    return _u(np.pad(np.asarray(x, dtype=np.uint64), ((0, 0), (0, 0), (p, p), (p, p))))


def dilate(x, st):
    if st == 1:
        return _u(x)
    B, C, h, w = x.shape
    out = np.zeros((B, C, (h - 1) * st + 1, (w - 1) * st + 1), dtype=np.uint64)
    out[:, :, ::st, ::st] = x
    return out


def conv_fwd(x, w, p, st):
    """(B,c_i,H,W) x (c_o,c_i,s,s) -> (B,c_o,oh,ow), mod 2^64."""
    y = OK.conv2d_wrap(pad(x, p), _u(w))
    return _u(y[:, :, ::st, ::st]) if st > 1 else y


def conv_bwdx(gy, w, H, W, p, st):
    """Adjoint of conv_fwd in x: (B,c_o,oh,ow) -> (B,c_i,H,W)."""
    s = w.shape[2]
    d = pad(dilate(gy, st), s - 1)
    wf = _u(np.transpose(np.asarray(w, dtype=np.uint64)[:, :, ::-1, ::-1], (1, 0, 2, 3)))
    full = OK.conv2d_wrap(d, wf)  # (B, c_i, (oh-1)st + s, ...)
    out = np.zeros((gy.shape[0], w.shape[1], H, W), dtype=np.uint64)
    hh, ww = min(H, full.shape[2] - p), min(W, full.shape[3] - p)
    out[:, :, :hh, :ww] = full[:, :, p:p + hh, p:p + ww]
    return out


def conv_gradw(x, gy, s, p, st):
    """(B,c_i,H,W), (B,c_o,oh,ow) -> (c_o,c_i,s,s) = sum over batch and positions."""
    xt = _u(np.transpose(pad(x, p), (1, 0, 2, 3)))  # (c_i, B, hp, wp)
    kt = _u(np.transpose(dilate(gy, st), (1, 0, 2, 3)))  # (c_o, B, sd, sd)
    full = OK.conv2d_wrap(xt, kt)  # (c_i, c_o, hp - sd + 1, ...)
    return _u(np.transpose(full[:, :, :s, :s], (1, 0, 2, 3)))


def pool_sum(x):
    """2x2 window sums (B,C,H,W) -> (B,C,H/2,W/2) mod 2^64."""
    x = np.asarray(x, dtype=np.uint64)
    return _u(x[:, :, 0::2, 0::2] + x[:, :, 0::2, 1::2] + x[:, :, 1::2, 0::2] + x[:, :, 1::2, 1::2])


def pool_replicate(g):
    """(B,C,h,w) -> (B,C,2h,2w), every value copied to its 2x2 window."""
    return _u(np.repeat(np.repeat(np.asarray(g, dtype=np.uint64), 2, axis=2), 2, axis=3))


__all__ = ["pad", "dilate", "conv_fwd", "conv_bwdx", "conv_gradw", "pool_sum", "pool_replicate", "conv_out_hw"]
