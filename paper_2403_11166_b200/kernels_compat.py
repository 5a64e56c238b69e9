"""Drop-in replacement of the reference kernel tier ``pencil._kernels``.

Same function names, argument order and ownership rules as
/root/reference/pkg/src/pencil/_kernels.py ("K"), over numpy uint64 arrays,
but every computation runs on the B200 through the C ABI: inputs are copied
to the device, the sm_100a kernel runs, results are copied back.  A
reference caller can do ``import paper_2403_11166_b200.kernels_compat as
_kernels``.

Preconditions (the reference's own, K:4-5, 46-49, tightened to this
engine's u32 residues): moduli are NTT-friendly primes q < 2^30, residues
are canonical (< q) for the NTTs and < 2^32 for the pointwise ops.
Violations raise ParamsError instead of returning garbage.
"""

from __future__ import annotations

import ctypes
from functools import lru_cache

import numpy as np
import torch

from . import _dev, _lib
from .errors import ParamsError, ShapeError
from .params import BfvParams, DeviceContext


def set_threads(n: int) -> None:  # K:18-19 — no host threads to size; kept for API parity
    return None


def _bitrev(i: int, logn: int) -> int:
    return int(format(i, f"0{logn}b")[::-1], 2) if logn else 0


@lru_cache(maxsize=64)
def _ctx(N: int, moduli: tuple, psis: tuple, prefix_inv: tuple = (), int_part: tuple = (), frac_part: tuple = ()):
    params = BfvParams(N=N, L=len(moduli), ell=59, moduli=moduli, psi_override=psis)
    c = params.to_c()
    for i, v in enumerate(prefix_inv):
        c.garner_prefix_inv[i] = int(v)
    for i, v in enumerate(int_part):
        c.scale_int[i] = int(v)
    for i, v in enumerate(frac_part):
        c.scale_frac[i] = float(v)
    return DeviceContext(params, c)


def _limb_map(q: np.ndarray):
    q = np.asarray(q, dtype=np.uint64)
    uniq, inv = np.unique(q, return_inverse=True)
    first = [int(np.nonzero(inv == k)[0][0]) for k in range(len(uniq))]
    return [int(u) for u in uniq], inv.astype(np.int32), first


def _tables_ctx(tab: np.ndarray, q: np.ndarray, inverse: bool):
    R, N = tab.shape
    logn = N.bit_length() - 1
    moduli, inv, first = _limb_map(q)
    psis = []
    for qq, r in zip(moduli, first):
        w = int(tab[r, N // 2 if N > 1 else 0])  # psi^{+-bitrev(N/2)} = psi^{+-1}
        psi = pow(w, -1, qq) if inverse else w
        for i in (1, 2, 3, N - 1):
            if i < N:
                e = _bitrev(i, logn)
                want = pow(psi, -e, qq) if inverse else pow(psi, e, qq)
                if int(tab[r, i]) != want:
                    raise ParamsError("twiddle table is not psi^bitrev(i) for a single psi")
        psis.append(psi)
    return _ctx(N, tuple(moduli), tuple(psis)), inv


def _check_rows(rows, q, bound_q: bool):
    rows = np.asarray(rows)
    if rows.dtype != np.uint64 or rows.ndim != 2:
        raise ShapeError("rows must be a 2-D uint64 array")
    lim = np.asarray(q, dtype=np.uint64)[:, None] if bound_q else np.uint64(1 << 32)
    if rows.size and np.any(rows >= lim):
        raise ParamsError("residues out of range for the device engine")


def _run_ntt(rows, tab, q, inverse):
    _check_rows(rows, q, True)
    ctx, limb = _tables_ctx(np.asarray(tab), np.asarray(q), inverse)
    d = _dev.u32_to_device(rows.astype(np.uint32))
    rl = _dev.i32_to_device(limb)
    R = rows.shape[0]
    st = _dev.stream()
    if inverse:  # K's bit-reversed order -> device order -> INTT
        _lib.call("pb_ntt_reorder", ctx.handle, _dev.ptr(d), R, 1, st)
        _lib.call("pb_ntt_inverse", ctx.handle, _dev.ptr(d), R, _dev.ptr(rl), st)
    else:  # NTT -> device order -> K's bit-reversed order
        _lib.call("pb_ntt_forward", ctx.handle, _dev.ptr(d), R, _dev.ptr(rl), st)
        _lib.call("pb_ntt_reorder", ctx.handle, _dev.ptr(d), R, 0, st)
    rows[...] = _dev.to_numpy_u32(d).astype(np.uint64)


def ntt_forward(rows, psi_brv, q):  # K:31-50
    _run_ntt(rows, psi_brv, q, False)


def ntt_inverse(rows, ipsi_brv, n_inv, q):  # K:53-77
    q = np.asarray(q, dtype=np.uint64)
    N = rows.shape[1]
    for r in range(len(q)):
        if int(n_inv[r]) != pow(N, -1, int(q[r])):
            raise ParamsError("n_inv must be N^-1 mod q")
    _run_ntt(rows, ipsi_brv, q, True)


def _pw(op, out, a, b, q):
    for x in (out, a, b):
        _check_rows(x, q, False)
    R, N = out.shape
    moduli, limb, _ = _limb_map(q)
    ctx = _ctx(N, tuple(moduli), tuple(BfvParams(N=N, L=len(moduli), moduli=tuple(moduli)).psi))
    do = _dev.u32_to_device(out.astype(np.uint32))
    da = _dev.u32_to_device(a.astype(np.uint32))
    db = _dev.u32_to_device(b.astype(np.uint32))
    rl = _dev.i32_to_device(limb)
    _lib.call("pb_pw", ctx.handle, op, _dev.ptr(do), _dev.ptr(da), _dev.ptr(db), R, R, _dev.ptr(rl), _dev.stream())
    out[...] = _dev.to_numpy_u32(do).astype(np.uint64)


def pw_mul(out, a, b, q):  # K:80-86
    _pw(_lib.PW_MUL, out, a, b, q)


def pw_mul_acc(out, a, b, q):  # K:89-95
    _pw(_lib.PW_MAC, out, a, b, q)


def pw_add(out, a, b, q):  # K:98-104
    _pw(_lib.PW_ADD, out, a, b, q)


def pw_sub(out, a, b, q):  # K:107-113
    _pw(_lib.PW_SUB, out, a, b, q)


def negacyclic_mul_wrap(a, b):  # K:135-147
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    N = a.shape[0]
    da, db = _dev.u64_to_device(a), _dev.u64_to_device(b)
    out = _dev.empty_u64(N)
    _lib.call("pb_negacyclic_mul_wrap", _dev.ptr(da), _dev.ptr(db), 1, N, _dev.ptr(out), _dev.stream())
    return _dev.to_numpy_u64(out).copy()


def negacyclic_mul_mod(a, b, q):  # K:116-132, via forward NTT / pointwise / inverse on device
    a = np.asarray(a, dtype=np.uint64) % np.uint64(q)
    b = np.asarray(b, dtype=np.uint64) % np.uint64(q)
    N = a.shape[0]
    params = BfvParams(N=N, L=1, moduli=(int(q),))
    ctx = _ctx(N, (int(q),), params.psi)
    d = _dev.u32_to_device(np.stack([a, b]).astype(np.uint32))
    _lib.call("pb_ntt_forward", ctx.handle, _dev.ptr(d), 2, None, _dev.stream())
    _lib.call("pb_pw", ctx.handle, _lib.PW_MUL, _dev.ptr(d[0]), _dev.ptr(d[0]), _dev.ptr(d[1]), 1, 1, None, _dev.stream())
    _lib.call("pb_ntt_inverse", ctx.handle, _dev.ptr(d[0]), 1, None, _dev.stream())
    return _dev.to_numpy_u32(d[0]).astype(np.uint64)


def _decode_ctx(q, prefix_inv=(), int_part=(), frac_part=(), L=None, N=None):
    moduli = tuple(int(x) for x in q)
    return _ctx(N, moduli, BfvParams(N=N, L=len(moduli), moduli=moduli).psi, tuple(int(x) for x in prefix_inv),
                tuple(int(x) for x in int_part), tuple(float(x) for x in frac_part))


def garner_digits(rows, q, prefix_inv):  # K:158-179
    rows = np.asarray(rows, dtype=np.uint64)
    L, N = rows.shape
    _check_rows(rows, q, False)
    ctx = _decode_ctx(q, prefix_inv, N=N)
    d = _dev.u32_to_device(rows.astype(np.uint32))
    out = _dev.empty_u32(L, N)
    _lib.call("pb_garner_digits", ctx.handle, _dev.ptr(d), 1, _dev.ptr(out), _dev.stream())
    return _dev.to_numpy_u32(out).astype(np.uint64)


def scale_round_digits(digits, int_part, frac_part, t_mask, q=None):  # K:182-199
    digits = np.asarray(digits, dtype=np.uint64)
    L, N = digits.shape
    ell = int(t_mask).bit_length()
    if int(t_mask) != (1 << ell) - 1:
        raise ParamsError("t_mask must be 2^ell - 1")
    mods = q if q is not None else BfvParams(N=max(N, 4), L=L).moduli
    ctx = _decode_ctx(mods, (), int_part, frac_part, N=N)
    if ctx.params.ell != ell:
        c = ctx._c
        c.ell = ell
        ctx = DeviceContext(BfvParams(N=N, L=L, ell=ell, moduli=ctx.params.moduli), c)
    d = _dev.u32_to_device(digits.astype(np.uint32))
    out = _dev.empty_u64(N)
    _lib.call("pb_scale_round_digits", ctx.handle, _dev.ptr(d), 1, _dev.ptr(out), _dev.stream())
    return _dev.to_numpy_u64(out).copy()


def matmul_wrap(a, b):  # K:206-218
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    n, k = a.shape
    m = b.shape[1]
    out = _dev.empty_u64(n, m)
    da, db = _dev.u64_to_device(a), _dev.u64_to_device(b)  # keep alive until the kernel is enqueued
    _lib.call("pb_ring_matmul", _dev.ptr(da), _dev.ptr(db), n, k, m, 0, 0, 64, _dev.ptr(out), _dev.stream())
    return _dev.to_numpy_u64(out).copy()


def im2col_wrap(x, s, stride):  # K:221-238
    x = np.ascontiguousarray(x, dtype=np.uint64)
    B, C, H, W = x.shape
    oh, ow = (H - s) // stride + 1, (W - s) // stride + 1
    out = _dev.empty_u64(C * s * s, B * oh * ow)
    dx = _dev.u64_to_device(x)
    _lib.call("pb_im2col", _dev.ptr(dx), B, C, H, W, s, stride, _dev.ptr(out), _dev.stream())
    return _dev.to_numpy_u64(out).copy()


def col2im_wrap(cols, B, C, H, W, s, stride):  # K:241-257
    cols = np.ascontiguousarray(cols, dtype=np.uint64)
    out = _dev.empty_u64(B, C, H, W)
    dc = _dev.u64_to_device(cols)
    _lib.call("pb_col2im", _dev.ptr(dc), B, C, H, W, s, stride, _dev.ptr(out), _dev.stream())
    return _dev.to_numpy_u64(out).copy()


def conv2d_wrap(x, w):  # K:260-278
    x = np.ascontiguousarray(x, dtype=np.uint64)
    w = np.ascontiguousarray(w, dtype=np.uint64)
    B, Ci, H, W = x.shape
    Co, _, s, _ = w.shape
    out = _dev.empty_u64(B, Co, H - s + 1, W - s + 1)
    dx, dw = _dev.u64_to_device(x), _dev.u64_to_device(w)
    _lib.call("pb_conv2d", _dev.ptr(dx), _dev.ptr(dw), B, Ci, H, W, Co, s, 64, _dev.ptr(out), _dev.stream())
    return _dev.to_numpy_u64(out).copy()
