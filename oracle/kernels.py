"""ORACLE — TEST INFRASTRUCTURE ONLY.

numpy-facing wrappers over ``liboracle_kernels.so`` (oracle/kernels.c) with the
exact names, argument order and ownership rules of the reference kernel tier
``pencil._kernels`` (/root/reference/pkg/src/pencil/_kernels.py, "K"):

* in place:           ntt_forward (K:31), ntt_inverse (K:53)
* caller-owned out:   pw_mul (K:80), pw_mul_acc (K:89), pw_add (K:98), pw_sub (K:107)
* return new arrays:  negacyclic_mul_mod (K:116), negacyclic_mul_wrap (K:135),
                      garner_digits (K:158), scale_round_digits (K:182),
                      matmul_wrap (K:206), im2col_wrap (K:221),
                      col2im_wrap (K:241), conv2d_wrap (K:260)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  The product package never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_kernels.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/kernels.c with oracle/Makefile (gcc + OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
        os.path.join(_HERE, "kernels.c")
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        U = ctypes.c_uint64
        sig = {
            "orc_set_threads": [ctypes.c_int],
            "orc_ntt_forward": [P, P, P, I, I],
            "orc_ntt_inverse": [P, P, P, P, I, I],
            "orc_pw_mul": [P, P, P, P, I, I],
            "orc_pw_mul_acc": [P, P, P, P, I, I],
            "orc_pw_add": [P, P, P, P, I, I],
            "orc_pw_sub": [P, P, P, P, I, I],
            "orc_negacyclic_mul_mod": [P, P, U, I, P],
            "orc_negacyclic_mul_wrap": [P, P, I, P],
            "orc_garner_digits": [P, P, P, I, I, P],
            "orc_scale_round_digits": [P, P, P, U, I, I, P],
            "orc_matmul_wrap": [P, P, I, I, I, P],
            "orc_im2col_wrap": [P, I, I, I, I, I, I, P],
            "orc_col2im_wrap": [P, I, I, I, I, I, I, P],
            "orc_conv2d_wrap": [P, P, I, I, I, I, I, I, P],
        }
        for name, args in sig.items():
            fn = getattr(_lib, name)
            fn.argtypes = args
            fn.restype = None
        _lib.orc_get_threads.restype = ctypes.c_int
    return _lib


def _u64(a):
    a = np.asarray(a)
    if a.dtype != np.uint64 or not a.flags.c_contiguous:
        raise TypeError("oracle kernels take C-contiguous uint64 arrays")
    return a


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int) -> None:  # K:18-19
    _load().orc_set_threads(max(1, int(n)))


def get_threads() -> int:
    return int(_load().orc_get_threads())


def ntt_forward(rows, psi_brv, q):  # K:31-50
    rows, psi_brv, q = _u64(rows), _u64(psi_brv), _u64(q)
    R, N = rows.shape
    _load().orc_ntt_forward(_p(rows), _p(psi_brv), _p(q), R, N)


def ntt_inverse(rows, ipsi_brv, n_inv, q):  # K:53-77
    rows, ipsi_brv, n_inv, q = _u64(rows), _u64(ipsi_brv), _u64(n_inv), _u64(q)
    R, N = rows.shape
    _load().orc_ntt_inverse(_p(rows), _p(ipsi_brv), _p(n_inv), _p(q), R, N)


def _pw(name, out, a, b, q):
    out, a, b, q = _u64(out), _u64(a), _u64(b), _u64(q)
    R, N = out.shape
    getattr(_load(), name)(_p(out), _p(a), _p(b), _p(q), R, N)


def pw_mul(out, a, b, q):  # K:80-86
    _pw("orc_pw_mul", out, a, b, q)


def pw_mul_acc(out, a, b, q):  # K:89-95
    _pw("orc_pw_mul_acc", out, a, b, q)


def pw_add(out, a, b, q):  # K:98-104
    _pw("orc_pw_add", out, a, b, q)


def pw_sub(out, a, b, q):  # K:107-113
    _pw("orc_pw_sub", out, a, b, q)


def negacyclic_mul_mod(a, b, q):  # K:116-132
    a, b = _u64(a), _u64(b)
    out = np.empty(a.shape[0], dtype=np.uint64)
    _load().orc_negacyclic_mul_mod(_p(a), _p(b), int(q), a.shape[0], _p(out))
    return out


def negacyclic_mul_wrap(a, b):  # K:135-147
    a, b = _u64(a), _u64(b)
    out = np.empty(a.shape[0], dtype=np.uint64)
    _load().orc_negacyclic_mul_wrap(_p(a), _p(b), a.shape[0], _p(out))
    return out


def garner_digits(rows, q, prefix_inv):  # K:158-179
    rows, q, prefix_inv = _u64(rows), _u64(q), _u64(prefix_inv)
    L, N = rows.shape
    digits = np.empty((L, N), dtype=np.uint64)
    _load().orc_garner_digits(_p(rows), _p(q), _p(prefix_inv), L, N, _p(digits))
    return digits


def scale_round_digits(digits, int_part, frac_part, t_mask):  # K:182-199
    digits, int_part = _u64(digits), _u64(int_part)
    frac_part = np.ascontiguousarray(frac_part, dtype=np.float64)
    L, N = digits.shape
    out = np.empty(N, dtype=np.uint64)
    _load().orc_scale_round_digits(
        _p(digits), _p(int_part), _p(frac_part), int(t_mask), L, N, _p(out)
    )
    return out


def matmul_wrap(a, b):  # K:206-218
    a, b = _u64(a), _u64(b)
    n, k = a.shape
    m = b.shape[1]
    out = np.empty((n, m), dtype=np.uint64)
    _load().orc_matmul_wrap(_p(a), _p(b), n, k, m, _p(out))
    return out


def im2col_wrap(x, s, stride):  # K:221-238
    x = _u64(x)
    B, C, H, W = x.shape
    oh = (H - s) // stride + 1
    ow = (W - s) // stride + 1
    out = np.empty((C * s * s, B * oh * ow), dtype=np.uint64)
    _load().orc_im2col_wrap(_p(x), B, C, H, W, s, stride, _p(out))
    return out


def col2im_wrap(cols, B, C, H, W, s, stride):  # K:241-257
    cols = _u64(cols)
    out = np.empty((B, C, H, W), dtype=np.uint64)
    _load().orc_col2im_wrap(_p(cols), B, C, H, W, s, stride, _p(out))
    return out


def conv2d_wrap(x, w):  # K:260-278
    x, w = _u64(x), _u64(w)
    B, Ci, H, W = x.shape
    Co, _, s, _ = w.shape
    out = np.empty((B, Co, H - s + 1, W - s + 1), dtype=np.uint64)
    _load().orc_conv2d_wrap(_p(x), _p(w), B, Ci, H, W, Co, s, _p(out))
    return out


# --- cyclic-limb batch helpers (same arithmetic as K; see kernels.c) -------

def _load_cyc():
    lib = _load()
    if not getattr(lib, "_cyc_ready", False):
        P, I, U = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64
        lib.orc_ntt_forward_cyc.argtypes = [P, P, P, I, I, I]
        lib.orc_ntt_inverse_cyc.argtypes = [P, P, P, P, I, I, I]
        lib.orc_pw_cyc.argtypes = [ctypes.c_int, P, P, P, P, I, I, I, I]
        lib.orc_decode_batch.argtypes = [P, P, P, P, P, U, I, I, I, P]
        for n in ("orc_ntt_forward_cyc", "orc_ntt_inverse_cyc", "orc_pw_cyc", "orc_decode_batch"):
            getattr(lib, n).restype = None
        lib._cyc_ready = True
    return lib


def ntt_forward_cyc(rows, psi_brv, q):
    """rows (R, N) with row r on limb r % L; psi_brv (L, N); q (L,)."""
    rows, psi_brv, q = _u64(rows), _u64(psi_brv), _u64(q)
    R, N = rows.shape
    _load_cyc().orc_ntt_forward_cyc(_p(rows), _p(psi_brv), _p(q), R, N, q.shape[0])


def ntt_inverse_cyc(rows, ipsi_brv, n_inv, q):
    rows, ipsi_brv, n_inv, q = _u64(rows), _u64(ipsi_brv), _u64(n_inv), _u64(q)
    R, N = rows.shape
    _load_cyc().orc_ntt_inverse_cyc(_p(rows), _p(ipsi_brv), _p(n_inv), _p(q), R, N, q.shape[0])


_OPS = {"mul": 0, "mul_acc": 1, "add": 2, "sub": 3}


def pw_cyc(op, out, a, b, q):
    """out/a (R, N); b (Rb, N) broadcast cyclically (row r uses b[r % Rb]); q (L,)."""
    out, a, b, q = _u64(out), _u64(a), _u64(b), _u64(q)
    R, N = out.shape
    _load_cyc().orc_pw_cyc(_OPS[op], _p(out), _p(a), _p(b), _p(q), R, N, q.shape[0], b.shape[0])


def decode_batch(rows, q, prefix_inv, int_part, frac_part, t_mask):
    """rows (P, L, N) -> (P, N): garner_digits + scale_round_digits per poly."""
    rows, q, prefix_inv, int_part = _u64(rows), _u64(q), _u64(prefix_inv), _u64(int_part)
    frac_part = np.ascontiguousarray(frac_part, dtype=np.float64)
    P, L, N = rows.shape
    out = np.empty((P, N), dtype=np.uint64)
    _load_cyc().orc_decode_batch(
        _p(rows), _p(q), _p(prefix_inv), _p(int_part), _p(frac_part), int(t_mask), P, L, N, _p(out)
    )
    return out
