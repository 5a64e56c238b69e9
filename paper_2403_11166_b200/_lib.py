"""ctypes binding of the C ABI in include/pencil_b200.h.

The shared library is built in-tree (``_build.py``) and loaded from the
package directory.  There is no CPU fallback: if the library or a CUDA
device is missing, every entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import STATUS_TO_ERROR, DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpencil_b200.so")

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U64 = ctypes.c_uint64
INT = ctypes.c_int
F64 = ctypes.c_double

MAX_LIMBS = 8


class PbParams(ctypes.Structure):
    _fields_ = [
        ("N", I32),
        ("L", I32),
        ("ell", I32),
        ("reserved", I32),
        ("q", ctypes.c_uint32 * MAX_LIMBS),
        ("psi", ctypes.c_uint32 * MAX_LIMBS),
        ("delta_mod_q", ctypes.c_uint32 * MAX_LIMBS),
        ("garner_prefix_inv", ctypes.c_uint32 * MAX_LIMBS),
        ("scale_int", ctypes.c_uint64 * MAX_LIMBS),
        ("scale_frac", ctypes.c_double * MAX_LIMBS),
    ]


# name -> argtypes (every function returns int status unless listed in _RET)
SIGNATURES = {
    "pb_abi_version": [],
    "pb_last_error": [],
    "pb_device_sm_count": [P],
    "pb_ctx_create": [P, P],
    "pb_ctx_destroy": [P],
    "pb_ntt_forward": [P, P, I64, P, P],
    "pb_ntt_inverse": [P, P, I64, P, P],
    "pb_ntt_reorder": [P, P, I64, INT, P],
    "pb_pw": [P, INT, P, P, P, I64, I64, P, P],
    "pb_garner_digits": [P, P, I64, P, P],
    "pb_scale_round_digits": [P, P, I64, P, P],
    "pb_decode": [P, P, I64, P, P],
    "pb_negacyclic_mul_wrap": [P, P, I64, I32, P, P],
    "pb_encode_plain": [P, P, P, P, I32, I64, P, P, P],
    "pb_lift": [P, P, I64, INT, P, P],
    "pb_unpack": [P, P, P, I32, I32, I64, P, P],
    "pb_encrypt_pk": [P, P, P, P, P, I32, I64, U64, P, U64, P, P],
    "pb_encrypt_pk_noise": [P, P, P, P, P, I32, I64, P, P, P, P, P],
    "pb_encrypt_sk": [P, P, P, P, P, P, I32, I64, U64, P, U64, P, P],
    "pb_shoup_rows": [P, P, P, I64, P],
    "pb_encrypt_sk_zero": [P, P, I64, U64, P, U64, P, P, P],
    "pb_encrypt_sk_add": [P, P, P, P, I32, I64, P, P, P],
    "pb_encrypt_sk_noise": [P, P, P, P, P, I32, I64, P, P, P, P],
    "pb_decrypt_coeffs": [P, P, P, I64, P, P],
    "pb_decrypt": [P, P, P, I64, P, P, P],
    "pb_decrypt_to_share": [P, P, P, I64, P, P, I32, P, P, P],
    "pb_ctpt_mac_mask": [P, P, P, P, P, I32, I64, P, P, I32, P, INT, U64, P, P, P],
    "pb_encode_plain_mont": [P, P, P, P, I32, I64, P, P],
    "pb_mask_ntt": [P, I64, P, P, I32, P, INT, U64, P, P, P],
    "pb_ctpt_mac_tiled": [P, P, P, P, P, I32, I32, I32, P, P],
    "pb_ring_binary": [INT, P, P, P, I64, I64, I32, P],
    "pb_ring_unary": [INT, P, P, U64, I64, I32, P],
    "pb_encode_fixed": [P, I64, I32, I32, P, P, P],
    "pb_decode_fixed": [P, I64, I32, I32, P, P],
    "pb_uniform_ring": [P, I64, U64, P, U64, U64, I32, P],
    "pb_share": [P, I64, U64, P, U64, U64, I32, P, P, P],
    "pb_ring_matmul": [P, P, I64, I64, I64, INT, INT, I32, P, P],
    "pb_ring_matmul_ex": [P, P, I64, I64, I64, INT, INT, I32, P, I32, P],
    "pb_scatter_u64": [P, P, P, I64, P],
    "pb_mask_mac": [P, P, P, P, P, I32, I32, I32, P, P, I32, P, INT, U64, P, P, P],
    "pb_nl_words": [INT],
    "pb_prep_scalars": [P, P, I32, U64, P, U64, U64, I32, P],
    "pb_nl_op": [INT, P, P, I64, I32, I32, P, P, U64, P, U64, U64, P, P, P],
    "pb_ring_matmul_add": [P, P, I64, I64, I64, INT, INT, P, I32, I32, P, P],
    "pb_host_softmax_pre": [P, I32, I32, I32, I32, P],
    "pb_host_softmax_post": [P, I32, I32, P, I32, I32, I32, P, P],
    "pb_host_mean": [P, I64],
    "pb_set_launch_cap": [I32],
    "pb_copy_async": [P, P, I64, P],
    "pb_host_handoff": [P, P, P, P, I64, I64, P, P],
    "pb_host_publish": [P, P, I64, P, P, P],
    "pb_step_prologue": [P, P, P, P, I64, P],
    "pb_wire_frame_bytes": [P, I32, P],
    "pb_mod_switch_drop": [P, P, P, I64, P, P, P],
    "pb_wire_serialize": [P, P, I64, I32, I32, P, P],
    "pb_wire_deserialize": [P, P, I64, I32, I32, P, P, P],
    "pb_ring_rowsum": [P, I64, I64, I32, P, P],
    "pb_ring_chansum": [P, I32, I32, I64, I32, P, P],
    "pb_im2col": [P, I32, I32, I32, I32, I32, I32, P, P],
    "pb_col2im": [P, I32, I32, I32, I32, I32, I32, P, P],
    "pb_conv2d": [P, P, I32, I32, I32, I32, I32, I32, I32, P, P],
    "pb_ring_conv": [INT, P, P, I32, I32, I32, I32, I32, I32, I32, I32, I32, P, P],
    "pb_ring_conv_ex": [INT, P, P, I32, I32, I32, I32, I32, I32, I32, I32, I32, P, I32, P],
    "pb_pool2": [INT, P, I64, I32, I32, I32, P, P],
    "pb_ring_lincomb": [INT, P, P, P, I32, P, I32, P, I64, I32, P],
    "pb_ring_add_bcast": [P, P, P, I64, I64, I64, I32, P],
    "pb_dealer_op": [INT, P, P, I64, I32, P, P, U64, P, U64, U64, I32, P],
    "pb_dealer_op_out": [INT, P, P, P, P, I64, I32, P, P, U64, P, U64, U64, I32, P],
    "pb_sgd_momentum": [P, P, P, I64, I32, F64, F64, I32, I32, P, P, P, P],
}
_RET = {"pb_last_error": ctypes.c_char_p, "pb_host_mean": ctypes.c_double}

# ring / pointwise / dealer op codes (mirror the enums in pencil_b200.h)
PW_MUL, PW_MAC, PW_ADD, PW_SUB = 0, 1, 2, 3
RING_ADD, RING_SUB, RING_MUL, RING_NEG, RING_SCALAR_MUL, RING_MASK, RING_ARITH_SHIFT = range(7)
DEALER_RELU, DEALER_TRUNC, DEALER_SELECT, DEALER_RESHARE, DEALER_RELU_TRUNC, DEALER_TRUNC_SELECT = range(6)
CONV_FWD, CONV_BWDX, CONV_GRADW = range(3)
BACKEND_AUTO, BACKEND_CUDA_CORE, BACKEND_TENSOR = range(3)
NL_DRELU, NL_MUX, NL_TRUNC, NL_RELU_TRUNC, NL_TRUNC_MUX = range(5)
POOL_SUM, POOL_REPLICATE = range(2)

_lib = None


ABI_VERSION = 2  # include/pencil_b200.h PB_ABI_VERSION


def load(build_if_missing: bool = True):
    """Load (building first if needed) the in-tree CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing:
        from . import _build

        _build.build()
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"CUDA engine library missing: {LIB_PATH} (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH)
    lib.pb_abi_version.restype = ctypes.c_int
    got = lib.pb_abi_version()
    if got != ABI_VERSION:  # a stale library would mis-bind the changed signatures
        raise DeviceError(f"{LIB_PATH}: C ABI version {got}, this package binds {ABI_VERSION} "
                          "(rebuild: __graft_entry__.build())")
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RET.get(name, ctypes.c_int)
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().pb_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    if status != 0:
        cls = STATUS_TO_ERROR.get(int(status), DeviceError)
        raise cls(f"{what}: {last_error()}" if what else last_error())


# Device kernels each entry point launches (for the bench's gpu_launches count).
KERNELS_PER_CALL = {
    "pb_encrypt_pk": 2, "pb_encrypt_sk": 2, "pb_decrypt": 2, "pb_decrypt_to_share": 1, "pb_unpack": 1,
    "pb_abi_version": 0, "pb_last_error": 0, "pb_set_launch_cap": 0, "pb_copy_async": 0, "pb_host_softmax_pre": 0,
    "pb_host_softmax_post": 0, "pb_host_mean": 0, "pb_device_sm_count": 0, "pb_ctx_create": 0, "pb_ctx_destroy": 0,
}


class CallStats:
    """Optional instrumentation: counts kernel launches and, for selected entry
    points, brackets each call with CUDA events on the current stream."""

    def __init__(self, timed=()):
        self.launches = 0
        self.calls = {}
        self.timed = set(timed)
        self.events = []  # (name, start_event, end_event, tag)
        self.tag = None

    def before(self, name, args=()):
        k = KERNELS_PER_CALL.get(name, 1)
        if name == "pb_decrypt_to_share" and len(args) > 6 and int(args[6]) >= 384:
            k = 2  # INTT + separate decode kernel for slot-heavy ciphertexts (pb_bfv.cu)
        self.launches += k
        self.calls[name] = self.calls.get(name, 0) + 1
        if name in self.timed:
            import torch

            s = torch.cuda.Event(enable_timing=True)
            s.record()
            return s
        return None

    def after(self, name, s):
        if s is not None:
            import torch

            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.events.append((name, s, e, self.tag))


STATS: CallStats | None = None


def call(name: str, *args) -> None:
    """Invoke a C ABI entry point and raise the mapped exception on failure."""
    st = STATS
    if st is None:
        check(getattr(load(), name)(*args), name)
        return
    ev = st.before(name, args)
    check(getattr(load(), name)(*args), name)
    st.after(name, ev)
