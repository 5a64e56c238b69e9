"""Z_{2^ell} tensors, fixed point and additive shares on the device.

Mirrors the reference ring layer ``pencil.ring`` (/root/reference/pkg/src/
pencil/ring.py, "R") name for name -- RingParams (R:24-45), SeededRng
(R:48-90), RingTensor (R:93-148), ShareTensor (R:151-171), encode_fixed /
decode_fixed / to_signed / encode_tensor (R:174-203), arith_shift
(R:206-211), share_tensor / reconstruct_tensor / zeros_like / zero_share
(R:214-233) -- with the same semantics and error behaviour, but the values
live in HBM (torch.int64 CUDA tensors holding the uint64 bit pattern) and
every arithmetic step is a vectorised sm_100a kernel (csrc/pb_ring.cu).

``SeededRng.uniform_ring`` is generated ON THE DEVICE and is bit-identical
to numpy's ``Generator(Philox(key=[seed, stream])).integers(0, 2**ell)``
(raw >> (64-ell)), so masks and shares match the CPU
oracle exactly.  Draws that numpy implements with rejection or float
transforms (ternary, uniform_mod, cbd, normal) stay on the host generator,
kept in lock-step with the device draws through the Philox counter.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .errors import EncodeRangeError, ScaleError, ShapeError

MO = "mo"
DO = "do"


@dataclass(frozen=True)
class RingParams:  # R:24-45
    """Plaintext ring Z_{2**ell} with f fraction bits of fixed-point scale."""

    ell: int = 59
    f: int = 25

    def __post_init__(self):
        if not (1 <= self.f and 2 * self.f < self.ell <= 62):
            raise ValueError(f"need 1 <= f, 2f < ell <= 62, got ell={self.ell} f={self.f}")

    @property
    def t(self) -> int:
        return 1 << self.ell

    @property
    def mask(self) -> np.uint64:
        return np.uint64((1 << self.ell) - 1)

    @property
    def headroom(self) -> int:
        return self.ell - 2 * self.f


class SeededRng:  # R:48-90
    """Counter-based Philox randomness; (seed, stream) fully determine the output."""

    def __init__(self, seed: int, stream: int = 0):
        self.seed_arg, self.stream_arg = seed, stream
        # the Philox key exactly as numpy derives it from [seed, stream]
        key = np.random.Philox(key=[seed, stream]).state["state"]["key"]
        self.seed = int(key[0])
        self.stream = int(key[1])
        self._pos = 0  # raw 64-bit outputs consumed so far
        self._gen = None  # host numpy Generator, synchronised lazily
        self._host_pos = 0  # position the host generator state corresponds to

    def child(self, stream: int) -> "SeededRng":
        return SeededRng(self.seed_arg, stream)

    seed_ptr = None  # device address of the step seed (CUDA-graph mode), see bind()

    def bind(self, seed_ptr: int) -> "SeededRng":
        """Read key word 0 from device memory at kernel run time (graph replay);
        the device value must equal this generator's seed whenever it runs."""
        self.seed_ptr = seed_ptr
        return self

    @property
    def _stream_const(self) -> int:
        return (self.stream * 0xD1B54A32D192ED03 + 0x632BE59BD9B4E019) & ((1 << 64) - 1)

    @property
    def device_key(self) -> int:
        """64-bit key for the device-only Philox4x32 streams (encryption noise,
        mask filler): fmix64(seed * G + C(stream)), distinct per stream
        (the same mixing as dev_key() in pb_common.cuh)."""
        M = (1 << 64) - 1
        z = (self.seed * 0x9E3779B97F4A7C15 + self._stream_const) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    def np_args(self):
        """(seed, seed_dev) for numpy-identical device streams."""
        return (0, self.seed_ptr) if self.seed_ptr else (self.seed, None)

    def dev_args(self):
        """(seed, seed_dev) for device-only streams."""
        return (self._stream_const, self.seed_ptr) if self.seed_ptr else (self.device_key, None)

    # -- position bookkeeping -------------------------------------------------
    def reserve(self, n: int) -> int:
        """Claim n raw outputs for a device kernel; returns their start offset."""
        off = self._pos
        self._pos += int(n)
        return off

    def _host(self) -> np.random.Generator:
        if self._gen is None:
            self._gen = np.random.Generator(np.random.Philox(key=[self.seed_arg, self.stream_arg]))
            self._host_pos = 0
        if self._host_pos != self._pos:
            bg = self._gen.bit_generator
            st = bg.state
            r = self._pos
            c = (r + 3) // 4
            tmp = np.random.Philox(key=[self.seed_arg, self.stream_arg], counter=[max(c - 1, 0), 0, 0, 0])
            if r % 4:
                tmp.random_raw(r % 4)
                ts = tmp.state
                st["state"]["counter"] = ts["state"]["counter"]
                st["buffer"] = ts["buffer"]
                st["buffer_pos"] = ts["buffer_pos"]
            else:
                st["state"]["counter"] = np.array([c, 0, 0, 0], dtype=np.uint64)
                st["buffer_pos"] = 4
            bg.state = st
            self._host_pos = r
        return self._gen

    def _after_host(self):
        st = self._gen.bit_generator.state
        c = int(st["state"]["counter"][0])
        self._pos = 4 * (c - 1) + int(st["buffer_pos"]) if c > 0 else 0
        self._host_pos = self._pos

    # -- draws ----------------------------------------------------------------
    def uniform_ring(self, shape, params: RingParams, out: torch.Tensor | None = None) -> torch.Tensor:  # R:60-61
        shape = tuple(shape) if isinstance(shape, (tuple, list)) else (int(shape),)
        n = int(np.prod(shape)) if shape else 1
        out = _dev.empty_u64(n) if out is None else out.view(-1)
        off = self.reserve(n)
        sd, sp = self.np_args()
        _lib.call("pb_uniform_ring", _dev.ptr(out), n, sd, sp, self.stream, off, params.ell, _dev.stream())
        return out.view(shape)

    def _host_draw(self, fn):
        g = self._host()
        out = fn(g)
        self._after_host()
        return out

    def uniform_mod(self, shape, mod: int) -> np.ndarray:  # R:63-64 (host)
        return self._host_draw(lambda g: g.integers(0, mod, size=shape, dtype=np.uint64))

    def ternary(self, shape) -> np.ndarray:  # R:70-72 (host)
        return self._host_draw(lambda g: g.integers(-1, 2, size=shape, dtype=np.int64))

    def cbd(self, shape, eta: int = 20) -> np.ndarray:  # R:74-78 (host)
        def f(g):
            a = g.binomial(eta, 0.5, size=shape).astype(np.int64)
            b = g.binomial(eta, 0.5, size=shape).astype(np.int64)
            return a - b

        return self._host_draw(f)

    def normal(self, shape, std: float) -> np.ndarray:  # R:80-81 (host)
        return self._host_draw(lambda g: g.normal(0.0, std, size=shape))

    def uniform_real(self, shape, lo: float, hi: float) -> np.ndarray:  # weight init
        return self._host_draw(lambda g: g.uniform(lo, hi, size=shape))


def _as_device_u64(values) -> torch.Tensor:
    if isinstance(values, torch.Tensor):
        t = values
        if t.dtype != torch.int64:
            raise ShapeError("ring tensors are stored as int64 bit patterns")
        return t if t.is_cuda else t.to(_dev.device())
    return _dev.u64_to_device(np.asarray(values, dtype=np.uint64))


class RingTensor:  # R:93-148
    """A shaped device array of Z_t residues carrying a fixed-point scale."""

    __slots__ = ("values", "scale", "params")

    def __init__(self, values, scale: int, params: RingParams, _canonical: bool = False):
        t = _as_device_u64(values).contiguous()
        if not _canonical:
            out = torch.empty_like(t)
            if t.numel():
                _lib.call("pb_ring_unary", _lib.RING_MASK, _dev.ptr(out), _dev.ptr(t), 0, t.numel(), params.ell,
                          _dev.stream())
            t = out
        self.values = t
        self.scale = int(scale)
        self.params = params

    @property
    def shape(self):
        return tuple(self.values.shape)

    @property
    def data(self) -> torch.Tensor:
        return self.values.reshape(-1)

    def numpy(self) -> np.ndarray:
        return _dev.to_numpy_u64(self.values).copy()

    def copy(self) -> "RingTensor":
        return RingTensor(self.values.clone(), self.scale, self.params, _canonical=True)

    def reshape(self, *shape) -> "RingTensor":
        return RingTensor(self.values.reshape(*shape), self.scale, self.params, _canonical=True)

    def transpose(self) -> "RingTensor":
        return RingTensor(self.values.t().contiguous(), self.scale, self.params, _canonical=True)

    def decode(self) -> torch.Tensor:
        return decode_fixed(self.values, self.params, self.scale)

    def with_scale(self, scale: int) -> "RingTensor":
        return RingTensor(self.values, scale, self.params, _canonical=True)

    def _check(self, other: "RingTensor"):
        if self.params != other.params:
            raise ScaleError("ring parameter mismatch")
        if self.scale != other.scale:
            raise ScaleError(f"scale mismatch: {self.scale} vs {other.scale}")
        if self.shape != other.shape:
            raise ShapeError(f"shape mismatch: {self.shape} vs {other.shape}")

    def _binary(self, op: int, other: "RingTensor") -> "RingTensor":
        self._check(other)
        out = torch.empty_like(self.values)
        n = out.numel()
        if n:
            a, b = self.values, other.values.contiguous()
            _lib.call("pb_ring_binary", op, _dev.ptr(out), _dev.ptr(a), _dev.ptr(b), n, n, self.params.ell,
                      _dev.stream())
        return RingTensor(out, self.scale, self.params, _canonical=True)

    def __add__(self, other):
        return self._binary(_lib.RING_ADD, other)

    def __sub__(self, other):
        return self._binary(_lib.RING_SUB, other)

    def _unary(self, op: int, k: int = 0, scale=None) -> "RingTensor":
        out = torch.empty_like(self.values)
        if out.numel():
            _lib.call("pb_ring_unary", op, _dev.ptr(out), _dev.ptr(self.values), int(k) & ((1 << 64) - 1),
                      out.numel(), self.params.ell, _dev.stream())
        return RingTensor(out, self.scale if scale is None else scale, self.params, _canonical=True)

    def __neg__(self):
        return self._unary(_lib.RING_NEG)

    def scalar_mul(self, k: int) -> "RingTensor":
        """Multiply by a plain ring scalar; the scale is unchanged (R:143-145)."""
        return self._unary(_lib.RING_SCALAR_MUL, k & int(self.params.mask))

    def __repr__(self):
        return f"RingTensor(shape={self.shape}, scale={self.scale}, ell={self.params.ell})"


class ShareTensor:  # R:151-171
    """One party's additive share of a logically shared RingTensor."""

    __slots__ = ("owner_role", "value")

    def __init__(self, owner_role: str, value: RingTensor):
        if owner_role not in (MO, DO):
            raise ValueError(f"unknown role {owner_role!r}")
        self.owner_role = owner_role
        self.value = value

    @property
    def scale(self) -> int:
        return self.value.scale

    @property
    def shape(self):
        return self.value.shape

    def __repr__(self):
        return f"ShareTensor({self.owner_role}, shape={self.shape}, scale={self.scale})"


def _check_flag(flag: torch.Tensor, msg: str):
    if int(flag.item()):
        raise EncodeRangeError(msg)


def encode_fixed(x, params: RingParams, scale: int | None = None) -> torch.Tensor:  # R:174-182
    """floor(x * 2**scale) embedded two's-complement into Z_{2**ell} (device)."""
    scale = params.f if scale is None else scale
    if isinstance(x, torch.Tensor):
        xd = x.to(device=_dev.device(), dtype=torch.float64).contiguous()
    else:
        xd = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(_dev.device())
    out = torch.empty(xd.shape, dtype=torch.int64, device=xd.device)
    flag = torch.zeros(1, dtype=torch.int32, device=xd.device)
    if xd.numel():
        _lib.call("pb_encode_fixed", _dev.ptr(xd), xd.numel(), params.ell, scale, _dev.ptr(out), _dev.ptr(flag),
                  _dev.stream())
    limit = float(1 << (params.ell - 1)) / float(1 << scale)
    _check_flag(flag, f"|x| must stay below {limit}")
    return out


def encode_fixed_into(xd: torch.Tensor, params: RingParams, out: torch.Tensor, flag: torch.Tensor,
                      scale: int | None = None) -> None:
    """encode_fixed of a contiguous device float64 tensor into ``out`` (int64,
    same size), asynchronously: ``flag`` (device int32[1]) is zeroed and set
    when some |x| is out of range -- the caller checks it at its next sync."""
    scale = params.f if scale is None else scale
    if xd.dtype != torch.float64 or not xd.is_contiguous() or out.numel() != xd.numel():
        raise ValueError("encode_fixed_into needs a contiguous float64 input and an output of the same size")
    flag.zero_()
    if xd.numel():
        _lib.call("pb_encode_fixed", _dev.ptr(xd), xd.numel(), params.ell, scale, _dev.ptr(out), _dev.ptr(flag),
                  _dev.stream())


def decode_fixed(v, params: RingParams, scale: int | None = None) -> torch.Tensor:  # R:185-191
    scale = params.f if scale is None else scale
    t = _as_device_u64(v).contiguous()
    out = torch.empty(t.shape, dtype=torch.float64, device=t.device)
    if t.numel():
        _lib.call("pb_decode_fixed", _dev.ptr(t), t.numel(), params.ell, scale, _dev.ptr(out), _dev.stream())
    return out


def to_signed(v, params: RingParams) -> torch.Tensor:  # R:194-198
    t = RingTensor(v, 0, params).values
    half = 1 << (params.ell - 1)
    return torch.where(t >= half, t - (1 << params.ell), t)


def encode_tensor(x, params: RingParams, scale: int | None = None) -> RingTensor:  # R:201-203
    scale = params.f if scale is None else scale
    return RingTensor(encode_fixed(x, params, scale), scale, params, _canonical=True)


def arith_shift(x: RingTensor, bits: int) -> RingTensor:  # R:206-211
    """Exact sign-extending right shift of a REVEALED value; scale -= bits."""
    return x._unary(_lib.RING_ARITH_SHIFT, bits, scale=x.scale - bits)


def share_tensor(x: RingTensor, rng: SeededRng) -> tuple[ShareTensor, ShareTensor]:  # R:214-219
    """Split into (MO share, DO share); the MO share is uniform in Z_t."""
    n = x.values.numel()
    mo = torch.empty_like(x.values)
    do = torch.empty_like(x.values)
    off = rng.reserve(n)
    if n:
        sd, sp = rng.np_args()
        _lib.call("pb_share", _dev.ptr(x.values), n, sd, sp, rng.stream, off, x.params.ell, _dev.ptr(mo),
                  _dev.ptr(do), _dev.stream())
    return (ShareTensor(MO, RingTensor(mo, x.scale, x.params, _canonical=True)),
            ShareTensor(DO, RingTensor(do, x.scale, x.params, _canonical=True)))


def reconstruct_tensor(a: ShareTensor, b: ShareTensor) -> RingTensor:  # R:222-225
    if a.owner_role == b.owner_role:
        raise ValueError("reconstruction needs one share from each role")
    return a.value + b.value


def zeros_like(x: RingTensor) -> RingTensor:  # R:228-229
    return RingTensor(torch.zeros_like(x.values), x.scale, x.params, _canonical=True)


def zero_share(role: str, shape, scale: int, params: RingParams) -> ShareTensor:  # R:232-233
    return ShareTensor(role, RingTensor(_dev.zeros_u64(*shape), scale, params, _canonical=True))
