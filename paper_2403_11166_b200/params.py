"""BFV parameter sets and the device context (SPEC.md:103-106 BfvParams).

Default: N = 8192, t = 2^59, L = 7 primes q_i < 2^30 with q_i = 1 mod 2N
(set A: log2 Q = 210, 4q < 2^32 so lazy u32 butterflies fit).
The reference kernels need q < 2^31 (K:4-5); this engine needs q < 2^30.

psi_i is g^((q-1)/2N) for the smallest g >= 2 with psi^N = -1, the convention
the CPU oracle shares (the params digest proves both sides agree).  All
big-integer constants (Delta = floor(Q/t), Garner inverses, scale-round
int/frac parts of t*P_{i-1}/Q, K:158-199) are derived here with Python ints
and handed to the C ABI as words.
"""

from __future__ import annotations

import ctypes
import hashlib
from dataclasses import dataclass
from functools import lru_cache

from . import _lib
from .errors import ParamsError


def _is_prime(n: int) -> bool:
    if n < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


@lru_cache(maxsize=None)
def default_moduli(N: int, L: int, bits: int = 30) -> tuple:
    """The L largest primes below 2^bits that are 1 mod 2N (descending)."""
    out, step = [], 2 * N
    c = ((1 << bits) - 1) // step * step + 1
    while len(out) < L:
        if c < (1 << bits) and _is_prime(c):
            out.append(c)
        c -= step
        if c <= step:
            raise ParamsError("not enough NTT-friendly primes")
    return tuple(out)


def primitive_2n_root(q: int, N: int) -> int:
    e = (q - 1) // (2 * N)
    g = 2
    while True:
        psi = pow(g, e, q)
        if pow(psi, N, q) == q - 1:
            return psi
        g += 1


@lru_cache(maxsize=None)
def _psis(moduli: tuple, N: int) -> tuple:
    return tuple(primitive_2n_root(q, N) for q in moduli)


@dataclass(frozen=True)
class BfvParams:
    """SPEC:103-106.  ``moduli`` empty -> the set-A default for (N, L)."""

    N: int = 8192
    L: int = 7
    ell: int = 59
    moduli: tuple = ()
    psi_override: tuple = ()  # explicit 2N-th roots (K-compat shim); default derived

    def __post_init__(self):
        if self.N & (self.N - 1) or not (4 <= self.N <= 32768):
            raise ParamsError("N must be a power of two in [4, 32768]")
        if not self.moduli:
            object.__setattr__(self, "moduli", default_moduli(self.N, self.L))
        object.__setattr__(self, "moduli", tuple(int(q) for q in self.moduli))
        object.__setattr__(self, "L", len(self.moduli))
        if not (1 <= self.L <= _lib.MAX_LIMBS):
            raise ParamsError("1 <= L <= 8 limbs")
        for q in self.moduli:
            if q >= (1 << 30) or (q - 1) % (2 * self.N) or not _is_prime(q):
                raise ParamsError(f"modulus {q} must be a prime < 2^30 with q = 1 mod 2N")
        if not (2 <= self.ell <= 62):
            raise ParamsError("ell must be in [2, 62]")

    @property
    def t(self) -> int:
        return 1 << self.ell

    @property
    def Q(self) -> int:
        out = 1
        for q in self.moduli:
            out *= q
        return out

    @property
    def psi(self) -> tuple:
        if self.psi_override:
            return tuple(int(p) for p in self.psi_override)
        return _psis(self.moduli, self.N)

    @property
    def delta(self) -> int:
        return self.Q // self.t

    def digest(self) -> str:
        """Identity of (N, t, moduli, psi, lift convention) shared with the oracle."""
        s = (
            f"N={self.N};ell={self.ell};q={','.join(map(str, self.moduli))};"
            f"psi={','.join(map(str, self.psi))};lift=centered"
        )
        return hashlib.sha256(s.encode()).hexdigest()[:16]

    def to_c(self) -> _lib.PbParams:
        c = _lib.PbParams()
        c.N, c.L, c.ell = self.N, self.L, self.ell
        Q, t = self.Q, self.t
        P = 1
        psi = self.psi
        for i, q in enumerate(self.moduli):
            c.q[i] = q
            c.psi[i] = psi[i]
            c.delta_mod_q[i] = self.delta % q
            c.garner_prefix_inv[i] = pow(P % q, -1, q) if P != 1 else 1
            num = t * P
            c.scale_int[i] = (num // Q) % (1 << 64)
            c.scale_frac[i] = (num % Q) / Q
            P *= q
        return c


class DeviceContext:
    """Owns a ``pb_ctx`` (device twiddle tables + constants) for one params set."""

    def __init__(self, params: BfvParams, c_params: _lib.PbParams | None = None):
        from . import _dev

        _dev.require_cuda()
        self.params = params
        self._c = c_params if c_params is not None else params.to_c()
        h = ctypes.c_void_p()
        _lib.call("pb_ctx_create", ctypes.byref(self._c), ctypes.byref(h))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib._lib is not None:
            try:
                _lib._lib.pb_ctx_destroy(h)
            except Exception:
                pass
            self.handle = None


_CTX_CACHE: dict = {}


def context(params: BfvParams) -> DeviceContext:
    import torch

    key = (params, torch.cuda.current_device() if torch.cuda.is_available() else -1)
    ctx = _CTX_CACHE.get(key)
    if ctx is None:
        ctx = DeviceContext(params)
        _CTX_CACHE[key] = ctx
    return ctx
