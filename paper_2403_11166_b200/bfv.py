"""RNS-BFV over R_{t,N} on the B200 (the SPEC-only ``bfv`` module).

Operations: ``ntt_transform``, ``keygen`` (:130-138),
``encrypt`` (:139-147), ``decrypt`` (:148-156), ``he_add`` incl. subtraction
and plaintext operands (:157-165), ``he_plain_mul`` (:166-174),
``noise_budget`` (:175-183).  Ciphertexts live in HBM as uint32 residues
[P, 2, L, N] in NTT form.  Conventions (draw order, centered
lift, decode) are the ones the CPU oracle restates (oracle/bfv.py).

Encryption randomness is drawn on the device (Philox4x32) unless the caller
supplies it: BFV decryption returns the exact plaintext for any valid
randomness, so decrypted values -- the only outputs the
protocol reveals -- stay bit-identical to the oracle's, while ciphertext
bytes match the oracle exactly when the oracle's noise is passed in
(``encrypt(..., noise=...)``, used by the parity tests).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .errors import FormError, ParamsError, ShapeError
from .params import BfvParams, context

NTT = "ntt"
COEFF = "coeff"


@dataclass
class RnsPoly:
    data: torch.Tensor  # int32 [P, L, N]
    form: str = NTT
    shoup: torch.Tensor | None = None  # Shoup quotients (plaintext multipliers)


@dataclass
class Ciphertext:
    data: torch.Tensor  # int32 [P, 2, L, N] (c0, c1), NTT form
    params: BfvParams

    @property
    def count(self) -> int:
        return self.data.shape[0]

    def nbytes_wire(self) -> int:
        """PBFV wire size: header + 2 L N little-endian u64 per ct."""
        p = self.params
        return self.count * (4 + 2 + 4 + 1 + 1 + 2 * p.L * p.N * 8)


@dataclass
class KeyPair:
    params: BfvParams
    sk_coeff: np.ndarray  # int64 [N] ternary (host copy for diagnostics)
    sk_ntt: torch.Tensor  # int32 [L, N]
    pk: torch.Tensor  # int32 [2, L, N]
    sk_sh: torch.Tensor | None = None  # int32 [L, N]: Shoup companions of sk_ntt (symmetric encryption)

    def __post_init__(self):
        if self.sk_sh is None:
            self.sk_sh = torch.empty_like(self.sk_ntt)
            _lib.call("pb_shoup_rows", _ctx(self.params), _dev.ptr(self.sk_ntt), _dev.ptr(self.sk_sh),
                      self.sk_ntt.shape[0], _dev.stream())


def _ctx(params: BfvParams):
    return context(params).handle


def _signed_to_zt(v: np.ndarray, params: BfvParams) -> torch.Tensor:
    """Small signed integers -> Z_t bit patterns (two's complement mod t) on device."""
    v = np.asarray(v, dtype=np.int64)
    return _dev.u64_to_device(v.astype(np.uint64) & np.uint64(params.t - 1))


def lift(params: BfvParams, vals: torch.Tensor, centered: bool, n_polys: int | None = None) -> torch.Tensor:
    """Dense Z_t coefficients [P, N] -> RNS residues [P, L, N] (coefficient form)."""
    P = n_polys if n_polys is not None else vals.numel() // params.N
    out = _dev.empty_u32(P, params.L, params.N)
    _lib.call("pb_lift", _ctx(params), _dev.ptr(vals), P, 1 if centered else 0, _dev.ptr(out), _dev.stream())
    return out


def _pack_args(pack):
    """pack = None (dense) or (pos, src) int32 device tensors [P, Z]."""
    if pack is None:
        return None, None, 0, None
    pos, src = pack
    return _dev.ptr(pos), _dev.ptr(src), pos.shape[1], pos.shape[0]


def ntt_transform(params: BfvParams, p: RnsPoly, direction: str) -> RnsPoly:
    if direction not in ("forward", "inverse"):
        raise ValueError("direction must be 'forward' or 'inverse'")
    want = COEFF if direction == "forward" else NTT
    if p.form != want:
        raise FormError(f"{direction} NTT needs {want}-form input, got {p.form}")
    out = p.data.clone()
    rows = out.numel() // params.N
    _lib.call("pb_ntt_forward" if direction == "forward" else "pb_ntt_inverse", _ctx(params), _dev.ptr(out), rows,
              None, _dev.stream())
    return RnsPoly(out, NTT if direction == "forward" else COEFF)


def keygen(params: BfvParams, rng) -> KeyPair:
    """s = ternary(N); a_l = uniform_mod(N, q_l) per limb (NTT domain); e = cbd(N);
    pk = (-(a*s + e), a) -- the oracle's draw order, so keys are bit-identical."""
    N, L = params.N, params.L
    h = _ctx(params)
    st = _dev.stream()
    s = rng.ternary((N,))
    a = np.stack([rng.uniform_mod((N,), q) for q in params.moduli])
    e = rng.cbd((N,))
    se = torch.cat([_signed_to_zt(s, params), _signed_to_zt(e, params)])
    res = lift(params, se, centered=True, n_polys=2)  # [2, L, N]
    _lib.call("pb_ntt_forward", h, _dev.ptr(res), 2 * L, None, st)
    sk = res[0].contiguous()
    en = res[1].contiguous()
    pk = _dev.empty_u32(2, L, N)
    a_d = _dev.u32_to_device(a.astype(np.uint32))
    # a is drawn in the reference's NTT-domain order; store it in device order
    _lib.call("pb_ntt_reorder", h, _dev.ptr(a_d), L, 1, st)
    pk[1].copy_(a_d)
    tmp = _dev.empty_u32(L, N)
    _lib.call("pb_pw", h, _lib.PW_MUL, _dev.ptr(tmp), _dev.ptr(a_d), _dev.ptr(sk), L, L, None, st)
    _lib.call("pb_pw", h, _lib.PW_ADD, _dev.ptr(tmp), _dev.ptr(tmp), _dev.ptr(en), L, L, None, st)
    zero = torch.zeros_like(tmp)
    pk0 = pk[0]
    _lib.call("pb_pw", h, _lib.PW_SUB, _dev.ptr(pk0), _dev.ptr(zero), _dev.ptr(tmp), L, L, None, st)
    return KeyPair(params, s, sk, pk)


def encrypt(kp: KeyPair, m: torch.Tensor, rng=None, *, pack=None, mode: str = "pk", noise=None,
            nonce: int | None = None) -> Ciphertext:
    """SPEC:139-147.  ``m``: Z_t coefficients, dense [P, N], or a flat tensor
    gathered through ``pack`` = (pos, src) int32 [P, Z] (packing maps, see
    poly_encoding.compact).  mode "pk" encrypts under the public key, "sk" is
    symmetric encryption by the key owner.  ``noise`` = (u, e1, e2) int8 [P, N]
    (pk) or (a [P,L,N] in reference NTT order, e int8 [P, N]) (sk)."""
    params = kp.params
    h = _ctx(params)
    m = m.contiguous()
    pp, ps, Z, Pk = _pack_args(pack)
    P = Pk if Pk is not None else m.numel() // params.N
    ct = _dev.empty_u32(P, 2, params.L, params.N)
    st = _dev.stream()
    if noise is not None:
        if mode == "pk":
            u, e1, e2 = (torch.as_tensor(np.asarray(x, dtype=np.int8)).to(_dev.device()) for x in noise)
            _lib.call("pb_encrypt_pk_noise", h, _dev.ptr(kp.pk), _dev.ptr(m), pp, ps, Z, P, _dev.ptr(u),
                      _dev.ptr(e1), _dev.ptr(e2), _dev.ptr(ct), st)
        else:
            a = _dev.u32_to_device(np.asarray(noise[0], dtype=np.uint32))  # reference NTT order
            _lib.call("pb_ntt_reorder", h, _dev.ptr(a), a.numel() // params.N, 1, st)
            e = torch.as_tensor(np.asarray(noise[1], dtype=np.int8)).to(_dev.device())
            _lib.call("pb_encrypt_sk_noise", h, _dev.ptr(kp.sk_ntt), _dev.ptr(m), pp, ps, Z, P, _dev.ptr(a),
                      _dev.ptr(e), _dev.ptr(ct), st)
        return Ciphertext(ct, params)
    if rng is not None:
        seed, sptr = rng.dev_args()
        if nonce is None:
            nonce = rng.reserve(P)
    else:  # SPEC:139-147's encrypt(pk, m) has no rng: fresh OS entropy per call (randomized encryption)
        seed, sptr = int.from_bytes(os.urandom(8), "little"), None
        nonce = int.from_bytes(os.urandom(4), "little") if nonce is None else nonce
    if mode == "pk":
        _lib.call("pb_encrypt_pk", h, _dev.ptr(kp.pk), _dev.ptr(m), pp, ps, Z, P, seed, sptr, nonce, _dev.ptr(ct), st)
    else:
        _lib.call("pb_encrypt_sk", h, _dev.ptr(kp.sk_ntt), _dev.ptr(kp.sk_sh), _dev.ptr(m), pp, ps, Z, P, seed, sptr,
                  nonce, _dev.ptr(ct), st)
    return Ciphertext(ct, params)


def encrypt_zero(kp: KeyPair, P: int, rng, nonce: int | None = None):
    """The message-independent half of ``encrypt(mode="sk")`` for P
    ciphertexts: returns (ct = (-a s, a), e int8 [P, N]).  ``a`` is the draw
    ``encrypt`` makes under the same (rng, nonce); the engine keeps a pool of
    these off the protocol's critical path."""
    params = kp.params
    ct = _dev.empty_u32(P, 2, params.L, params.N)
    e = torch.empty(P, params.N, dtype=torch.int8, device=_dev.device())
    seed, sptr = rng.dev_args()
    if nonce is None:
        nonce = rng.reserve(P)
    _lib.call("pb_encrypt_sk_zero", _ctx(params), _dev.ptr(kp.sk_ntt), P, seed, sptr, nonce, _dev.ptr(ct),
              _dev.ptr(e), _dev.stream())
    return Ciphertext(ct, params), e


def encrypt_add(pre, m: torch.Tensor, *, pack=None) -> Ciphertext:
    """In place on ``pre`` = encrypt_zero(...): c0 += NTT(e + Delta m), giving
    the ciphertext ``encrypt(..., mode="sk", noise=(a, e))`` would."""
    ct, e = pre
    params = ct.params
    m = m.contiguous()
    pp, ps, Z, Pk = _pack_args(pack)
    P = Pk if Pk is not None else m.numel() // params.N
    if P != ct.data.shape[0] or P != e.shape[0]:
        raise ShapeError(f"{P} message polynomials for {ct.data.shape[0]} ciphertexts")
    _lib.call("pb_encrypt_sk_add", _ctx(params), _dev.ptr(m), pp, ps, Z, P, _dev.ptr(e), _dev.ptr(ct.data),
              _dev.stream())
    return ct


def to_reference_order(params: BfvParams, ntt_rows: torch.Tensor) -> np.ndarray:
    """NTT-domain device rows -> host uint64 array in the reference's
    bit-reversed order (what K's ntt_forward produces)."""
    t = ntt_rows.contiguous().clone()
    _lib.call("pb_ntt_reorder", _ctx(params), _dev.ptr(t), t.numel() // params.N, 0, _dev.stream())
    return _dev.to_numpy_u32(t).astype(np.uint64)


def from_reference_order(params: BfvParams, rows) -> torch.Tensor:
    """Host NTT-domain rows in the reference's order -> device-order int32 tensor."""
    t = _dev.u32_to_device(np.asarray(rows, dtype=np.uint32))
    _lib.call("pb_ntt_reorder", _ctx(params), _dev.ptr(t), t.numel() // params.N, 1, _dev.stream())
    return t


def decrypt_coeffs(kp: KeyPair, ct: Ciphertext) -> torch.Tensor:
    """x = INTT(c0 + c1*s), [P, L, N] coefficient residues."""
    p = kp.params
    x = _dev.empty_u32(ct.count, p.L, p.N)
    _lib.call("pb_decrypt_coeffs", _ctx(p), _dev.ptr(kp.sk_ntt), _dev.ptr(ct.data), ct.count, _dev.ptr(x),
              _dev.stream())
    return x


def decrypt(kp: KeyPair, ct: Ciphertext) -> torch.Tensor:
    """Plaintext polynomials [P, N] (Z_t, uint64 bit patterns)."""
    p = kp.params
    m = _dev.empty_u64(ct.count, p.N)
    scratch = _dev.empty_u32(ct.count, p.L, p.N)
    _lib.call("pb_decrypt", _ctx(p), _dev.ptr(kp.sk_ntt), _dev.ptr(ct.data), ct.count, _dev.ptr(m), _dev.ptr(scratch),
              _dev.stream())
    return m


def encode_plain(params: BfvParams, m: torch.Tensor, pack=None) -> RnsPoly:
    """Plaintext multiplier: centered lift + NTT + Shoup quotients.
    ``m`` dense [P, N] Z_t coefficients, or flat values gathered through ``pack``."""
    m = m.contiguous()
    pp, ps, Z, Pk = _pack_args(pack)
    P = Pk if Pk is not None else m.numel() // params.N
    pt = _dev.empty_u32(P, params.L, params.N)
    sh = _dev.empty_u32(P, params.L, params.N)
    _lib.call("pb_encode_plain", _ctx(params), _dev.ptr(m), pp, ps, Z, P, _dev.ptr(pt), _dev.ptr(sh), _dev.stream())
    return RnsPoly(pt, NTT, sh)


def _check_pair(a: Ciphertext, b: Ciphertext):
    if a.params != b.params:
        raise ParamsError("ciphertexts under different parameters")
    if a.data.shape != b.data.shape:
        raise ShapeError("ciphertext batch shapes differ")


def he_add(a: Ciphertext, b, subtract: bool = False) -> Ciphertext:
    """ct + ct, or ct + plaintext (Z_t coefficients [P, N]); subtract=True for ct - b."""
    p = a.params
    h = _ctx(p)
    st = _dev.stream()
    out = a.data.clone()
    rows = out.numel() // p.N
    op = _lib.PW_SUB if subtract else _lib.PW_ADD
    if isinstance(b, Ciphertext):
        _check_pair(a, b)
        _lib.call("pb_pw", h, op, _dev.ptr(out), _dev.ptr(a.data), _dev.ptr(b.data), rows, rows, None, st)
        return Ciphertext(out, p)
    m = torch.as_tensor(b).to(_dev.device()).contiguous()
    P = a.count
    if m.numel() != P * p.N:
        raise ShapeError("plaintext batch does not match the ciphertext batch")
    # Delta*m in the NTT domain: lift unsigned, scale by Delta via a ct-free MAC is
    # not needed -- Delta*m mod q is a pointwise product with the Delta row.
    dm = lift(p, m, centered=False, n_polys=P)
    delta = _dev.u32_to_device(np.array([[p.delta % q] * p.N for q in p.moduli], dtype=np.uint32))
    _lib.call("pb_pw", h, _lib.PW_MUL, _dev.ptr(dm), _dev.ptr(dm), _dev.ptr(delta), P * p.L, p.L, None, st)
    _lib.call("pb_ntt_forward", h, _dev.ptr(dm), P * p.L, None, st)
    c0 = out[:, 0].contiguous()
    _lib.call("pb_pw", h, op, _dev.ptr(c0), _dev.ptr(c0), _dev.ptr(dm), P * p.L, P * p.L, None, st)
    out[:, 0].copy_(c0)
    return Ciphertext(out, p)


def he_plain_mul(ct: Ciphertext, w) -> Ciphertext:
    """ct (*) w for a plaintext multiplier w: an RnsPoly from encode_plain, or
    Z_t coefficients [P, N] / [N] (centered-lifted here)."""
    p = ct.params
    if not isinstance(w, RnsPoly):
        w = encode_plain(p, torch.as_tensor(w).to(_dev.device()).reshape(-1, p.N))
    if w.form != NTT:
        raise FormError("plaintext multiplier must be in NTT form")
    P = ct.count
    npt = w.data.shape[0]
    if npt not in (1, P):
        raise ShapeError("one plaintext, or one per ciphertext")
    terms = np.zeros((P, 1, 2), dtype=np.int32)
    terms[:, 0, 0] = np.arange(P)
    terms[:, 0, 1] = 0 if npt == 1 else np.arange(P)
    terms_d = _dev.i32_to_device(terms)
    out = _dev.empty_u32(P, 2, p.L, p.N)
    _lib.call("pb_ctpt_mac_mask", _ctx(p), _dev.ptr(ct.data), _dev.ptr(w.data), _dev.ptr(w.shoup), _dev.ptr(terms_d), 1,
              P, None, None, 0, None, 0, 0, None, _dev.ptr(out), _dev.stream())
    return Ciphertext(out, p)


def noise_budget(kp: KeyPair, ct: Ciphertext, slots=None) -> int:
    """Invariant noise budget log2(Q) - log2(|t*x mod Q|_inf) - 1 of ct[0].
    A diagnostic: the INTT runs on the device, the CRT lift on the host.
    ``slots`` restricts the maximum to the given coefficient positions (the
    useful slots of a masked protocol ciphertext, whose other coefficients
    carry uniform filler by design)."""
    p = kp.params
    x = _dev.to_numpy_u32(decrypt_coeffs(kp, Ciphertext(ct.data[:1].contiguous(), p)))[0]
    Q, t = p.Q, p.t
    idx = list(range(p.N)) if slots is None else [int(j) for j in slots if int(j) >= 0]
    comp = [0] * len(idx)
    for l, q in enumerate(p.moduli):
        Ml = Q // q
        c = Ml * pow(Ml % q, -1, q)
        row = x[l]
        for n, j in enumerate(idx):
            comp[n] += int(row[j]) * c
    worst = 0
    for v in comp:
        w = (v % Q) * t % Q
        worst = max(worst, min(w, Q - w))
    if worst == 0:
        return int(math.log2(Q)) - 1
    return max(0, int(math.floor(math.log2(Q) - math.log2(worst) - 1)))


def drop_params(params: BfvParams) -> BfvParams:
    """The parameter set after one modulus switch: q_0..q_{L-2}."""
    if params.L < 2:
        raise ParamsError("modulus switching needs at least 2 limbs")
    return BfvParams(N=params.N, ell=params.ell, moduli=params.moduli[:-1])


def drop_keys(kp: KeyPair) -> KeyPair:
    """The key pair restricted to q_0..q_{L-2} (the NTT rows of the kept limbs)."""
    p = drop_params(kp.params)
    return KeyPair(p, kp.sk_coeff, kp.sk_ntt[: p.L].contiguous(), kp.pk[:, : p.L].contiguous())


def mod_switch_drop(ct: Ciphertext) -> Ciphertext:
    """Response compaction: drop the last RNS limb, c' = round(c * Q'/Q).
    Decrypts under ``drop_keys(kp)`` to the same plaintext; wire bytes
    shrink by 1/L.  OFF by default in the protocols, as SPEC:196 says."""
    p = ct.params
    lo = drop_params(p)
    last = BfvParams(N=p.N, ell=p.ell, moduli=p.moduli[-1:])
    out = _dev.empty_u32(ct.count, 2, lo.L, p.N)
    scratch = _dev.empty_u32(ct.count * 2, p.N)
    _lib.call("pb_mod_switch_drop", _ctx(lo), _ctx(last), _dev.ptr(ct.data.contiguous()), 2 * ct.count,
              _dev.ptr(out), _dev.ptr(scratch), _dev.stream())
    return Ciphertext(out, lo)
