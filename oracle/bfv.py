"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the SPEC-only ``bfv`` module (PAPER.md
§II-B, 744-750) built exclusively from the reference kernel arithmetic
(K = pencil._kernels): every NTT / pointwise / decode step calls either the C
restatement in oracle/kernels.c (default) or -- when generating golden
vectors in the build container -- the real K functions themselves
(``Arith(params, kernels=pencil._kernels)``).  Only lifts, RNG draws and
index glue live here.

Conventions fixed by this oracle (and shared bit-for-bit by the device
engine):
  * ciphertexts and keys are stored in NTT form, shape (2, L, N);
  * keygen draw order: s = ternary(N); a_l = uniform_mod(N, q_l) for each
    limb l (sampled directly in the NTT domain); e = cbd(N);
    pk = (-(a*s + e), a);
  * encrypt_pk draw order: u = ternary(N), e1 = cbd(N), e2 = cbd(N);
    c0 = pk0*NTT(u) + NTT(e1 + Delta*m), c1 = pk1*NTT(u) + NTT(e2);
  * encrypt_sk draw order: a_l = uniform_mod(N, q_l) per limb, e = cbd(N);
    c1 = a, c0 = NTT(e + Delta*m) - a*s;
  * plaintext multipliers use the CENTERED lift v >= t/2 -> v - t
    (the unsigned lift fails decryption);
  * decrypt: x = INTT(c0 + c1*s); m = garner_digits + scale_round_digits.
"""

from __future__ import annotations

import math

import numpy as np

from . import kernels as OK
from .params import OracleBfvParams


class Arith:
    """Batched (P, L, N) polynomial arithmetic routed to the K algorithms."""

    def __init__(self, params: OracleBfvParams, kernels=None):
        self.p = params
        self.K = kernels  # None -> oracle C (cyclic tables); else a K-API module
        tb = params.tables
        self.q = tb["q"]
        self.psi_brv = tb["psi_brv"]
        self.ipsi_brv = tb["ipsi_brv"]
        self.n_inv = tb["n_inv"]

    # -- helpers for the real-K path: K wants one table row per data row --
    def _tile(self, tab, P):
        return np.ascontiguousarray(np.tile(tab, (P, 1)))

    def ntt_fwd(self, a):
        P, L, N = a.shape
        rows = a.reshape(P * L, N)
        if self.K is None:
            OK.ntt_forward_cyc(rows, self.psi_brv, self.q)
        else:
            self.K.ntt_forward(rows, self._tile(self.psi_brv, P), np.tile(self.q, P))
        return a

    def ntt_inv(self, a):
        P, L, N = a.shape
        rows = a.reshape(P * L, N)
        if self.K is None:
            OK.ntt_inverse_cyc(rows, self.ipsi_brv, self.n_inv, self.q)
        else:
            self.K.ntt_inverse(
                rows, self._tile(self.ipsi_brv, P), np.tile(self.n_inv, P), np.tile(self.q, P)
            )
        return a

    def _pw(self, op, out, a, b):
        P, L, N = a.shape
        if self.K is None:
            bb = b.reshape(-1, N)
            OK.pw_cyc(op, out.reshape(P * L, N), a.reshape(P * L, N), bb, self.q)
            return out
        bfull = np.ascontiguousarray(np.broadcast_to(b, a.shape)).reshape(P * L, N)
        fn = {"mul": self.K.pw_mul, "mul_acc": self.K.pw_mul_acc, "add": self.K.pw_add,
              "sub": self.K.pw_sub}[op]
        fn(out.reshape(P * L, N), a.reshape(P * L, N), bfull, np.tile(self.q, P))
        return out

    def mul(self, a, b):
        return self._pw("mul", np.empty_like(a), a, b)

    def mac(self, acc, a, b):
        return self._pw("mul_acc", acc, a, b)

    def add(self, a, b):
        return self._pw("add", np.empty_like(a), a, b)

    def sub(self, a, b):
        return self._pw("sub", np.empty_like(a), a, b)

    def decode(self, x):
        """x (P, L, N) coefficient-form residues -> (P, N) round(t x / q) mod t."""
        tb = self.p.tables
        tmask = np.uint64(self.p.t - 1)
        if self.K is None:
            return OK.decode_batch(x, self.q, tb["prefix_inv"], tb["int_part"], tb["frac_part"], tmask)
        out = np.empty((x.shape[0], x.shape[2]), dtype=np.uint64)
        for i in range(x.shape[0]):
            d = self.K.garner_digits(np.ascontiguousarray(x[i]), self.q, tb["prefix_inv"])
            out[i] = self.K.scale_round_digits(d, tb["int_part"], tb["frac_part"], tmask)
        return out


# ---------------------------------------------------------------- lifts ---

def lift_signed(v, p: OracleBfvParams):
    """int64 (..., N) small signed values -> (..., L, N) residues."""
    v = np.asarray(v, dtype=np.int64)
    q = np.array(p.moduli, dtype=np.int64)
    return (v[..., None, :] % q[:, None]).astype(np.uint64)


def lift_unsigned(m, p: OracleBfvParams):
    """Z_t values (uint64) -> residues m mod q_l."""
    m = np.asarray(m, dtype=np.uint64)
    q = np.array(p.moduli, dtype=np.uint64)
    return np.ascontiguousarray(m[..., None, :] % q[:, None])


def lift_centered(m, p: OracleBfvParams):
    """Centered lift of Z_t values: v >= t/2 -> v - t."""
    m = np.asarray(m, dtype=np.uint64)
    half = np.uint64(p.t // 2)
    neg = m >= half
    q = np.array(p.moduli, dtype=np.uint64)
    pos_part = m[..., None, :] % q[:, None]
    # t - v for the negative branch, reduced, then q - (.) mod q
    negmag = (np.uint64(p.t) - m)[..., None, :] % q[:, None]
    negres = (q[:, None] - negmag) % q[:, None]
    return np.ascontiguousarray(np.where(neg[..., None, :], negres, pos_part))


def delta_m(m, p: OracleBfvParams, ar: Arith):
    """Delta * m mod q_l for Z_t values m (..., N) -> (P, L, N)."""
    mm = lift_unsigned(m, p).reshape(-1, p.L, p.N)
    dl = np.broadcast_to(p.tables["delta_mod_q"][:, None], (p.L, p.N)).astype(np.uint64)
    return ar.mul(mm, np.ascontiguousarray(dl))


# -------------------------------------------------------------- scheme ---

class KeyPair:
    def __init__(self, sk_coeff, sk_ntt, pk):
        self.sk_coeff = sk_coeff  # int64 (N,)
        self.sk_ntt = sk_ntt  # uint64 (L, N)
        self.pk = pk  # uint64 (2, L, N)


def keygen(p: OracleBfvParams, rng, ar: Arith) -> KeyPair:
    s = rng.ternary((p.N,))
    a = np.stack([rng.uniform_mod((p.N,), q) for q in p.moduli])
    e = rng.cbd((p.N,))
    sk = ar.ntt_fwd(lift_signed(s, p)[None].copy())[0]
    en = ar.ntt_fwd(lift_signed(e, p)[None].copy())
    a3 = np.ascontiguousarray(a[None])
    as_ = ar.add(ar.mul(a3, sk), en)
    pk0 = ar.sub(np.zeros_like(as_), as_)
    return KeyPair(s, sk, np.concatenate([pk0, a3], axis=0))


def encrypt_pk(p: OracleBfvParams, kp: KeyPair, m, rng, ar: Arith):
    """m (P, N) Z_t -> ct (P, 2, L, N); draws u, e1, e2 per ciphertext in order."""
    m = np.atleast_2d(np.asarray(m, dtype=np.uint64))
    P = m.shape[0]
    out = np.empty((P, 2, p.L, p.N), dtype=np.uint64)
    dm = delta_m(m, p, ar)
    for i in range(P):
        u = rng.ternary((p.N,))
        e1 = rng.cbd((p.N,))
        e2 = rng.cbd((p.N,))
        U = ar.ntt_fwd(lift_signed(u, p)[None].copy())
        E1 = ar.ntt_fwd(ar.add(lift_signed(e1, p)[None].copy(), dm[i : i + 1]))
        E2 = ar.ntt_fwd(lift_signed(e2, p)[None].copy())
        out[i, 0] = ar.add(ar.mul(U, kp.pk[0]), E1)[0]
        out[i, 1] = ar.add(ar.mul(U, kp.pk[1]), E2)[0]
    return out


def encrypt_sk(p: OracleBfvParams, kp: KeyPair, m, rng, ar: Arith):
    """Symmetric-key BFV encryption (the DO encrypts under its own key)."""
    m = np.atleast_2d(np.asarray(m, dtype=np.uint64))
    P = m.shape[0]
    out = np.empty((P, 2, p.L, p.N), dtype=np.uint64)
    dm = delta_m(m, p, ar)
    for i in range(P):
        a = np.stack([rng.uniform_mod((p.N,), q) for q in p.moduli])[None]
        e = rng.cbd((p.N,))
        E = ar.ntt_fwd(ar.add(lift_signed(e, p)[None].copy(), dm[i : i + 1]))
        out[i, 0] = ar.sub(E, ar.mul(np.ascontiguousarray(a), kp.sk_ntt))[0]
        out[i, 1] = a[0]
    return out


def decrypt_coeffs(p: OracleBfvParams, kp: KeyPair, ct, ar: Arith):
    """x = INTT(c0 + c1*s): (P, L, N) coefficient residues."""
    ct = np.asarray(ct, dtype=np.uint64).reshape(-1, 2, p.L, p.N)
    c0 = np.ascontiguousarray(ct[:, 0])
    c1 = np.ascontiguousarray(ct[:, 1])
    x = ar.add(ar.mul(c1, kp.sk_ntt), c0)
    return ar.ntt_inv(x)


def decrypt(p: OracleBfvParams, kp: KeyPair, ct, ar: Arith):
    return ar.decode(decrypt_coeffs(p, kp, ct, ar))


def encode_plain(p: OracleBfvParams, m, ar: Arith):
    """Plaintext multiplier: centered lift + NTT -> (P, L, N)."""
    m = np.atleast_2d(np.asarray(m, dtype=np.uint64))
    return ar.ntt_fwd(lift_centered(m, p).reshape(-1, p.L, p.N).copy())


def he_add(a, b, ar: Arith):  # SPEC:157-165 (ct + ct)
    P = a.shape[0]
    L, N = a.shape[2], a.shape[3]
    return ar.add(a.reshape(P * 2, L, N), b.reshape(P * 2, L, N)).reshape(a.shape)


def he_add_plain(p, ct, m, ar: Arith, subtract=False):  # SPEC:157-165 (ct +/- plaintext)
    out = ct.copy()
    dm = ar.ntt_fwd(delta_m(m, p, ar))
    c0 = np.ascontiguousarray(out[:, 0])
    out[:, 0] = ar.sub(c0, dm) if subtract else ar.add(c0, dm)
    return out


def he_plain_mul(ct, pt, ar: Arith):
    """ct (P, 2, L, N) * pt (P, L, N) or (L, N)."""
    P, _, L, N = ct.shape
    pt = np.asarray(pt).reshape(-1, L, N)
    ptr = np.repeat(pt, 2, axis=0) if pt.shape[0] == P else pt
    return ar.mul(np.ascontiguousarray(ct.reshape(P * 2, L, N)), np.ascontiguousarray(ptr)).reshape(ct.shape)


def noise_budget(p: OracleBfvParams, kp: KeyPair, ct, ar: Arith) -> int:
    """SEAL-style invariant noise budget: log2(q) - log2(|t*x mod q|_inf) - 1."""
    x = decrypt_coeffs(p, kp, ct, ar)[0]
    Q, t = p.q, p.t
    mods = p.moduli
    # CRT compose with Python ints
    comp = [0] * p.N
    for l, q in enumerate(mods):
        Ml = Q // q
        c = Ml * pow(Ml % q, -1, q)
        xl = x[l].tolist()
        for j in range(p.N):
            comp[j] += xl[j] * c
    worst = 0
    for j in range(p.N):
        v = (comp[j] % Q) * t % Q
        if v > Q // 2:
            v = Q - v
        worst = max(worst, v)
    if worst == 0:
        return int(math.log2(Q)) - 1
    return max(0, int(math.floor(math.log2(Q) - math.log2(worst) - 1)))


def mod_switch_drop(p: OracleBfvParams, ct):
    """SPEC:196 response compaction (OFF by default; the reference ships no
    implementation, so this restates the textbook BFV modulus switch):
    ct (P, 2, L, N) NTT form, reference order -> (params', ct') under
    Q' = Q / q_{L-1}, c'_i = (c_i - [c]_{q_{L-1}}) * q_{L-1}^-1 mod q_i with the
    centered coefficient-form residue of the dropped limb."""
    from .params import make_params

    ct = np.asarray(ct, dtype=np.uint64)
    P, _, L, N = ct.shape
    q_last = int(p.moduli[-1])
    lo = make_params(N, ell=p.ell, moduli=p.moduli[:-1])
    last = make_params(N, ell=p.ell, moduli=(q_last,))
    a = ct[:, :, L - 1, :].reshape(P * 2, 1, N).copy()
    Arith(last).ntt_inv(a)
    a = a.reshape(P * 2, N).astype(np.int64)
    ac = np.where(a > q_last // 2, a - q_last, a)
    x = np.stack([np.mod(ac, q) for q in lo.moduli], axis=1).astype(np.uint64)
    Arith(lo).ntt_fwd(x)
    qv = np.array(lo.moduli, dtype=np.uint64)[None, :, None]
    inv = np.array([pow(q_last, -1, int(q)) for q in lo.moduli], dtype=np.uint64)[None, :, None]
    c = ct[:, :, : L - 1, :].reshape(P * 2, L - 1, N)
    out = ((c + qv - x) % qv) * inv % qv
    return lo, out.reshape(P, 2, L - 1, N)
