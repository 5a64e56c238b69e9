"""ORACLE — TEST INFRASTRUCTURE ONLY.

BFV parameter derivation for the CPU oracle (restated independently of the
product's ``paper_2403_11166_b200.params``; tests assert the two agree
through the params digest).

Follows SURVEY.md Appendix A ("NTT tables (K convention)", "BFV from K"):
  * moduli: the L largest primes q < 2^30 with q = 1 (mod 2N)  (set A, SURVEY §0 fact 3;
    K:4-5 requires q < 2^31, the device engine requires q < 2^30 for lazy u32 butterflies);
  * psi: g^((q-1)/2N) for the smallest g >= 2 with psi^N = -1 (mod q);
  * psi_brv[i] = psi^bitrev(i), ipsi_brv[i] = psi^-bitrev(i), n_inv = N^-1   (K:22-29);
  * Delta = floor(q/t); Garner prefix_inv[i] = (q_0...q_{i-1})^-1 mod q_i  (K:158-179);
  * scale_round int_part[i] = floor(t*P_{i-1}/q) mod 2^64,
    frac_part[i] = frac(t*P_{i-1}/q) as float64  (K:182-199).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np


def _is_prime(n: int) -> bool:
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


@lru_cache(maxsize=None)
def ntt_primes(N: int, L: int, bits: int = 30) -> tuple[int, ...]:
    """The L largest primes below 2^bits with q = 1 mod 2N, descending."""
    out = []
    step = 2 * N
    c = ((1 << bits) - 1) // step * step + 1
    while len(out) < L:
        if c < (1 << bits) and _is_prime(c):
            out.append(c)
        c -= step
        if c <= step:
            raise ValueError("not enough NTT primes")
    return tuple(out)


def find_psi(q: int, N: int) -> int:
    e = (q - 1) // (2 * N)
    g = 2
    while True:
        psi = pow(g, e, q)
        if pow(psi, N, q) == q - 1:
            return psi
        g += 1


def bitrev(i: int, logn: int) -> int:
    return int(format(i, f"0{logn}b")[::-1], 2) if logn else 0


@dataclass(frozen=True)
class OracleBfvParams:
    N: int = 8192
    L: int = 7
    ell: int = 59
    moduli: tuple = ()
    psi: tuple = ()
    tables: dict = field(default_factory=dict, compare=False, hash=False, repr=False)

    @property
    def t(self) -> int:
        return 1 << self.ell

    @property
    def q(self) -> int:
        out = 1
        for m in self.moduli:
            out *= m
        return out

    def digest(self) -> str:
        s = f"N={self.N};ell={self.ell};q={','.join(map(str, self.moduli))};psi={','.join(map(str, self.psi))};lift=centered"
        return hashlib.sha256(s.encode()).hexdigest()[:16]


def make_params(N: int = 8192, L: int = 7, ell: int = 59, moduli=None) -> OracleBfvParams:
    moduli = tuple(int(m) for m in (moduli or ntt_primes(N, L)))
    psi = tuple(find_psi(q, N) for q in moduli)
    p = OracleBfvParams(N=N, L=len(moduli), ell=ell, moduli=moduli, psi=psi)
    p.tables.update(_tables(p))
    return p


def _tables(p: OracleBfvParams) -> dict:
    N, L = p.N, p.L
    logn = N.bit_length() - 1
    brv = np.array([bitrev(i, logn) for i in range(N)], dtype=np.int64)
    psi_brv = np.empty((L, N), dtype=np.uint64)
    ipsi_brv = np.empty((L, N), dtype=np.uint64)
    for l, (q, psi) in enumerate(zip(p.moduli, p.psi)):
        pw = np.empty(N, dtype=object)
        ipsi = pow(psi, -1, q)
        acc, iacc = 1, 1
        pows, ipows = [0] * N, [0] * N
        for k in range(N):
            pows[k], ipows[k] = acc, iacc
            acc = acc * psi % q
            iacc = iacc * ipsi % q
        psi_brv[l] = np.array([pows[b] for b in brv], dtype=np.uint64)
        ipsi_brv[l] = np.array([ipows[b] for b in brv], dtype=np.uint64)
        del pw
    q_arr = np.array(p.moduli, dtype=np.uint64)
    n_inv = np.array([pow(N, -1, q) for q in p.moduli], dtype=np.uint64)
    Q, t = p.q, p.t
    delta = Q // t
    prefix_inv, int_part, frac_part = [], [], []
    P = 1
    for q in p.moduli:
        prefix_inv.append(pow(P % q, -1, q) if P != 1 else 1)
        num = t * P
        int_part.append((num // Q) % (1 << 64))
        frac_part.append((num % Q) / Q)  # correctly rounded int/int division
        P *= q
    return dict(
        psi_brv=psi_brv,
        ipsi_brv=ipsi_brv,
        q=q_arr,
        n_inv=n_inv,
        delta_mod_q=np.array([delta % q for q in p.moduli], dtype=np.uint64),
        prefix_inv=np.array(prefix_inv, dtype=np.uint64),
        int_part=np.array(int_part, dtype=np.uint64),
        frac_part=np.array(frac_part, dtype=np.float64),
        delta=delta,
    )
