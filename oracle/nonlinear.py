"""ORACLE — TEST INFRASTRUCTURE ONLY.

The OT-based non-linear protocols of SPEC:491-581 (PAPER:1248-1268,
CrypTFlow2-style), restated in numpy with SPEC:479's dealer OT backend (the
receiver obtains message[choice]); the checker for
paper_2403_11166_b200/csrc/pb_nonlinear.cu.  Party 0 is the MO, party 1 the DO.

    cmp_lt      XOR shares of 1{a < b}: 4-bit blocks, one 1-of-16 OT per block
                of P0's (lt, eq) table masked with P0's random bits, blocks
                combined pairwise (lo = 2i, hi = 2i + 1, an odd last node
                passes through) by lt = lt_hi ^ (eq_hi & lt_lo),
                eq = eq_hi & eq_lo with Beaver bit triples (u0,u1,v0,v1,w0
                = 5 consecutive bits of the triple words)
    drelu       1{x >= 0} = 1 ^ MSB(x0) ^ MSB(x1) ^ 1{2^(l-1)-1-x0' < x1'}
    mux         d * x with two 1-of-2 OTs (CrypTFlow2 Alg. 6)
    trunc       faithful arith_shift(x, k) by the wrap / low-carry comparisons + B2A

Randomness: raw draw (raw_offset + i * WORDS + k) of the numpy Philox stream
SeededRng(seed, stream_id) -- R:48-58's generator -- per element i.
"""

from __future__ import annotations

import numpy as np

U64 = np.uint64
W_DRELU, W_MUX, W_TRUNC = 4, 2, 9
WORDS = {"drelu": W_DRELU, "mux": W_MUX, "trunc": W_TRUNC, "relu_trunc": W_DRELU + W_MUX + W_TRUNC,
         "trunc_mux": W_TRUNC + W_MUX}


def raw_words(seed: int, stream: int, n: int, words: int, offset: int = 0) -> np.ndarray:
    """(n, words) raw Philox4x64 outputs of the numpy stream key=[seed, stream], from raw index offset."""
    bg = np.random.Philox(key=[seed, stream])
    return bg.random_raw(offset + n * words)[offset:].astype(U64).reshape(n, words)


def _bits(v, s, k=1):
    return (np.asarray(v, dtype=U64) >> U64(s)) & U64((1 << k) - 1)


def _and(x0, x1, y0, y1, t):
    u0, u1, v0, v1, w0 = (_bits(t, i) for i in range(5))
    w1 = ((u0 ^ u1) & (v0 ^ v1)) ^ w0
    d = (x0 ^ u0) ^ (x1 ^ u1)
    e = (y0 ^ v0) ^ (y1 ^ v1)
    return w0 ^ (d & v0) ^ (e & u0) ^ (d & e), w1 ^ (d & v1) ^ (e & u1)


def _triple(tw, t):
    """5 bits number t of the little-endian bit string of the triple words tw (n, k)."""
    bit = 5 * t
    i, o = bit // 64, bit % 64
    v = tw[:, i] >> U64(o)
    if o > 59:
        v = v | (tw[:, i + 1] << U64(64 - o))
    return v & U64(31)


def cmp_lt(a, b, nbits, lt0m, eq0m, tw):
    """(c0, c1) XOR shares of 1{a < b} per element (vectors of u64)."""
    q = (nbits + 3) // 4
    L0, L1, E0, E1 = [], [], [], []
    for j in range(q):
        aj, bj = _bits(a, 4 * j, 4), _bits(b, 4 * j, 4)
        l0, e0 = _bits(lt0m, j), _bits(eq0m, j)
        L0.append(l0)
        E0.append(e0)
        L1.append(l0 ^ (aj < bj).astype(U64))
        E1.append(e0 ^ (aj == bj).astype(U64))
    t = 0
    while len(L0) > 1:
        nL0, nL1, nE0, nE1 = [], [], [], []
        for i in range(0, len(L0) - 1, 2):
            a0, a1 = _and(E0[i + 1], E1[i + 1], L0[i], L1[i], _triple(tw, t))
            b0, b1 = _and(E0[i + 1], E1[i + 1], E0[i], E1[i], _triple(tw, t + 1))
            t += 2
            nL0.append(L0[i + 1] ^ a0)
            nL1.append(L1[i + 1] ^ a1)
            nE0.append(b0)
            nE1.append(b1)
        if len(L0) & 1:
            nL0.append(L0[-1])
            nL1.append(L1[-1])
            nE0.append(E0[-1])
            nE1.append(E1[-1])
        L0, L1, E0, E1 = nL0, nL1, nE0, nE1
    return L0[0], L1[0]


def _lmask(ell):
    return U64((1 << ell) - 1)


def drelu(x0, x1, ell, w):
    """w: (n, >= 4) words. Returns (d0, d1)."""
    h = ell - 1
    hm = U64((1 << h) - 1)
    lw = w[:, 0]
    c0, c1 = cmp_lt(hm - (x0 & hm), x1 & hm, h, lw & U64(0xFFFF), (lw >> U64(16)) & U64(0xFFFF), w[:, 1:4])
    return U64(1) ^ _bits(x0, h) ^ c0, _bits(x1, h) ^ c1


def mux(d0, d1, x0, x1, ell, w):
    """w: (n, >= 2) words (r0, r1). Returns arithmetic shares of d * x."""
    m = _lmask(ell)
    r0, r1 = w[:, 0] & m, w[:, 1] & m
    zero = np.zeros_like(x0)
    m0 = (U64(0) - r0 + np.where(d0 == 1, x0, zero), U64(0) - r0 + np.where(d0 == 1, zero, x0))  # P0 sends
    m1 = (U64(0) - r1 + np.where(d1 == 1, x1, zero), U64(0) - r1 + np.where(d1 == 1, zero, x1))  # P1 sends
    y1 = np.where(d1 == 1, m0[1], m0[0])  # 1-of-2 OT, P1's choice d1
    y0 = np.where(d0 == 1, m1[1], m1[0])  # 1-of-2 OT, P0's choice d0
    return (r0 + y0) & m, (r1 + y1) & m


def trunc(x0, x1, ell, k, w):
    """w: (n, >= 9) words. Faithful arith_shift(x, k) shares."""
    m = _lmask(ell)
    km = U64((1 << k) - 1)
    xb = (x0 + U64(1 << (ell - 1))) & m
    lw = w[:, 0]
    w0, w1 = cmp_lt(m - xb, x1, ell, lw & U64(0xFFFF), (lw >> U64(16)) & U64(0xFFFF), w[:, 1:4])
    c0, c1 = cmp_lt(km - (xb & km), x1 & km, k, (lw >> U64(32)) & U64(0xFFFF), (lw >> U64(48)) & U64(0xFFFF),
                    w[:, 4:5])
    ones, zeros = np.ones_like(x0), np.zeros_like(x0)
    C0, C1 = mux(c0, c1, ones, zeros, ell, w[:, 5:7])
    W0, W1 = mux(w0, w1, np.full_like(x0, U64(1 << (ell - k))), zeros, ell, w[:, 7:9])
    y0 = ((xb >> U64(k)) + C0 - W0 - U64(1 << (ell - 1 - k))) & m
    y1 = ((x1 >> U64(k)) + C1 - W1) & m
    return y0, y1


def nl_op(op, x0, x1, ell, k=0, d=None, seed=0, stream=0, offset=0):
    """The device op pb_nl_op restated: returns (y0, y1, d_out) (d packed d0 | d1 << 1)."""
    x0 = np.ascontiguousarray(x0, dtype=U64).ravel() & _lmask(ell)
    x1 = np.ascontiguousarray(x1, dtype=U64).ravel() & _lmask(ell)
    n = x0.size
    w = raw_words(seed, stream, n, WORDS[op], offset)
    if d is not None:
        d = np.asarray(d, dtype=U64).ravel()
        dd0, dd1 = d & U64(1), (d >> U64(1)) & U64(1)
    if op == "drelu":
        d0, d1 = drelu(x0, x1, ell, w)
        return None, None, (d0 | (d1 << U64(1))).astype(np.uint8)
    if op == "mux":
        y0, y1 = mux(dd0, dd1, x0, x1, ell, w)
        return y0, y1, None
    if op == "trunc":
        y0, y1 = trunc(x0, x1, ell, k, w)
        return y0, y1, None
    if op == "relu_trunc":
        d0, d1 = drelu(x0, x1, ell, w[:, :W_DRELU])
        u0, u1 = mux(d0, d1, x0, x1, ell, w[:, W_DRELU:W_DRELU + W_MUX])
        y0, y1 = trunc(u0, u1, ell, k, w[:, W_DRELU + W_MUX:])
        return y0, y1, (d0 | (d1 << U64(1))).astype(np.uint8)
    if op == "trunc_mux":
        u0, u1 = trunc(x0, x1, ell, k, w[:, :W_TRUNC])
        y0, y1 = mux(dd0, dd1, u0, u1, ell, w[:, W_TRUNC:])
        return y0, y1, None
    raise ValueError(op)
