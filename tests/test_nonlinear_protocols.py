"""The OT-based non-linear protocols in the oracle
(oracle/nonlinear.py, dealer OT backend SPEC:479): functionality checks per
SPEC's examples and invariants -- every reconstruction equals the plaintext
oracle (DReLU = sign, MUX = d * x, faithful truncation = arith_shift),
including the boundary set {0, +-1 ULP, +-max}."""

import numpy as np
import pytest

from oracle import nonlinear as NL
from oracle import ring as OR

R = OR.RingParams()
M = np.uint64((1 << 59) - 1)


def _share(x, seed):
    r = np.random.default_rng(seed).integers(0, 1 << 59, size=x.shape, dtype=np.uint64)
    return r, (x - r) & M


def _values(n, seed):
    rng = np.random.default_rng(seed)
    x = OR.encode_fixed(rng.uniform(-200, 200, n), R, 50)  # 2f-scale values
    edge = np.array([0, 1, (1 << 59) - 1, 1 << 58, (1 << 58) - 1, (1 << 58) + 1, 2, (1 << 59) - 2], dtype=np.uint64)
    return np.concatenate([x, edge])


def test_secure_compare_examples_and_random():
    n = 10000
    rng = np.random.default_rng(1)
    a = rng.integers(0, 1 << 59, size=n, dtype=np.uint64)
    b = rng.integers(0, 1 << 59, size=n, dtype=np.uint64)
    a[:3] = [3, 7, 0]
    b[:3] = [5, 7, 0]
    w = NL.raw_words(5, 6, n, 4)
    c0, c1 = NL.cmp_lt(a, b, 59, w[:, 0] & np.uint64(0xFFFF), w[:, 0] >> np.uint64(16), w[:, 1:4])
    assert np.array_equal(c0 ^ c1, (a < b).astype(np.uint64))
    assert (c0 ^ c1)[:3].tolist() == [1, 0, 0]


def test_drelu_sign_oracle():  # SPEC:508-511 + invariant "DReLU correctness"
    x = _values(100000, 2)
    x0, x1 = _share(x, 3)
    _, _, d = NL.nl_op("drelu", x0, x1, 59, seed=9, stream=4)
    got = (d & 1) ^ (d >> 1)
    want = (OR.to_signed(x, R) >= 0).astype(np.uint8)
    assert np.array_equal(got, want)
    x = OR.encode_fixed(np.array([5.0, -3.0, 0.0]), R)  # encode(5) -> 1, encode(-3) -> 0, 0 -> 1
    x0, x1 = _share(x, 4)
    _, _, d = NL.nl_op("drelu", x0, x1, 59, seed=1, stream=2)
    assert ((d & 1) ^ (d >> 1)).tolist() == [1, 0, 1]


def test_mux_bit_injection():
    n = 10000
    rng = np.random.default_rng(5)
    x = rng.integers(0, 1 << 59, size=n, dtype=np.uint64)
    dbit = rng.integers(0, 2, size=n, dtype=np.uint8)
    d0 = rng.integers(0, 2, size=n, dtype=np.uint8)
    dp = d0 | ((d0 ^ dbit) << 1)
    x0, x1 = _share(x, 6)
    y0, y1, _ = NL.nl_op("mux", x0, x1, 59, d=dp, seed=3, stream=8)
    assert np.array_equal((y0 + y1) & M, np.where(dbit == 1, x, np.uint64(0)))


@pytest.mark.parametrize("k", [2, 25])
def test_faithful_truncation_exact(k):  # SPEC:542-550, invariant "faithful truncation is exact"
    x = _values(100000, 7)
    x = x[np.abs(OR.to_signed(x, R)) < (1 << 57)]  # precondition |x| < 2^(l-2)
    x0, x1 = _share(x, 8)
    y0, y1, _ = NL.nl_op("trunc", x0, x1, 59, k=k, seed=11, stream=12)
    want = OR.arith_shift(OR.RingTensor(x, 50, R), k).values
    assert np.array_equal((y0 + y1) & M, want)
    x = np.array([60, (1 << 59) - 60], dtype=np.uint64)  # 60 -> 15, -60 -> -15 at shift 2
    x0, x1 = _share(x, 9)
    y0, y1, _ = NL.nl_op("trunc", x0, x1, 59, k=2, seed=1, stream=1)
    assert ((y0 + y1) & M).tolist() == [15, (1 << 59) - 15]


def test_relu_trunc_and_backward_compositions():
    x = _values(20000, 10)
    x = x[np.abs(OR.to_signed(x, R)) < (1 << 57)]
    x0, x1 = _share(x, 11)
    y0, y1, d = NL.nl_op("relu_trunc", x0, x1, 59, k=25, seed=2, stream=3)
    relu = np.where(OR.to_signed(x, R) >= 0, x, np.uint64(0))
    assert np.array_equal((y0 + y1) & M, OR.arith_shift(OR.RingTensor(relu, 50, R), 25).values)
    g = np.resize(_values(20000, 12), x.size)
    g = np.where(np.abs(OR.to_signed(g, R)) < (1 << 57), g, np.uint64(0))
    g0, g1 = _share(g, 13)
    z0, z1, _ = NL.nl_op("trunc_mux", g0, g1, 59, k=25, d=d, seed=2, stream=4)
    dbit = (d & 1) ^ (d >> 1)
    want = np.where(dbit == 1, OR.arith_shift(OR.RingTensor(g, 50, R), 25).values, np.uint64(0))
    assert np.array_equal((z0 + z1) & M, want)
