"""DP hook of Alg. 2 and the bias reveal in the oracle:
sample_dp_noise statistics, the hook's placement, and the
private step with sigma > 0 == the reference engine with the same DP draws
("same DP hook")."""

import copy

import numpy as np

from oracle import nn as ON
from oracle import protocols as PR
from oracle import ring as OR


def test_sample_dp_noise_zero_when_sigma_zero():
    dp = PR.DpConfig(sigma=0.0, C=8.0, B=64, enabled=True)
    assert not PR.sample_dp_noise((5, 7), dp, OR.SeededRng(1, 2)).any()
    assert PR.dp_noise(1, 0, PR.OP_GRAD_W, (3, 4), 50, PR.DpConfig(), OR.RingParams()) is None


def test_sample_dp_noise_statistics():  # SPEC:354-355 (10^6 draws)
    dp = PR.DpConfig(sigma=0.01, C=8.0, B=64, enabled=True)
    e = PR.sample_dp_noise((1_000_000,), dp, OR.SeededRng(7, 3))
    want = dp.sigma * dp.C / np.sqrt(dp.B)  # = 0.01
    assert abs(e.std() - want) <= 0.05 * want
    assert abs(e.mean()) <= 4 * want / np.sqrt(e.size)


def test_reveal_grad_bias_adds_encoded_noise():
    R = OR.RingParams()
    rng = np.random.default_rng(0)
    gy_mo = rng.integers(0, 1 << 59, size=(4, 16), dtype=np.uint64)
    gy_do = rng.integers(0, 1 << 59, size=(4, 16), dtype=np.uint64)
    dp = PR.DpConfig(sigma=0.5, C=1.0, B=16, enabled=True)
    e = PR.dp_noise(9, 0, PR.OP_GRAD_B, (4,), R.f, dp, R)
    got = PR.reveal_grad_bias(type("C", (), {"ring": R})(), 0, gy_mo, gy_do, e=e)
    base = (gy_mo.sum(axis=1, dtype=np.uint64) + gy_do.sum(axis=1, dtype=np.uint64)) & R.mask
    assert np.array_equal(got, (base + e) & R.mask)
    # the noise decodes to N(0, (sigma C)^2 / B) draws of the documented stream
    draw = OR.SeededRng(9, PR.stream_id(0, PR.OP_GRAD_B, PR.P_DP)).normal((4,), 0.5 / 4)
    assert np.array_equal(OR.decode_fixed(e, R, R.f), np.floor(draw * 2.0 ** R.f) / 2.0 ** R.f)


def test_private_step_with_dp_equals_reference_engine():
    """sigma > 0: the private MLP step's revealed gradients and updated weights
    equal the reference engine's under the same DP streams."""
    from oracle import bfv as OB
    from oracle.params import make_params

    R = OR.RingParams()
    p = make_params(8192, 7)
    ar = OB.Arith(p)
    ctx = PR.Ctx(p, R, OB.keygen(p, OR.SeededRng(1, 0), ar), seed=11, ar=ar)
    m1 = ON.Model([784, 8, 10], R, seed=3)
    m2 = copy.deepcopy(m1)
    x, labels = ON.synthetic_mnist(4, 4, R)
    dp = PR.DpConfig(sigma=1.0, C=4.0, B=4, enabled=True)
    l1, gw1, gb1 = ON.reference_train_step(m1, x, labels, dp=dp, dp_seed=11)
    l2, gw2, gb2 = ON.private_train_step(ctx, m2, x, labels, dp=dp)
    assert l1 == l2
    m3 = ON.Model([784, 8, 10], R, seed=3)
    _, gw3, gb3 = ON.reference_train_step(m3, x, labels)  # sigma = 0
    for l in range(m1.n_layers):
        assert np.array_equal(gw1[l], gw2[l]) and np.array_equal(gb1[l], gb2[l]), l
        assert np.array_equal(m1.w[l], m2.w[l])
        assert not np.array_equal(gw1[l], gw3[l])  # the noise is really there
