"""Conv-layer parity on the B200: the local ring
conv kernels equal the oracle's conv2d_wrap compositions; the DO's decrypted
shares of the three conv protocols equal the oracle's under the same seeds;
private CNN training steps reveal exactly the gradients of
``reference_train_step`` (σ = 0, faithful truncation) -- at the full
MNIST-CNN and CIFAR-CNN sizes, batch 64."""

import copy

import numpy as np
import pytest

from oracle import bfv as OB
from oracle import convops as CO
from oracle import nn as ON
from oracle import protocols as OPR
from oracle import ring as OR
from oracle.params import make_params

pytestmark = pytest.mark.gpu

RING = OR.RingParams()
CASES = [  # B, c_i, c_o, H, W, s, pad, stride
    (2, 1, 3, 6, 6, 3, 1, 2), (2, 2, 3, 5, 5, 3, 1, 1), (3, 1, 2, 8, 8, 5, 2, 2), (2, 3, 2, 4, 4, 1, 0, 1),
    (4, 1, 5, 28, 28, 5, 2, 2), (2, 5, 5, 14, 14, 5, 2, 1), (2, 3, 8, 32, 32, 5, 2, 1), (2, 2, 2, 9, 9, 3, 1, 3),
    (2, 4, 3, 8, 8, 4, 1, 2),
]


@pytest.fixture(scope="module")
def env():
    from paper_2403_11166_b200 import bfv, ring
    from paper_2403_11166_b200.linear_protocols import Session
    from paper_2403_11166_b200.params import BfvParams

    op = make_params(8192, 7)
    ar = OB.Arith(op)
    okp = OB.keygen(op, OR.SeededRng(1, 0), ar)
    pp = BfvParams()
    pkp = bfv.keygen(pp, ring.SeededRng(1, 0))
    pr = ring.RingParams()
    return dict(octx=OPR.Ctx(op, RING, okp, seed=77, ar=ar), sess=Session(pp, pr, pkp, seed=77), pr=pr)


def _dev(a):
    from paper_2403_11166_b200 import _dev as D

    return D.u64_to_device(a)


def _np(t):
    from paper_2403_11166_b200 import _dev as D

    return D.to_numpy_u64(t).copy()


@pytest.mark.parametrize("case", CASES)
def test_ring_conv_kernels_bit_exact(case):
    from paper_2403_11166_b200 import _lib
    from paper_2403_11166_b200.linear_protocols import _ring_conv

    B, ci, co, H, W, s, p, st = case
    rng = np.random.default_rng(3)
    x = rng.integers(0, 1 << 59, size=(B, ci, H, W), dtype=np.uint64)
    w = rng.integers(0, 1 << 59, size=(co, ci, s, s), dtype=np.uint64)
    y = CO.conv_fwd(x, w, p, st) & RING.mask
    gy = rng.integers(0, 1 << 59, size=y.shape, dtype=np.uint64)
    args = (B, ci, co, H, W, s, p, st, 59)
    assert np.array_equal(_np(_ring_conv(_lib.CONV_FWD, _dev(x), _dev(w), *args, y.shape)), y)
    gx = CO.conv_bwdx(gy, w, H, W, p, st) & RING.mask
    assert np.array_equal(_np(_ring_conv(_lib.CONV_BWDX, _dev(gy), _dev(w), *args, gx.shape)), gx)
    gw = CO.conv_gradw(x, gy, s, p, st) & RING.mask
    assert np.array_equal(_np(_ring_conv(_lib.CONV_GRADW, _dev(x), _dev(gy), *args, gw.shape)), gw)


def test_pool_kernels_bit_exact():
    from paper_2403_11166_b200 import _lib
    from paper_2403_11166_b200.nonlinear import _pool_local

    x = np.random.default_rng(4).integers(0, 1 << 59, size=(3, 4, 6, 8), dtype=np.uint64)
    assert np.array_equal(_np(_pool_local(_lib.POOL_SUM, _dev(x), (3, 4), 59)), CO.pool_sum(x) & RING.mask)
    assert np.array_equal(_np(_pool_local(_lib.POOL_REPLICATE, _dev(x), (12, 16), 59)), CO.pool_replicate(x))


@pytest.mark.parametrize("shape", [(64, 64, 32, 32), (64, 128, 8, 8), (3, 5, 7, 9), (1, 1, 1, 1), (2, 3, 1, 1),
                                   (5, 2, 16, 16), (0, 4, 3, 3), (7, 1, 300, 1)])
def test_chansum_bit_exact(shape):
    """pb_ring_chansum (conv bias gradient) vs the numpy sum over
    (b, h, w) mod 2^59, straight from NCHW -- every split of the range."""
    from paper_2403_11166_b200 import _dev as D
    from paper_2403_11166_b200 import _lib

    B, c, h, w = shape
    x = np.random.default_rng(B * 7 + c).integers(0, 1 << 64, size=shape, dtype=np.uint64)
    want = x.reshape(B, c, h * w).transpose(1, 0, 2).reshape(c, -1).sum(axis=1, dtype=np.uint64) & RING.mask
    out = D.empty_u64(c)
    xd = _dev(x)
    _lib.call("pb_ring_chansum", D.ptr(xd), B, c, h * w, 59, D.ptr(out), D.stream())
    assert np.array_equal(_np(out), want)


def _shares(pr, mo, do, scale):
    from paper_2403_11166_b200.ring import DO, MO, RingTensor, ShareTensor

    return (ShareTensor(MO, RingTensor(mo, scale, pr)), ShareTensor(DO, RingTensor(do, scale, pr)))


def _rand_shares(seed, shape, amp=2.0):
    x = OR.encode_fixed(np.random.default_rng(seed).uniform(-amp, amp, size=shape), RING)
    mo = OR.SeededRng(seed, 1).uniform_ring(shape, RING)
    return x, mo, (x - mo) & RING.mask


@pytest.mark.parametrize("case", [CASES[0], CASES[2], CASES[4], CASES[5], CASES[7]])
def test_conv_protocol_shares_bit_exact(env, case):
    """conv_forward / conv_backward_input / conv_grad_weight: DO shares (and the
    MO's) equal the oracle's; reconstructions equal the plaintext operators."""
    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200.ring import RingTensor

    B, ci, co, H, W, s, p, st = case
    pr, sess, octx = env["pr"], env["sess"], env["octx"]
    Wt = OR.encode_fixed(np.random.default_rng(1).uniform(-0.3, 0.3, size=(co, ci, s, s)), RING)
    b = OR.encode_fixed(np.random.default_rng(2).uniform(-0.3, 0.3, size=co), RING, 50)
    x, x_mo, x_do = _rand_shares(3, (B, ci, H, W))
    oh, ow = CO.conv_out_hw(H, W, s, p, st)
    gy, gy_mo, gy_do = _rand_shares(5, (B, co, oh, ow), 1.0)
    WR, bR = RingTensor(Wt, 25, pr), RingTensor(b, 50, pr)
    for layer, zero in ((1, False), (0, True)):
        xm = np.zeros_like(x) if zero else x_mo
        xd = x if zero else x_do
        o_mo, o_do = OPR.conv_forward(octx, layer, Wt, b, xm, xd, p, st, mo_x_zero=zero)
        y_mo, y_do = LP.conv_forward(sess, layer, WR, bR, *_shares(pr, xm, xd, 25), p, st, mo_x_zero=zero)
        assert np.array_equal(y_do.value.numpy(), o_do) and np.array_equal(y_mo.value.numpy(), o_mo)
        want = (CO.conv_fwd(x, Wt, p, st) + b[None, :, None, None]) & RING.mask
        assert np.array_equal((o_mo + o_do) & RING.mask, want)
    g_mo, g_do = OPR.conv_backward_input(octx, 2, Wt, gy_mo, gy_do, H, W, p, st)
    a_mo, a_do = LP.conv_backward_input(sess, 2, WR, *_shares(pr, gy_mo, gy_do, 25), H, W, p, st)
    assert np.array_equal(a_do.value.numpy(), g_do) and np.array_equal(a_mo.value.numpy(), g_mo)
    assert np.array_equal((g_mo + g_do) & RING.mask, CO.conv_bwdx(gy, Wt, H, W, p, st) & RING.mask)
    ow_ = OPR.conv_grad_weight(octx, 3, x_mo, x_do, gy_mo, gy_do, s, p, st)
    pw_ = LP.conv_grad_weight(sess, 3, *_shares(pr, x_mo, x_do, 25), *_shares(pr, gy_mo, gy_do, 25), s, p, st)
    assert np.array_equal(pw_.numpy(), ow_)
    assert np.array_equal(ow_, CO.conv_gradw(x, gy, s, p, st) & RING.mask)
    ob = OPR.reveal_grad_bias_conv(octx, 3, gy_mo, gy_do)
    pb = LP.reveal_grad_bias_conv(sess, 3, *_shares(pr, gy_mo, gy_do, 25))
    assert np.array_equal(pb.numpy(), ob)


def _private_vs_reference(env, arch, B, steps=1, seed=3):
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.ring import RingTensor, encode_fixed

    pr = env["pr"]
    om = ON.Model(arch, RING, seed=seed)
    pm = PN.Model(arch, pr, seed=seed)
    xo, labels = ON.synthetic_images(5, B, om.in_shape, RING)
    xh, plabels = PN.synthetic_images(5, B, pm.in_shape, pr)
    assert np.array_equal(labels, plabels)
    xp = RingTensor(encode_fixed(xh, pr), 25, pr, _canonical=True)
    assert np.array_equal(xp.numpy(), xo)
    for step in range(steps):
        env["sess"].reseed(2000 + step)
        ref_loss, ref_gw, ref_gb = ON.reference_train_step(om, xo, labels)
        loss, gw, gb = PN.private_train_step(env["sess"], pm, xp, plabels)
        assert loss == ref_loss
        for l in range(om.n_layers):
            assert np.array_equal(gw[l].numpy(), ref_gw[l]), (step, l)
            assert np.array_equal(gb[l].numpy(), ref_gb[l]), (step, l)
            assert np.array_equal(pm.w[l].cpu().numpy(), om.w[l])
            assert np.array_equal(pm.W[l].numpy(), om.W(l))


SMALL_CNN = ((2, 8, 8), [("conv", 2, 3, 3, 1, 1), ("pool",), ("conv", 3, 4, 3, 1, 2), ("flatten",),
                         ("fc", 16, 6), ("fc", 6, 10)])


def test_small_cnn_step_matches_reference_engine(env):
    _private_vs_reference(env, SMALL_CNN, 3, steps=2)


@pytest.mark.parametrize("name", ["mnist_cnn", "mnist_cnn2"])
def test_mnist_cnn_step_b64_matches_reference_engine(env, name):
    _private_vs_reference(env, name, 64, steps=2)


def test_cifar_cnn_step_b64_matches_reference_engine(env):
    _private_vs_reference(env, "cifar_cnn", 64, steps=1)


def test_small_cnn_shares_match_oracle_private_step(env):
    """Share level: every layer's DO / MO output shares equal the oracle's private step."""
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.ring import RingTensor, encode_fixed

    pr = env["pr"]
    om, pm = ON.Model(SMALL_CNN, RING, seed=9), PN.Model(SMALL_CNN, pr, seed=9)
    xo, labels = ON.synthetic_images(11, 2, om.in_shape, RING)
    xh, _ = PN.synthetic_images(11, 2, pm.in_shape, pr)
    env["octx"].seed = 4243
    env["sess"].reseed(4243)
    ot, pt = [], []
    ON.private_train_step(env["octx"], copy.deepcopy(om), xo, labels, trace=ot)
    PN.private_train_step(env["sess"], pm, RingTensor(encode_fixed(xh, pr), 25, pr, _canonical=True), labels,
                          trace=pt)
    env["octx"].seed = 77
    assert len(ot) == len(pt) == om.n_layers
    for (l1, y1, gb1, gw1), (l2, y2, gb2, gw2) in zip(ot, pt):
        assert l1 == l2
        assert np.array_equal(y2[1].value.numpy(), y1[1]) and np.array_equal(y2[0].value.numpy(), y1[0])
        assert np.array_equal(gw2.numpy(), gw1) and np.array_equal(gb2.numpy(), gb1)
