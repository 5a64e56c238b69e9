"""Protocol-level parity (SURVEY §8c ii/iii): the DO's decrypted shares of every
linear-layer procedure are bit-identical to the CPU oracle's under the same
seeds, reconstructions equal the fixed-point reference, and a private
training step reveals exactly the gradients of ``reference_train_step``."""

import copy

import numpy as np
import pytest

from oracle import bfv as OB
from oracle import kernels as OK
from oracle import nn as ON
from oracle import protocols as OPR
from oracle import ring as OR
from oracle.params import make_params

pytestmark = pytest.mark.gpu

RING = OR.RingParams()


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


def _shares(pr, mo, do, scale):
    from paper_2403_11166_b200.ring import DO, MO, RingTensor, ShareTensor

    return (ShareTensor(MO, RingTensor(mo, scale, pr)), ShareTensor(DO, RingTensor(do, scale, pr)))


def _rand_shares(seed, shape, scale_val=2.0):
    x = OR.encode_fixed(np.random.default_rng(seed).uniform(-scale_val, scale_val, size=shape), RING)
    mo = OR.SeededRng(seed, 1).uniform_ring(shape, RING)
    return x, mo, (x - mo) & RING.mask


@pytest.mark.parametrize("n_i,n_o,B,zero", [(784, 128, 64, True), (128, 128, 64, False), (20, 9, 5, False)])
def test_linear_forward_shares_bit_exact(env, n_i, n_o, B, zero):
    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200.ring import RingTensor

    pr = env["pr"]
    W = OR.encode_fixed(np.random.default_rng(1).uniform(-0.1, 0.1, size=(n_o, n_i)), RING)
    b = OR.encode_fixed(np.random.default_rng(2).uniform(-0.1, 0.1, size=n_o), RING, 50)
    x, x_mo, x_do = _rand_shares(3, (n_i, B))
    if zero:
        x_mo, x_do = np.zeros_like(x), x
    o_mo, o_do = OPR.linear_forward(env["octx"], 0, W, b, x_mo, x_do, mo_x_zero=zero)
    y_mo, y_do = LP.linear_forward(env["sess"], 0, RingTensor(W, 25, pr), RingTensor(b, 50, pr),
                                   *_shares(pr, x_mo, x_do, 25), mo_x_zero=zero)
    assert np.array_equal(y_do.value.numpy(), o_do)
    assert np.array_equal(y_mo.value.numpy(), o_mo)
    rec = (y_mo.value + y_do.value).numpy()
    assert np.array_equal(rec, (OK.matmul_wrap(W, x) + b[:, None]) & RING.mask)


def test_backward_input_and_grad_weight_bit_exact(env):
    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200.ring import RingTensor

    pr = env["pr"]
    n_i, n_o, B = 128, 10, 64
    W = OR.encode_fixed(np.random.default_rng(4).uniform(-0.1, 0.1, size=(n_o, n_i)), RING)
    x, x_mo, x_do = _rand_shares(5, (n_i, B))
    gy, g_mo, g_do = _rand_shares(6, (n_o, B), 0.01)
    o_mo, o_do = OPR.linear_backward_input(env["octx"], 2, W, g_mo, g_do)
    p_mo, p_do = LP.linear_backward_input(env["sess"], 2, RingTensor(W, 25, pr), *_shares(pr, g_mo, g_do, 25))
    assert np.array_equal(p_do.value.numpy(), o_do) and np.array_equal(p_mo.value.numpy(), o_mo)
    assert np.array_equal((p_mo.value + p_do.value).numpy(), OK.matmul_wrap(np.ascontiguousarray(W.T), gy) & RING.mask)
    ogw = OPR.grad_weight(env["octx"], 2, x_mo, x_do, g_mo, g_do)
    pgw = LP.grad_weight(env["sess"], 2, *_shares(pr, x_mo, x_do, 25), *_shares(pr, g_mo, g_do, 25))
    assert np.array_equal(pgw.numpy(), ogw)
    assert np.array_equal(pgw.numpy(), OK.matmul_wrap(gy, np.ascontiguousarray(x.T)) & RING.mask)
    ogb = OPR.reveal_grad_bias(env["octx"], 2, g_mo, g_do)
    pgb = LP.reveal_grad_bias(env["sess"], 2, *_shares(pr, g_mo, g_do, 25))
    assert np.array_equal(pgb.numpy(), ogb) and np.array_equal(ogb, gy.sum(axis=1, dtype=np.uint64) & RING.mask)


def test_spec_linear_examples(env):
    """SPEC:318-319, 327-328, 345-346."""
    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200.ring import RingTensor

    pr = env["pr"]
    sess = env["sess"]
    I2 = OR.encode_fixed(np.eye(2), RING)
    b = OR.encode_fixed([1.0, 1.0], RING, 50)
    x = OR.encode_fixed(np.array([[2.0], [3.0]]), RING)
    xm = OR.SeededRng(3, 3).uniform_ring((2, 1), RING)
    y_mo, y_do = LP.linear_forward(sess, 0, RingTensor(I2, 25, pr), RingTensor(b, 50, pr),
                                   *_shares(pr, xm, (x - xm) & RING.mask, 25))
    assert OR.decode_fixed((y_mo.value + y_do.value).numpy(), RING, 50).ravel().tolist() == [3.0, 4.0]
    W = OR.encode_fixed(np.array([[1.0, 2, 3], [4, 5, 6]]), RING)
    gy = OR.encode_fixed(np.array([[1.0], [0.0]]), RING)
    g_mo, g_do = LP.linear_backward_input(sess, 1, RingTensor(W, 25, pr), *_shares(pr, np.zeros_like(gy), gy, 25))
    assert OR.decode_fixed((g_mo.value + g_do.value).numpy(), RING, 50).ravel().tolist() == [1.0, 2.0, 3.0]
    X = OR.encode_fixed(np.array([[1.0], [2.0]]), RING)
    G = OR.encode_fixed(np.array([[3.0]]), RING)
    gw = LP.grad_weight(sess, 1, *_shares(pr, np.zeros_like(X), X, 25), *_shares(pr, np.zeros_like(G), G, 25))
    assert OR.decode_fixed(gw.numpy(), RING, 50).ravel().tolist() == [3.0, 6.0]


@pytest.mark.parametrize("sizes,B", [([784, 32, 10], 8), ([784, 128, 128, 10], 64)])
def test_private_step_matches_reference_engine(env, sizes, B):
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.ring import RingTensor, encode_fixed

    pr = env["pr"]
    om = ON.Model(sizes, RING, seed=3)
    pm = PN.Model(sizes, pr, seed=3)
    xo, labels = ON.synthetic_mnist(5, B, RING)
    xh, plabels = PN.synthetic_mnist(5, B, pr)
    assert np.array_equal(labels, plabels)
    xp = RingTensor(encode_fixed(xh, pr), 25, pr, _canonical=True)
    assert np.array_equal(xp.numpy(), xo)
    for step in range(2):
        env["sess"].reseed(1000 + step)
        ref_loss, ref_gw, ref_gb = ON.reference_train_step(om, xo, labels)
        loss, gw, gb = PN.private_train_step(env["sess"], pm, xp, plabels)
        assert loss == ref_loss
        for l in range(len(sizes) - 1):
            assert np.array_equal(gw[l].numpy(), ref_gw[l]), (step, l)
            assert np.array_equal(gb[l].numpy(), ref_gb[l]), (step, l)
            assert np.array_equal(pm.w[l].cpu().numpy(), om.w[l])
            assert np.array_equal(pm.W[l].numpy(), om.W(l))


def test_private_step_shares_match_oracle_private_step(env):
    """Beyond revealed values: every DO share of the forward pass equals the oracle's."""
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.ring import RingTensor, encode_fixed

    pr = env["pr"]
    sizes, B = [784, 16, 10], 4
    om, pm = ON.Model(sizes, RING, seed=9), PN.Model(sizes, pr, seed=9)
    xo, labels = ON.synthetic_mnist(11, B, RING)
    xh, _ = PN.synthetic_mnist(11, B, pr)
    env["octx"].seed = 4242
    env["sess"].reseed(4242)
    ot, pt = [], []
    ON.private_train_step(env["octx"], om, xo, labels, trace=ot)
    PN.private_train_step(env["sess"], pm, RingTensor(encode_fixed(xh, pr), 25, pr, _canonical=True), labels, trace=pt)
    env["octx"].seed = 77
    for (l1, y1, gb1, gw1), (l2, y2, gb2, gw2) in zip(ot, pt):
        assert l1 == l2
        assert np.array_equal(y2[1].value.numpy(), y1[1]) and np.array_equal(y2[0].value.numpy(), y1[0])
        assert np.array_equal(gw2.numpy(), gw1) and np.array_equal(gb2.numpy(), gb1)
