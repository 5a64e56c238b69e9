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


def test_linear_forward_with_encryption_predraw_bit_exact(env):
    """Inside a phase (Session.begin_phase) the DO's encryption is split: the
    message-independent half pre-drawn on its own stream, c0 += NTT(e + Delta
    m) on the critical path.  The ciphertexts are fresh encryptions; the
    decrypted shares stay bit-identical to the oracle's."""
    import torch

    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200.ring import RingTensor

    pr, sess = env["pr"], env["sess"]
    n_i, n_o, B = 128, 128, 64
    W = OR.encode_fixed(np.random.default_rng(11).uniform(-0.1, 0.1, size=(n_o, n_i)), RING)
    b = OR.encode_fixed(np.random.default_rng(12).uniform(-0.1, 0.1, size=n_o), RING, 50)
    x, x_mo, x_do = _rand_shares(13, (n_i, B))
    o_mo, o_do = OPR.linear_forward(env["octx"], 1, W, b, x_mo, x_do)
    sess._predraw_bufs.clear()
    sess.begin_phase()
    try:
        y_mo, y_do = LP.linear_forward(sess, 1, RingTensor(W, 25, pr), RingTensor(b, 50, pr),
                                       *_shares(pr, x_mo, x_do, 25))
    finally:
        sess.join_side()
    torch.cuda.synchronize()
    assert (1, LP.OP_FWD, "A_ct") in sess._predraw_bufs  # the split path ran
    assert np.array_equal(y_do.value.numpy(), o_do)
    assert np.array_equal(y_mo.value.numpy(), o_mo)


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


# ----------------------------------------------------------- DP hook ---
# the DO's perturbation e of the bias reveal and of Alg. 2.

def test_dp_noise_statistics_on_device_path(env):
    """sigma=0.01, C=8, B=64: the encoded noise the engine adds decodes to
    draws with std within 5 % of sigma C / sqrt(B) and a mean within 4
    standard errors of 0, and sigma=0 adds nothing."""
    from paper_2403_11166_b200 import linear_protocols as LP

    sess = env["sess"]
    try:
        sess.dp = LP.DpConfig(sigma=0.01, C=8.0, B=64, enabled=True)
        e = LP.dp_noise(sess, 0, LP.OP_GRAD_W, (1000, 1000), 50)
        v = OR.decode_fixed(e.cpu().numpy().view(np.uint64), RING, 50)
        assert abs(v.std() - 0.01) <= 0.05 * 0.01 and abs(v.mean()) <= 4 * 0.01 / 1000
        sess.dp = LP.DpConfig(sigma=0.0, C=8.0, B=64, enabled=True)
        assert not LP.dp_noise(sess, 0, LP.OP_GRAD_W, (10, 10), 50).cpu().numpy().any()
    finally:
        sess.dp = None


@pytest.mark.parametrize("sigma", [0.01, 0.5])
def test_reveal_grad_bias_and_grad_weight_with_given_e_equal_oracle(env, sigma):
    """With a given e both reveals equal the oracle's bit for bit."""
    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200.ring import RingTensor

    pr, sess, octx = env["pr"], env["sess"], env["octx"]
    n_i, n_o, B = 96, 24, 16
    x, x_mo, x_do = _rand_shares(21, (n_i, B))
    g, g_mo, g_do = _rand_shares(22, (n_o, B), 0.1)
    dp = OPR.DpConfig(sigma=sigma, C=4.0, B=B, enabled=True)
    eb = OPR.dp_noise(5, 1, OPR.OP_GRAD_B, (n_o,), 25, dp, RING)
    ew = OPR.dp_noise(5, 1, OPR.OP_GRAD_W, (n_o, n_i), 50, dp, RING)
    sess.reseed(77)
    octx.seed = 77
    gb = LP.reveal_grad_bias(sess, 1, *_shares(pr, g_mo, g_do, 25), e=RingTensor(eb, 25, pr).values)
    assert np.array_equal(gb.numpy(), OPR.reveal_grad_bias(octx, 1, g_mo, g_do, e=eb))
    gw = LP.grad_weight(sess, 1, *_shares(pr, x_mo, x_do, 25), *_shares(pr, g_mo, g_do, 25),
                        e=RingTensor(ew, 50, pr).values)
    want = OPR.grad_weight(octx, 1, x_mo, x_do, g_mo, g_do, e=ew)
    assert np.array_equal(gw.numpy(), want)
    # and the perturbation is exactly e on top of the sigma = 0 reveal
    plain = (OK.matmul_wrap(g, np.ascontiguousarray(x.T)) + ew) & RING.mask
    assert np.array_equal(gw.numpy(), plain)


def test_private_step_with_dp_matches_reference_engine(env):
    """sigma > 0: revealed gradients, master weights and re-quantised weights of
    a private MLP step equal the reference engine's with the same DP streams."""
    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.ring import RingTensor, encode_fixed

    pr, sess = env["pr"], env["sess"]
    sizes, B = [784, 32, 10], 8
    om, pm = ON.Model(sizes, RING, seed=3), PN.Model(sizes, pr, seed=3)
    xo, labels = ON.synthetic_mnist(5, B, RING)
    xh, _ = PN.synthetic_mnist(5, B, pr)
    xp = RingTensor(encode_fixed(xh, pr), 25, pr, _canonical=True)
    dp = OPR.DpConfig(sigma=1.0, C=2.0, B=B, enabled=True)
    try:
        sess.dp = LP.DpConfig(sigma=1.0, C=2.0, B=B, enabled=True)
        for step in range(2):
            sess.reseed(3000 + step)
            ref_loss, ref_gw, ref_gb = ON.reference_train_step(om, xo, labels, dp=dp, dp_seed=3000 + step)
            loss, gw, gb = PN.private_train_step(sess, pm, xp, labels)
            assert loss == ref_loss
            for l in range(len(sizes) - 1):
                assert np.array_equal(gw[l].numpy(), ref_gw[l]) and np.array_equal(gb[l].numpy(), ref_gb[l])
                assert np.array_equal(pm.w[l].cpu().numpy(), om.w[l])
                assert np.array_equal(pm.W[l].numpy(), om.W(l))
        with pytest.raises(Exception):
            PN.GraphStep(sess, pm, xp)  # DP steps are eager-only (per-step host draw)
    finally:
        sess.dp = None


# ------------------------------------------------- ring API on the device ---
# R:140-145 (__neg__, scalar_mul) and R:185-198 (decode_fixed, to_signed).

def test_ring_neg_scalar_mul_decode_to_signed_match_reference():
    from paper_2403_11166_b200 import ring as PRG

    pr = PRG.RingParams()
    rng = np.random.default_rng(5)
    edge = np.array([0, 1, (1 << 58) - 1, 1 << 58, (1 << 58) + 1, (1 << 59) - 1], dtype=np.uint64)
    v = np.concatenate([edge, rng.integers(0, 1 << 59, size=4096, dtype=np.uint64)])
    ot = OR.RingTensor(v, 25, RING)
    dt = PRG.RingTensor(v, 25, pr)
    assert np.array_equal((-dt).numpy(), (-ot).values)
    for k in (0, 1, 3, -7, (1 << 59) - 1, 1 << 40, 123456789):
        assert np.array_equal(dt.scalar_mul(k).numpy(), ot.scalar_mul(k).values), k
    assert np.array_equal(PRG.to_signed(dt.values, pr).cpu().numpy(), OR.to_signed(v, RING))
    for scale in (25, 50, 0):
        got = PRG.decode_fixed(dt.values, pr, scale).cpu().numpy()
        assert np.array_equal(got, OR.decode_fixed(v, RING, scale)), scale
    # the reference's own outputs on edge residues (tests/golden/ring.npz, generated from R)
    g = dict(np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "ring.npz")))
    e = PRG.RingTensor(g["edge_in"], 25, pr)
    assert np.array_equal((-e).numpy(), g["edge_neg"])
    for k, want in zip(g["edge_smul_ks"], g["edge_smul"]):
        assert np.array_equal(e.scalar_mul(int(k)).numpy(), want)
    assert np.array_equal(PRG.to_signed(e.values, pr).cpu().numpy(), g["edge_signed"])
    assert np.array_equal(PRG.decode_fixed(e.values, pr, 50).cpu().numpy(), g["edge_dec_f50"])
    assert np.array_equal(PRG.decode_fixed(g["enc_f25"], pr).cpu().numpy(), g["dec_f25"])
    # round trip through the device encoder, including the range edge
    x = np.array([0.0, -1.0, 2.5, -(2.0 ** 33) + 2.0 ** -18, 2.0 ** 33 - 2.0 ** -18, 1e-9, -1e-9])
    enc = PRG.encode_fixed(x, pr)
    assert np.array_equal(enc.cpu().numpy().view(np.uint64), OR.encode_fixed(x, RING))
    assert np.array_equal(PRG.decode_fixed(enc, pr).cpu().numpy(), OR.decode_fixed(OR.encode_fixed(x, RING), RING))
