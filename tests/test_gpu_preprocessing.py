"""Pencil+ preprocessing on the B200: the device banks
(masks and the DO's decrypted u'_i o v'_j - s_ij) and the online shares are
bit-identical to the CPU oracle's; a prep-mode private training step
(Alg. 4) reveals exactly the reference engine's gradients at full MNIST-MLP
and MNIST-CNN size; the online phase sends no ciphertext."""

import copy

import numpy as np
import pytest

from oracle import bfv as OB
from oracle import nn as ON
from oracle import preprocessing as OPP
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
    pr = ring.RingParams()
    sess = Session(pp, pr, bfv.keygen(pp, ring.SeededRng(1, 0)), seed=61)
    return dict(octx=OPR.Ctx(op, RING, okp, seed=61, ar=ar), sess=sess, pr=pr)


@pytest.mark.parametrize("spec,hw", [(("fc", 40, 9), None), (("conv", 2, 3, 3, 1, 2), (6, 6)),
                                     (("conv", 3, 4, 5, 2, 1), (8, 8))])
def test_banks_and_online_shares_bit_exact(env, spec, hw):
    from paper_2403_11166_b200 import _dev
    from paper_2403_11166_b200 import preprocessing as PP

    for op in range(4):
        o_opd = OPP.Operator(spec, op, 4, hw)
        p_opd = PP.Operator(spec, op, 4, hw)
        ob = OPP.prep_operator(env["octx"], 2, o_opd, 3, bank_seed=7)
        pb = PP.prep_operator(env["sess"], 2, p_opd, 3, bank_seed=7)
        for name in ("u", "v", "s", "d"):
            assert np.array_equal(_dev.to_numpy_u64(getattr(pb, name)), getattr(ob, name)), (op, name)
        rng = np.random.default_rng(op)
        u = rng.integers(0, 1 << 59, size=o_opd.u_shape, dtype=np.uint64)
        v = rng.integers(0, 1 << 59, size=o_opd.v_shape, dtype=np.uint64)
        env["octx"].seed = 900 + op
        env["sess"].reseed(900 + op)
        omo, odo = OPP.online_shared_product(env["octx"], 2, ob, u, v)
        pmo, pdo = PP.online_shared_product(env["sess"], 2, pb, _dev.u64_to_device(u), _dev.u64_to_device(v))
        assert np.array_equal(_dev.to_numpy_u64(pmo), omo) and np.array_equal(_dev.to_numpy_u64(pdo), odo), op
        assert np.array_equal((omo + odo) & RING.mask, o_opd.apply(u, v) & RING.mask)


@pytest.mark.parametrize("name,B,m", [("mnist_mlp", 64, 8), ("mnist_cnn", 64, 4)])
def test_prep_step_matches_reference_engine(env, name, B, m):
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200 import preprocessing as PP
    from paper_2403_11166_b200.linear_protocols import Channel
    from paper_2403_11166_b200.ring import RingTensor, encode_fixed

    pr, sess = env["pr"], env["sess"]
    om = ON.Model(name, RING, seed=3)
    pm = PN.Model(name, pr, seed=3)
    if len(om.in_shape) == 1:
        xo, labels = ON.synthetic_mnist(5, B, RING)
        xh, _ = PN.synthetic_mnist(5, B, pr)
    else:
        xo, labels = ON.synthetic_images(5, B, om.in_shape, RING)
        xh, _ = PN.synthetic_images(5, B, pm.in_shape, pr)
    state = PP.PrepState(sess, pm, B, m=m, bank_seed=11)
    sess.channel = Channel()  # census of the online phase only
    xp = RingTensor(encode_fixed(xh, pr), 25, pr, _canonical=True)
    for step in range(2):
        sess.reseed(3000 + step)
        ref_loss, ref_gw, ref_gb = ON.reference_train_step(om, xo, labels)
        loss, gw, gb = PN.private_train_step(sess, pm, xp, labels, prep=state)
        assert loss == ref_loss
        for l in range(om.n_layers):
            assert np.array_equal(gw[l].numpy(), ref_gw[l]) and np.array_equal(gb[l].numpy(), ref_gb[l]), (step, l)
            assert np.array_equal(pm.W[l].numpy(), om.W(l))
    census = sess.channel.census
    assert not any(t in census for t in (0x10, 0x11, 0x20, 0x21, 0x40, 0x41)), census  # no ciphertext frames online
    assert 0x42 in census and 0x43 in census


@pytest.mark.parametrize("n,ma,mb,shift,sub", [(4096, 8, 8, 0, 1), (4097, 8, 8, 0, 0), (1000, 3, 5, 1, 1),
                                                (2, 8, 1, 0, 0), (513, 1, 1, 1, 0), (64, 16, 16, 0, 1)])
def test_ring_lincomb_bit_exact(n, ma, mb, shift, sub):
    """pb_ring_lincomb (Alg. 3 steps 7-10 mask combination) vs numpy, including
    odd lengths and 8-byte-offset views (the scalar path) beside the 16-byte path."""
    import torch

    from paper_2403_11166_b200 import _dev as D
    from paper_2403_11166_b200 import _lib

    rng = np.random.default_rng(n + ma * 31 + mb)
    T = rng.integers(0, 1 << 64, size=(ma * mb, n), dtype=np.uint64)
    a = rng.integers(0, 1 << 59, size=ma, dtype=np.uint64)
    b = rng.integers(0, 1 << 59, size=mb, dtype=np.uint64)
    base = rng.integers(0, 1 << 59, size=n, dtype=np.uint64)
    coef = (a[:, None] * b[None, :]).reshape(-1)
    acc = (coef[:, None] * T).sum(axis=0, dtype=np.uint64)
    want = ((base - acc) if sub else (base + acc)) & RING.mask
    td = D.u64_to_device(T)
    bd = torch.cat([torch.zeros(shift, dtype=torch.int64, device="cuda"), D.u64_to_device(base)])[shift:]
    out_buf = torch.zeros(n + shift, dtype=torch.int64, device="cuda")
    out = out_buf[shift:]
    ad, bv = D.u64_to_device(a), D.u64_to_device(b)  # kept alive until the kernel has run
    _lib.call("pb_ring_lincomb", sub, D.ptr(out), D.ptr(bd), D.ptr(ad), ma, D.ptr(bv), mb, D.ptr(td), n, 59,
              D.stream())
    torch.cuda.synchronize()
    assert np.array_equal(D.to_numpy_u64(out), want)
