"""OT-based non-linear protocols on the B200 (csrc/pb_nonlinear.cu, SPEC:491-581
with the SPEC:479 dealer OT functionality): every output share is
bit-identical to the oracle restatement (oracle/nonlinear.py) under the same
Philox streams, and private training steps through this backend equal the
oracle's OT-mode step share for share and the reference engine on every
revealed gradient."""

import copy

import numpy as np
import pytest

from oracle import bfv as OB
from oracle import nn as ON
from oracle import nonlinear as NL
from oracle import protocols as OPR
from oracle import ring as OR
from oracle.params import make_params

pytestmark = pytest.mark.gpu

R = OR.RingParams()
M = np.uint64((1 << 59) - 1)
KINDS = {"drelu": 0, "mux": 1, "trunc": 2, "relu_trunc": 3, "trunc_mux": 4}


def _inputs(n, seed):
    rng = np.random.default_rng(seed)
    x = OR.encode_fixed(rng.uniform(-200, 200, n), R, 50)
    x[:6] = [0, 1, (1 << 59) - 1, 2, (1 << 57) - 1, (1 << 59) - (1 << 57) + 1]
    r = rng.integers(0, 1 << 59, size=n, dtype=np.uint64)
    d = rng.integers(0, 4, size=n, dtype=np.uint8)
    return r, (x - r) & M, d


@pytest.mark.parametrize("kind", list(KINDS))
@pytest.mark.parametrize("k", [2, 25])
def test_nl_ops_bit_exact_vs_oracle(kind, k):
    import torch

    from paper_2403_11166_b200 import _dev, _lib

    n, off, seed, stream = 5003, 12, 77, 1_000_123
    x0, x1, d = _inputs(n, k + KINDS[kind])
    words = int(_lib.load().pb_nl_words(KINDS[kind]))
    assert words == NL.WORDS[kind]
    want = NL.nl_op(kind, x0, x1, 59, k=k, d=d if kind in ("mux", "trunc_mux") else None, seed=seed, stream=stream,
                    offset=off)
    dx0, dx1 = _dev.u64_to_device(x0), _dev.u64_to_device(x1)
    y0, y1 = _dev.empty_u64(n), _dev.empty_u64(n)
    dd = torch.from_numpy(d).cuda()
    dout = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.call("pb_nl_op", KINDS[kind], _dev.ptr(dx0), _dev.ptr(dx1), n, 59, k, _dev.ptr(dd), _dev.ptr(dout), seed,
              None, stream, off, _dev.ptr(y0), _dev.ptr(y1), _dev.stream())
    torch.cuda.synchronize()
    if want[0] is not None:
        assert np.array_equal(_dev.to_numpy_u64(y0), want[0])
        assert np.array_equal(_dev.to_numpy_u64(y1), want[1])
    if want[2] is not None:
        assert np.array_equal(dout.cpu().numpy(), want[2])


@pytest.mark.parametrize("ell,k", [(40, 7), (62, 13), (21, 9), (8, 3)])
def test_nl_relu_trunc_other_widths_bit_exact(ell, k):
    """Ring widths / shifts beyond the engine's ell = 59, f = 25: the
    comparison tree's other compile-time leaf counts (ceil(bits / 4) = 1..16)."""
    import torch

    from paper_2403_11166_b200 import _dev, _lib

    n, off, seed, stream = 3001, 5, 91, 2_000_321
    m = np.uint64((1 << ell) - 1)
    rng = np.random.default_rng(ell * 100 + k)
    x0 = rng.integers(0, 1 << ell, size=n, dtype=np.uint64)
    x1 = rng.integers(0, 1 << ell, size=n, dtype=np.uint64)
    x1[:4] = [0, 1, m, m - x0[3]]
    for kind in ("relu_trunc", "trunc", "drelu"):
        want = NL.nl_op(kind, x0, x1, ell, k=k, seed=seed, stream=stream, offset=off)
        y0, y1 = _dev.empty_u64(n), _dev.empty_u64(n)
        dout = torch.empty(n, dtype=torch.uint8, device="cuda")
        dx0, dx1 = _dev.u64_to_device(x0), _dev.u64_to_device(x1)  # referenced until the kernel ran
        _lib.call("pb_nl_op", KINDS[kind], _dev.ptr(dx0), _dev.ptr(dx1), n, ell,
                  k, None, _dev.ptr(dout), seed, None, stream, off, _dev.ptr(y0), _dev.ptr(y1), _dev.stream())
        torch.cuda.synchronize()
        if want[0] is not None:
            assert np.array_equal(_dev.to_numpy_u64(y0), want[0]), kind
            assert np.array_equal(_dev.to_numpy_u64(y1), want[1]), kind
        if want[2] is not None:
            assert np.array_equal(dout.cpu().numpy(), want[2]), kind


@pytest.mark.parametrize("arch,B", [([784, 32, 10], 8), (((2, 8, 8), [("conv", 2, 3, 3, 1, 1), ("pool",),
                                                                   ("conv", 3, 4, 3, 1, 2), ("flatten",),
                                                                   ("fc", 16, 6), ("fc", 6, 10)]), 3)])
def test_private_step_ot_backend_matches_oracle_and_reference(arch, B):
    from paper_2403_11166_b200 import bfv
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.linear_protocols import Session
    from paper_2403_11166_b200.params import BfvParams
    from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed

    op = make_params(8192, 7)
    ar = OB.Arith(op)
    octx = OPR.Ctx(op, R, OB.keygen(op, OR.SeededRng(1, 0), ar), seed=5, ar=ar)
    pr, pp = RingParams(), BfvParams()
    sess = Session(pp, pr, bfv.keygen(pp, SeededRng(1, 0)), seed=5)
    sess.nonlinear = "ot"
    om, rm = ON.Model(arch, R, seed=3), ON.Model(arch, R, seed=3)
    pm = PN.Model(arch, pr, seed=3)
    if isinstance(arch, list):
        xo, labels = ON.synthetic_mnist(4, B, R)
        xh, _ = PN.synthetic_mnist(4, B, pr)
    else:
        xo, labels = ON.synthetic_images(4, B, om.in_shape, R)
        xh, _ = PN.synthetic_images(4, B, om.in_shape, pr)
    xp = RingTensor(encode_fixed(xh, pr), 25, pr, _canonical=True)
    for step in range(2):
        octx.seed = 700 + step
        sess.reseed(700 + step)
        ot, pt = [], []
        l1, gw1, gb1 = ON.private_train_step(octx, om, xo, labels, trace=ot, nonlinear="ot")
        l2, gw2, gb2 = PN.private_train_step(sess, pm, xp, labels, trace=pt)
        l3, gw3, gb3 = ON.reference_train_step(rm, xo, labels)
        assert l1 == l2 == l3
        for (la, ya, _, _), (lb, yb, _, _) in zip(ot, pt):  # every layer's output shares
            assert np.array_equal(yb[0].value.numpy(), ya[0]) and np.array_equal(yb[1].value.numpy(), ya[1])
        for l in range(pm.n_layers):
            assert np.array_equal(gw2[l].numpy(), gw3[l]) and np.array_equal(gb2[l].numpy(), gb3[l])
            assert np.array_equal(gw1[l], gw3[l])
            assert np.array_equal(pm.W[l].numpy(), rm.W(l))


def test_graph_step_ot_backend_matches_eager():
    from paper_2403_11166_b200 import bfv
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.linear_protocols import Session
    from paper_2403_11166_b200.params import BfvParams
    from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed

    pr, pp = RingParams(), BfvParams()
    kp = bfv.keygen(pp, SeededRng(3, 0))
    sizes, B = [784, 32, 10], 16
    xh, labels = PN.synthetic_mnist(7, B, pr)
    s1, s2 = Session(pp, pr, kp, seed=1), Session(pp, pr, kp, seed=1)
    s1.nonlinear = s2.nonlinear = "ot"
    m1, m2 = PN.Model(sizes, pr, seed=4), PN.Model(sizes, pr, seed=4)
    x1 = RingTensor(encode_fixed(xh, pr), 25, pr, _canonical=True)
    runner = PN.GraphStep(s2, m2, RingTensor(encode_fixed(xh, pr), 25, pr, _canonical=True))
    for step in range(3):
        s1.reseed(900 + step)
        l1, _, _ = PN.private_train_step(s1, m1, x1, labels)
        l2 = runner.step(900 + step, labels)
        assert l1 == l2
        for l in range(len(sizes) - 1):
            assert np.array_equal(m1.W[l].numpy(), m2.W[l].numpy())
