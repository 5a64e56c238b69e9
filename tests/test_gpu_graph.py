"""CUDA-graph replay of the private step == the eager step, bit for bit
(the graphs re-key every random stream through the device seed word)."""

import copy

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_graph_step_matches_eager_and_reference():
    from oracle import nn as ON
    from oracle import ring as OR
    from paper_2403_11166_b200 import bfv
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.linear_protocols import Session
    from paper_2403_11166_b200.params import BfvParams
    from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed

    ring = RingParams()
    params = BfvParams()
    kp = bfv.keygen(params, SeededRng(3, 0))
    sizes, B = [784, 64, 10], 16
    xh, labels = PN.synthetic_mnist(7, B, ring)
    # eager reference run
    s1 = Session(params, ring, kp, seed=1)
    m1 = PN.Model(sizes, ring, seed=4)
    x1 = RingTensor(encode_fixed(xh, ring), 25, ring, _canonical=True)
    # graph run
    s2 = Session(params, ring, kp, seed=1)
    m2 = PN.Model(sizes, ring, seed=4)
    x2 = RingTensor(encode_fixed(xh, ring), 25, ring, _canonical=True)
    runner = PN.GraphStep(s2, m2, x2)  # warm-up/capture use a zero loss gradient: weights unchanged
    om = ON.Model(sizes, OR.RingParams(), seed=4)
    xo, _ = ON.synthetic_mnist(7, B, OR.RingParams())
    for step in range(3):
        s1.reseed(100 + step)
        l1, _, _ = PN.private_train_step(s1, m1, x1, labels)
        l2 = runner.step(100 + step, labels)
        l3, _, _ = ON.reference_train_step(om, xo, labels)
        assert l1 == l2 == l3
        for l in range(len(sizes) - 1):
            assert np.array_equal(m1.W[l].numpy(), m2.W[l].numpy())
            assert np.array_equal(m2.W[l].numpy(), om.W(l))
            assert np.array_equal(m2.w[l].cpu().numpy(), om.w[l])


def test_graph_step_load_batch():
    """load_batch (pinned H2D + device encode, deferred range check) feeds the
    graphs the same input as encode_fixed; an out-of-range batch raises at
    the step's sync."""
    import torch

    from paper_2403_11166_b200 import bfv
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.errors import EncodeRangeError
    from paper_2403_11166_b200.linear_protocols import Session
    from paper_2403_11166_b200.params import BfvParams
    from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed

    ring, params = RingParams(), BfvParams()
    kp = bfv.keygen(params, SeededRng(3, 0))
    sizes, B = [784, 32, 10], 8
    xh, labels = PN.synthetic_mnist(7, B, ring)
    x2h, _ = PN.synthetic_mnist(8, B, ring)
    s1, s2 = Session(params, ring, kp, seed=1), Session(params, ring, kp, seed=1)
    m1, m2 = PN.Model(sizes, ring, seed=4), PN.Model(sizes, ring, seed=4)
    r1 = PN.GraphStep(s1, m1, RingTensor(encode_fixed(xh, ring), 25, ring, _canonical=True))
    r2 = PN.GraphStep(s2, m2, RingTensor(encode_fixed(xh, ring), 25, ring, _canonical=True))
    r1.x.values.copy_(encode_fixed(x2h, ring))
    r2.load_batch(torch.from_numpy(np.ascontiguousarray(x2h)).pin_memory())
    assert r1.step(5, labels) == r2.step(5, labels)
    assert np.array_equal(r1.x.values.cpu().numpy(), r2.x.values.cpu().numpy())
    bad = np.ascontiguousarray(x2h).copy()
    bad[0, 0] = 1e30
    r2.load_batch(torch.from_numpy(bad).pin_memory())
    with pytest.raises(EncodeRangeError):
        r2.step(6, labels)


def test_graph_step_prefetched_input_encryption():
    """prefetch_input: the first layer's input encryption is produced beside the
    previous step (DO-owned key stream); losses and weights still equal the
    eager step's and the oracle's -- with the input resident and via load_batch."""
    import torch

    from oracle import nn as ON
    from oracle import ring as OR
    from paper_2403_11166_b200 import bfv
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.linear_protocols import Session
    from paper_2403_11166_b200.params import BfvParams
    from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed

    ring, params = RingParams(), BfvParams()
    kp = bfv.keygen(params, SeededRng(3, 0))
    sizes, B = [784, 32, 10], 16
    xh, labels = PN.synthetic_mnist(7, B, ring)
    x2h, labels2 = PN.synthetic_mnist(8, B, ring)
    s1, s2 = Session(params, ring, kp, seed=1), Session(params, ring, kp, seed=1)
    m1, m2 = PN.Model(sizes, ring, seed=4), PN.Model(sizes, ring, seed=4)
    x1 = RingTensor(encode_fixed(xh, ring), 25, ring, _canonical=True)
    runner = PN.GraphStep(s2, m2, RingTensor(encode_fixed(xh, ring), 25, ring, _canonical=True), prefetch_input=True)
    om = ON.Model(sizes, OR.RingParams(), seed=4)
    xo, _ = ON.synthetic_mnist(7, B, OR.RingParams())
    x2o, _ = ON.synthetic_mnist(8, B, OR.RingParams())
    for step in range(4):
        if step >= 2:  # switch to a new batch through load_batch
            x1 = RingTensor(encode_fixed(x2h, ring), 25, ring, _canonical=True)
            runner.load_batch(torch.from_numpy(np.ascontiguousarray(x2h)).pin_memory())
            xo, lab = x2o, labels2
        else:
            lab = labels
        s1.reseed(200 + step)
        l1, _, _ = PN.private_train_step(s1, m1, x1, lab)
        l2 = runner.step(200 + step, lab)
        l3, _, _ = ON.reference_train_step(om, xo, lab)
        assert l1 == l2 == l3
        for l in range(len(sizes) - 1):
            assert np.array_equal(m1.W[l].numpy(), m2.W[l].numpy())
            assert np.array_equal(m2.W[l].numpy(), om.W(l))
