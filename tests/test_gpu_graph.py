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
