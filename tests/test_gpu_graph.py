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


def test_graph_step_abort_leaves_weights_untouched():
    """A step whose host loss raises (EncodeRangeError from load_batch) still
    releases the already-launched backward graph, but with the abort word set:
    its SGD launches are no-ops, so weights, master weights and momentum stay
    bit-identical; the next good step matches the eager engine and the oracle
    (which never saw the bad batch)."""
    import torch

    from oracle import nn as ON
    from oracle import ring as OR
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
    s1, s2 = Session(params, ring, kp, seed=1), Session(params, ring, kp, seed=1)
    m1, m2 = PN.Model(sizes, ring, seed=4), PN.Model(sizes, ring, seed=4)
    x1 = RingTensor(encode_fixed(xh, ring), 25, ring, _canonical=True)
    runner = PN.GraphStep(s2, m2, RingTensor(encode_fixed(xh, ring), 25, ring, _canonical=True))
    om = ON.Model(sizes, OR.RingParams(), seed=4)
    xo, _ = ON.synthetic_mnist(7, B, OR.RingParams())

    def snap(m):
        return [t.detach().cpu().numpy().copy() for l in range(len(sizes) - 1)
                for t in (m.W[l].values if hasattr(m.W[l], "values") else m.W[l], m.w[l], m.vw[l], m.b[l], m.vb[l])]

    s1.reseed(300)
    PN.private_train_step(s1, m1, x1, labels)
    runner.step(300, labels)
    ON.reference_train_step(om, xo, labels)
    before = snap(m2)
    bad = np.ascontiguousarray(xh).copy()
    bad[0, 0] = 1e30
    runner.load_batch(torch.from_numpy(bad).pin_memory())
    with pytest.raises(EncodeRangeError):
        runner.step(301, labels)
    torch.cuda.synchronize()
    after = snap(m2)
    assert all(np.array_equal(a, b) for a, b in zip(before, after)), "aborted step changed the model"
    assert int(m2.skip.item()) == 0
    # recovery: a good batch again; the step equals eager and the oracle
    runner.load_batch(torch.from_numpy(np.ascontiguousarray(xh)).pin_memory())
    s1.reseed(302)
    l1, _, _ = PN.private_train_step(s1, m1, x1, labels)
    l2 = runner.step(302, labels)
    l3, _, _ = ON.reference_train_step(om, xo, labels)
    assert l1 == l2 == l3
    for l in range(len(sizes) - 1):
        assert np.array_equal(m1.W[l].numpy(), m2.W[l].numpy())
        assert np.array_equal(m2.W[l].numpy(), om.W(l))


def test_host_handoff_timeout_sets_skip():
    """pb_host_handoff with no release: after the timeout it acks UINT32_MAX and
    sets the skip word, and pb_sgd_momentum under that word is a no-op."""
    import torch

    from paper_2403_11166_b200 import _lib

    dev = torch.device("cuda:0")
    flag = torch.zeros(3, dtype=torch.int32).pin_memory()
    seq = torch.zeros(1, dtype=torch.int32, device=dev)
    src = torch.arange(16, dtype=torch.int64).pin_memory()
    dst = torch.zeros(16, dtype=torch.int64, device=dev)
    skip = torch.zeros(1, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("pb_host_handoff", flag.data_ptr(), seq.data_ptr(), src.data_ptr(), dst.data_ptr(), 16,
              2_000_000, skip.data_ptr(), st)  # 2 ms, never released
    torch.cuda.synchronize()
    assert int(skip.item()) == 1 and int(flag[1]) == -1
    w = torch.ones(8, dtype=torch.float64, device=dev)
    v = torch.zeros(8, dtype=torch.float64, device=dev)
    g = torch.full((8,), 1 << 25, dtype=torch.int64, device=dev)
    wr = torch.zeros(8, dtype=torch.int64, device=dev)
    fl = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("pb_sgd_momentum", w.data_ptr(), v.data_ptr(), g.data_ptr(), 8, 25, 0.5, 0.8, 59, 25, wr.data_ptr(),
              fl.data_ptr(), skip.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.all(w == 1) and torch.all(v == 0) and torch.all(wr == 0)
    # released on time: skip cleared, gradient copied
    flag[0] = 0  # seq was poisoned to UINT32_MAX: the next want is 0
    _lib.call("pb_host_handoff", flag.data_ptr(), seq.data_ptr(), src.data_ptr(), dst.data_ptr(), 16,
              2_000_000_000, skip.data_ptr(), st)
    torch.cuda.synchronize()
    assert int(skip.item()) == 0 and torch.equal(dst.cpu(), src)


def test_graph_step_pipelined_next_batch():
    """step(..., next_batch=...) stages the next input during this step; the
    trajectory equals loading each batch before its step (and the oracle)."""
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
    sizes, B = [784, 32, 10], 8
    batches = [PN.synthetic_mnist(20 + i, B, ring) for i in range(4)]
    pins = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x, _ in batches]
    s1, s2 = Session(params, ring, kp, seed=1), Session(params, ring, kp, seed=1)
    m1, m2 = PN.Model(sizes, ring, seed=4), PN.Model(sizes, ring, seed=4)
    x0 = RingTensor(encode_fixed(batches[0][0], ring), 25, ring, _canonical=True)
    r1 = PN.GraphStep(s1, m1, x0, prefetch_input=True)
    r2 = PN.GraphStep(s2, m2, RingTensor(encode_fixed(batches[0][0], ring), 25, ring, _canonical=True),
                      prefetch_input=True)
    om = ON.Model(sizes, OR.RingParams(), seed=4)
    r2.load_batch(pins[0])
    for i in range(4):
        r1.load_batch(pins[i])
        l1 = r1.step(500 + i, batches[i][1])
        l2 = r2.step(500 + i, batches[i][1], next_batch=pins[(i + 1) % 4])
        xo, _ = ON.synthetic_mnist(20 + i, B, OR.RingParams())
        l3, _, _ = ON.reference_train_step(om, xo, batches[i][1])
        assert l1 == l2 == l3
        for l in range(len(sizes) - 1):
            assert np.array_equal(m1.W[l].numpy(), m2.W[l].numpy())
            assert np.array_equal(m2.W[l].numpy(), om.W(l))
