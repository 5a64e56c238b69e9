"""The DO's host loss step (nn.SoftmaxCE: pb_host_softmax_* + numpy exp/log,
pb_host_mean) is bit-identical to the oracle's numpy softmax_ce_grad
(oracle/protocols.py) -- loss and encoded gradient -- over random logit
scales, class counts and batch sizes (incl. B = 1, where numpy reduces the
class axis pairwise).  Host code only: runs without a GPU."""

import ctypes

import numpy as np

from oracle.protocols import softmax_ce_grad as oracle_sce
from oracle.ring import RingParams as ORing


def test_softmax_ce_bit_exact_vs_oracle():
    from paper_2403_11166_b200.nn import softmax_ce_grad
    from paper_2403_11166_b200.ring import RingParams

    ring, oring = RingParams(), ORing()
    rng = np.random.default_rng(11)
    for _ in range(1500):
        sc = int(rng.integers(8, 58))
        C, B = int(rng.integers(2, 12)), int(rng.integers(1, 140))
        logits = rng.integers(-(1 << sc), 1 << sc, size=(C, B)).astype(np.int64).view(np.uint64) & ring.mask
        labels = rng.integers(0, C, size=B)
        l1, g1 = softmax_ce_grad(logits, labels, ring)
        l2, g2 = oracle_sce(logits, labels, oring)
        assert l1 == l2
        assert np.array_equal(g1, g2)


def test_host_mean_is_numpy_mean():
    from paper_2403_11166_b200 import _lib

    f = _lib.load().pb_host_mean
    rng = np.random.default_rng(12)
    for _ in range(3000):
        n = int(rng.integers(1, 600))
        a = rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3)
        assert f(a.ctypes.data_as(ctypes.c_void_p), n) == np.mean(a)
