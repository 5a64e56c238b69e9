"""Noise-budget guards: the masked ciphertexts the
MO returns in the worst-case evaluations of every BASELINE config still hold
a positive margin before decryption -- dense full-range share x share cross
terms (Alg. 2), the longest homomorphic accumulations (CIFAR conv1 weight
gradient: 65 536 products per coefficient), and the Pencil+ banks (uniform
masks on both sides)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MARGIN_BITS = 8  # the decryption fails at 0


@pytest.fixture(scope="module")
def sess():
    from paper_2403_11166_b200 import bfv, ring
    from paper_2403_11166_b200.linear_protocols import Session
    from paper_2403_11166_b200.params import BfvParams

    pp = BfvParams()
    return Session(pp, ring.RingParams(), bfv.keygen(pp, ring.SeededRng(5, 0)), seed=3)


def _shares(sess, shape, seed):
    from paper_2403_11166_b200.ring import DO, MO, RingTensor, SeededRng, ShareTensor

    r = sess.ring
    full = SeededRng(seed, 1).uniform_ring(shape, r)  # dense full-range values: the worst case
    mo = SeededRng(seed, 2).uniform_ring(shape, r)
    do = (full - mo) & ((1 << r.ell) - 1)
    return ShareTensor(MO, RingTensor(mo, r.f, r, _canonical=True)), ShareTensor(DO, RingTensor(do, r.f, r, _canonical=True))


def _min_budget(sess, cts, k=2):
    """Smallest budget over the USEFUL slots of k sampled output ciphertexts per
    batch (the other coefficients carry the MO's uniform filler by design)."""
    from paper_2403_11166_b200 import bfv

    worst = 10 ** 9
    for ct, pos in cts:
        pos = pos.cpu().numpy()  # int32, -1 = no slot
        for i in np.linspace(0, ct.shape[0] - 1, num=min(k, ct.shape[0])).astype(int):
            slots = np.asarray(pos[i]).astype(np.int64)
            slots = slots[slots >= 0]
            if slots.size:
                worst = min(worst, bfv.noise_budget(sess.kp, bfv.Ciphertext(ct[i:i + 1].contiguous(), sess.p), slots))
    return worst


def test_fc_weight_gradient_dense_cross_terms(sess):
    from paper_2403_11166_b200 import linear_protocols as LP

    sess.capture = []
    LP.grad_weight(sess, 0, *_shares(sess, (784, 64), 1), *_shares(sess, (128, 64), 2))
    b = _min_budget(sess, sess.capture)
    sess.capture = None
    assert b >= MARGIN_BITS, b


def test_cifar_conv1_weight_gradient_longest_accumulation(sess):
    from paper_2403_11166_b200 import linear_protocols as LP

    sess.capture = []
    LP.conv_grad_weight(sess, 0, *_shares(sess, (64, 3, 32, 32), 3), *_shares(sess, (64, 64, 32, 32), 4), 5, 2, 1)
    b = _min_budget(sess, sess.capture)
    sess.capture = None
    assert b >= MARGIN_BITS, b


def test_cifar_conv2_input_gradient(sess):
    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200.ring import RingTensor, SeededRng

    r = sess.ring
    W = RingTensor(SeededRng(9, 0).uniform_ring((64, 64, 5, 5), r), r.f, r, _canonical=True)  # full-range weights
    sess.capture = []
    LP.conv_backward_input(sess, 1, W, *_shares(sess, (64, 64, 16, 16), 5), 16, 16, 2, 1)
    b = _min_budget(sess, sess.capture)
    sess.capture = None
    assert b >= MARGIN_BITS, b


def test_prep_bank_uniform_masks(sess):
    from paper_2403_11166_b200 import preprocessing as PP

    sess.capture = []
    PP.prep_operator(sess, 0, PP.Operator(("fc", 784, 128), PP.GRADW, 64), 1, bank_seed=2)
    b = _min_budget(sess, sess.capture)
    sess.capture = None
    assert b >= MARGIN_BITS, b
