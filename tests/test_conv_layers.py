"""Conv-layer operators (CPU): the conv-layer block plans (padding, stride,
flips and transpositions folded into the index maps of the native conv
packing) evaluated in the clear equal the plaintext ring operators, for the
engine's plans (cost and SPEC tilings) and the oracle's; the oracle's private
CNN step (HE conv protocols + dealer ReLU / truncation / AvgPool2) reveals
exactly the gradients of ``reference_train_step``."""

import copy
import itertools

import numpy as np
import pytest

from oracle import convops as CO
from oracle import kernels as OK
from oracle import nn as ON
from oracle import packing as OP
from paper_2403_11166_b200 import poly_encoding as PE

M64 = (1 << 64) - 1

CASES = [  # B, c_i, c_o, H, W, s, pad, stride
    (2, 1, 3, 6, 6, 3, 1, 2), (2, 2, 3, 5, 5, 3, 1, 1), (1, 2, 2, 7, 7, 5, 2, 2), (3, 1, 2, 8, 8, 5, 2, 2),
    (2, 3, 2, 4, 4, 1, 0, 1), (2, 1, 2, 28, 28, 5, 2, 2), (1, 4, 3, 6, 6, 3, 0, 1), (2, 2, 2, 9, 9, 3, 1, 3),
]


def _brute_fwd(x, w, p, st):
    B, ci, H, W = x.shape
    co, _, s, _ = w.shape
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p))).astype(object)
    oh, ow = OP.conv_out_hw(H, W, s, p, st)
    y = np.zeros((B, co, oh, ow), dtype=object)
    for b, o, yy, xx in itertools.product(range(B), range(co), range(oh), range(ow)):
        y[b, o, yy, xx] = int((xp[b, :, yy * st:yy * st + s, xx * st:xx * st + s] * w[o].astype(object)).sum()) & M64
    return y.astype(np.uint64)


def _dot(a, b):
    return int((a.astype(object) * b.astype(object)).sum()) % (1 << 64)


@pytest.mark.parametrize("case", CASES[:5])
def test_plaintext_conv_ops(case):
    B, ci, co, H, W, s, p, st = case
    rng = np.random.default_rng(1)
    x = rng.integers(0, 1 << 62, size=(B, ci, H, W), dtype=np.uint64)
    w = rng.integers(0, 1 << 62, size=(co, ci, s, s), dtype=np.uint64)
    y = CO.conv_fwd(x, w, p, st)
    assert np.array_equal(y, _brute_fwd(x, w, p, st))
    gy = rng.integers(0, 1 << 62, size=y.shape, dtype=np.uint64)
    # adjoint identities: <fwd(x), gy> = <x, bwdx(gy)> = <w, gradw(x, gy)>
    assert _dot(y, gy) == _dot(x, CO.conv_bwdx(gy, w, H, W, p, st)) == _dot(w, CO.conv_gradw(x, gy, s, p, st))


def _pack_eval(plan, v, W, n_out):
    N = plan.N
    vin = OP.pack(plan.in_src, v)
    wpt = OP.pack(plan.pt_src, W)
    outs = np.zeros((plan.n_out, N), dtype=np.uint64)
    for r in range(plan.n_out):
        for k in range(plan.terms.shape[1]):
            a, b = plan.terms[r, k]
            outs[r] += OK.negacyclic_mul_wrap(vin[a], wpt[b])
    return OP.unpack(outs, plan, n_out)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("kind", ["fwd", "bwdx", "gradw"])
def test_conv_layer_plans_equal_ring_ops(case, kind):
    B, ci, co, H, W, s, p, st = case
    rng = np.random.default_rng(2)
    x = rng.integers(0, 1 << 59, size=(B, ci, H, W), dtype=np.uint64)
    w = rng.integers(0, 1 << 59, size=(co, ci, s, s), dtype=np.uint64)
    oh, ow = OP.conv_out_hw(H, W, s, p, st)
    gy = rng.integers(0, 1 << 59, size=(B, co, oh, ow), dtype=np.uint64)
    v, Wt, want = {"fwd": (x, w, CO.conv_fwd(x, w, p, st)),
                   "bwdx": (gy, w, CO.conv_bwdx(gy, w, H, W, p, st)),
                   "gradw": (x, gy, CO.conv_gradw(x, gy, s, p, st))}[kind]
    N = 2048
    plans = [OP.plan_conv_layer(kind, B, ci, co, H, W, s, p, st, N),
             PE.plan_conv_layer(kind, B, ci, co, H, W, s, p, st, N, "spec"),
             PE.plan_conv_layer(kind, B, ci, co, H, W, s, p, st, N, "cost")]
    for plan in plans:
        got = _pack_eval(plan, v, Wt, want.size).reshape(want.shape)
        assert np.array_equal(got, want), (kind, case)


def test_oracle_private_cnn_step_equals_reference_engine():
    from oracle import bfv as OB
    from oracle import protocols as PR
    from oracle import ring as OR
    from oracle.params import make_params

    R = OR.RingParams()
    p = make_params(8192, 7)
    ar = OB.Arith(p)
    ctx = PR.Ctx(p, R, OB.keygen(p, OR.SeededRng(1, 0), ar), seed=5, ar=ar)
    arch = ((2, 8, 8), [("conv", 2, 3, 3, 1, 1), ("pool",), ("conv", 3, 4, 3, 1, 2), ("flatten",),
                        ("fc", 16, 6), ("fc", 6, 10)])
    m1 = ON.Model(arch, R, seed=3)
    m2 = copy.deepcopy(m1)
    x, labels = ON.synthetic_images(4, 3, m1.in_shape, R)
    l1, gw1, gb1 = ON.reference_train_step(m1, x, labels)
    l2, gw2, gb2 = ON.private_train_step(ctx, m2, x, labels)
    assert l1 == l2
    for l in range(m1.n_layers):
        assert np.array_equal(gw1[l], gw2[l]) and np.array_equal(gb1[l], gb2[l]), l
        assert np.array_equal(m1.w[l], m2.w[l])


def test_model_zoo_shapes():
    assert ON.Model("mnist_cnn", ON.RingParams() if hasattr(ON, "RingParams") else __import__("oracle.ring").ring.RingParams()).io[-1][1] == (10,)
    for name in ("mnist_cnn2", "cifar_cnn", "mnist_mlp"):
        m = ON.Model(name, __import__("oracle.ring").ring.RingParams())
        assert m.io[-1][1] == (10,)
