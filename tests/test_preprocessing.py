"""Pencil+ preprocessing (PAPER Alg. 3/4) in the oracle (CPU):
the mask-bank online product reconstructs u o v exactly for every operator
kind, and a prep-mode private training step (Alg. 4) reveals exactly the
gradients of reference_train_step ("private (fullhe) == private
(prep) == reference")."""

import copy

import numpy as np
import pytest

from oracle import bfv as OB
from oracle import nn as ON
from oracle import preprocessing as PP
from oracle import protocols as PR
from oracle import ring as OR
from oracle.params import make_params

R = OR.RingParams()


@pytest.fixture(scope="module")
def ctx():
    p = make_params(8192, 7)
    ar = OB.Arith(p)
    return PR.Ctx(p, R, OB.keygen(p, OR.SeededRng(1, 0), ar), seed=5, ar=ar)


@pytest.mark.parametrize("spec,hw", [(("fc", 12, 5), None), (("conv", 2, 3, 3, 1, 2), (6, 6))])
@pytest.mark.parametrize("op", range(4))
def test_online_product_reconstructs(ctx, spec, hw, op):
    opd = PP.Operator(spec, op, 3, hw)
    bank = PP.prep_operator(ctx, 1, opd, 2, bank_seed=4)
    # trusted check of the bank: s_ij + D_ij = u'_i o v'_j
    for i in range(2):
        for j in range(2):
            assert np.array_equal((bank.s[i, j] + bank.d[i, j]) & R.mask, opd.apply(bank.u[i], bank.v[j]) & R.mask)
    rng = np.random.default_rng(op)
    for trial in range(2):
        ctx.seed = 50 + trial
        u = rng.integers(0, 1 << 59, size=opd.u_shape, dtype=np.uint64)
        v = rng.integers(0, 1 << 59, size=opd.v_shape, dtype=np.uint64)
        mo, do = PP.online_shared_product(ctx, 1, bank, u, v)
        assert np.array_equal((mo + do) & R.mask, opd.apply(u, v) & R.mask)
    assert bank.n_used == 2
    ctx.seed = 5


def test_prep_step_equals_reference_engine(ctx):
    arch = ((2, 8, 8), [("conv", 2, 3, 3, 1, 1), ("pool",), ("conv", 3, 4, 3, 1, 2), ("flatten",),
                        ("fc", 16, 6), ("fc", 6, 10)])
    m1 = ON.Model(arch, R, seed=3)
    m2 = copy.deepcopy(m1)
    x, labels = ON.synthetic_images(4, 3, m1.in_shape, R)
    state = PP.PrepState(ctx, m2, 3, m=2, bank_seed=9)
    for step in range(2):
        ctx.seed = 100 + step
        l1, gw1, gb1 = ON.reference_train_step(m1, x, labels)
        l2, gw2, gb2 = ON.private_train_step(ctx, m2, x, labels, prep=state)
        assert l1 == l2
        for a, b in zip(gw1 + gb1, gw2 + gb2):
            assert np.array_equal(a, b)
    ctx.seed = 5
