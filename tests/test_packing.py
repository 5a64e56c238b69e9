"""Packing codecs and block plans (CPU): SPEC:237-281 examples and invariants,
and the product's index maps == the oracle's (both must pack identically)."""

import numpy as np
import pytest

from oracle import kernels as OK
from oracle import packing as OP
from paper_2403_11166_b200 import poly_encoding as PE
from paper_2403_11166_b200.errors import GeometryError

MATMUL = [(3, 2, 1, 64), (7, 5, 3, 64), (20, 9, 4, 64), (100, 7, 3, 64), (784, 128, 64, 8192), (128, 128, 64, 8192),
          (64, 128, 784, 8192), (128, 10, 64, 8192), (10, 128, 64, 8192), (64, 784, 128, 8192), (2048, 1001, 1, 8192)]
CONV = [(1, 1, 1, 2, 2, 1, 16), (2, 3, 4, 5, 6, 3, 256), (3, 2, 5, 4, 4, 2, 64), (2, 5, 5, 14, 14, 5, 2048),
        (4, 64, 64, 16, 16, 5, 8192), (64, 1, 5, 32, 32, 5, 8192)]


@pytest.mark.parametrize("mode", ["cost", "spec"])
@pytest.mark.parametrize("ni,no,B,N", MATMUL)
def test_matmul_maps_match_oracle(ni, no, B, N, mode):
    g = PE.MatmulGeometry(ni, no, B)
    a, b = PE.plan_blocks(g, N, mode), OP.plan_blocks(OP.MatmulGeometry(ni, no, B), N, mode)
    for f in ("in_src", "pt_src", "out_pos", "out_dst", "terms"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.blk == b.blk and a.nblk == b.nblk


@pytest.mark.parametrize("B,ci,co,h,w,s,N", CONV)
def test_conv_maps_match_oracle(B, ci, co, h, w, s, N):
    g = PE.ConvGeometry(B, ci, co, h, w, s)
    a, b = PE.plan_blocks(g, N), OP.plan_blocks(OP.ConvGeometry(B, ci, co, h, w, s), N)
    for f in ("in_src", "pt_src", "out_pos", "out_dst", "terms"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def _plain_eval(plan, v, W, N):
    vin = OP.pack(plan.in_src, v)
    vw = OP.pack(plan.pt_src, W)
    outs = np.zeros((plan.n_out, N), dtype=np.uint64)
    for r in range(plan.n_out):
        for a, b in plan.terms[r]:
            outs[r] += OK.negacyclic_mul_wrap(vin[a].copy(), vw[b].copy())
    return outs


@pytest.mark.parametrize("mode", ["cost", "spec"])
@pytest.mark.parametrize("ni,no,B,N", MATMUL[:6])
def test_matmul_identity(ni, no, B, N, mode):
    """decode(pi_W(W) pi_v(v)) == W v, incl. input-dimension blocks."""
    rng = np.random.default_rng(ni * 7 + no)
    v = rng.integers(0, 1 << 63, size=(ni, B), dtype=np.uint64)
    W = rng.integers(0, 1 << 63, size=(no, ni), dtype=np.uint64)
    plan = PE.plan_blocks(PE.MatmulGeometry(ni, no, B), N, mode)
    y = OP.unpack(_plain_eval(plan, v, W, N), plan, no * B).reshape(no, B)
    assert np.array_equal(y, OK.matmul_wrap(W, v))


@pytest.mark.parametrize("B,ci,co,h,w,s,N", CONV[:4])
def test_conv_identity(B, ci, co, h, w, s, N):
    rng = np.random.default_rng(B + ci + co)
    v = rng.integers(0, 1 << 63, size=(B, ci, h, w), dtype=np.uint64)
    W = rng.integers(0, 1 << 63, size=(co, ci, s, s), dtype=np.uint64)
    plan = PE.plan_blocks(PE.ConvGeometry(B, ci, co, h, w, s), N)
    e = OK.conv2d_wrap(v, W)
    assert np.array_equal(OP.unpack(_plain_eval(plan, v, W, N), plan, e.size).reshape(e.shape), e)


def test_spec_examples():
    N = 64
    g = PE.MatmulGeometry(3, 2, 1)
    v = PE.matmul_poly_encode("input", [1, 2, 3], g, N)
    assert v[:3].tolist() == [1, 2, 3] and not v[3:].any()
    w = PE.matmul_poly_encode("weight", [[1, 2, 3], [4, 5, 6]], g, N)
    assert w[2] == 1 and w[5] == 4
    y = OK.negacyclic_mul_wrap(v, w)
    assert PE.matmul_poly_decode(y, g, N).ravel().tolist() == [14, 32]
    gc = PE.ConvGeometry(1, 1, 1, 2, 2, 1)
    x = PE.conv_poly_encode("input", [[1, 2], [3, 4]], gc, 16)
    assert x[:4].tolist() == [1, 2, 3, 4]
    k = PE.conv_poly_encode("weight", [[[[2]]]], gc, 16)
    assert k[0] == 2 and not k[1:].any()
    assert PE.conv_poly_decode(OK.negacyclic_mul_wrap(x, k), gc, 16).ravel().tolist() == [2, 4, 6, 8]
    g3 = PE.ConvGeometry(1, 1, 1, 3, 3, 2)
    a = PE.conv_poly_encode("input", np.arange(1, 10).reshape(1, 1, 3, 3), g3, 64)
    b = PE.conv_poly_encode("weight", np.array([[[[1, 0], [0, 1]]]]), g3, 64)
    assert PE.conv_poly_decode(OK.negacyclic_mul_wrap(a, b), g3, 64).ravel().tolist() == [6, 8, 12, 14]
    with pytest.raises(GeometryError):
        PE.matmul_poly_encode("input", np.zeros((100, 1)), PE.MatmulGeometry(100, 1, 1), 64)


def test_compact_maps():
    plan = PE.plan_blocks(PE.MatmulGeometry(100, 7, 3), 64)
    pos, src = PE.compact(plan.in_src)
    dense = np.full_like(plan.in_src, -1)
    for p in range(pos.shape[0]):
        ok = pos[p] >= 0
        dense[p, pos[p][ok]] = src[p][ok]
    assert np.array_equal(dense, plan.in_src)


@pytest.mark.parametrize("mode", ["cost", "spec"])
def test_plan_examples(mode):
    assert PE.plan_blocks(PE.MatmulGeometry(3, 2, 1), 8192, mode).n_out == 1
    p = PE.plan_blocks(PE.MatmulGeometry(2048, 1001, 1), 8192, mode)  # SPEC:274 tiling
    covered = np.zeros(1001, dtype=int)
    ok = p.out_pos >= 0
    np.add.at(covered, p.out_dst[ok], 1)
    assert (covered == 1).all()
    pc = PE.plan_blocks(PE.ConvGeometry(4, 64, 64, 16, 16, 5), 8192)  # SPEC:275 coverage
    used = set(map(tuple, pc.terms.reshape(-1, 2).tolist()))
    nB, nO, nI = pc.nblk
    assert len(used) == nB * nO * nI
