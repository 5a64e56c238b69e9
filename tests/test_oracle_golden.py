"""Pin the CPU oracle to the reference (CPU-only).

Every vector in tests/golden/*.npz was produced by the unmodified reference
(``pencil._kernels`` / ``pencil.ring``) by tests/golden/make_golden.py.  The
oracle restatement (oracle/kernels.c, oracle/ring.py) must reproduce them
bit-for-bit before it is trusted as the parity checker for the GPU path.
"""

import numpy as np
import pytest

from oracle import kernels as OK
from oracle import ring as OR
from oracle.params import make_params


@pytest.mark.parametrize("N,L", [(16, 2), (256, 3), (2048, 2), (8192, 1)])
def test_ntt_and_pointwise_match_reference(golden, N, L):
    g = golden["kernels"]
    p = make_params(N, L)
    tb = p.tables
    rows = g[f"ntt_{N}_{L}_in"]
    P = rows.shape[0] // L
    q = np.tile(tb["q"], P)
    fwd = rows.copy()
    OK.ntt_forward(fwd, np.ascontiguousarray(np.tile(tb["psi_brv"], (P, 1))), q)
    assert np.array_equal(fwd, g[f"ntt_{N}_{L}_fwd"])
    inv = rows.copy()
    OK.ntt_inverse(inv, np.ascontiguousarray(np.tile(tb["ipsi_brv"], (P, 1))), np.tile(tb["n_inv"], P), q)
    assert np.array_equal(inv, g[f"ntt_{N}_{L}_inv"])
    # cyclic-table variants used by the oracle glue are the same arithmetic
    f2 = rows.copy()
    OK.ntt_forward_cyc(f2, tb["psi_brv"], tb["q"])
    assert np.array_equal(f2, fwd)
    i2 = rows.copy()
    OK.ntt_inverse_cyc(i2, tb["ipsi_brv"], tb["n_inv"], tb["q"])
    assert np.array_equal(i2, inv)
    b = np.ascontiguousarray(np.roll(rows, 1, axis=1))
    for name, fn, op in (("mul", OK.pw_mul, "mul"), ("mac", OK.pw_mul_acc, "mul_acc"),
                         ("add", OK.pw_add, "add"), ("sub", OK.pw_sub, "sub")):
        o = fwd.copy()
        fn(o, rows, b, q)
        assert np.array_equal(o, g[f"pw_{name}_{N}_{L}"]), name
        o2 = fwd.copy()
        OK.pw_cyc(op, o2, rows, b, tb["q"])
        assert np.array_equal(o2, o), name


def test_spec_ntt_examples(golden):
    """(1+x)^2 -> [1,2,1,0]; x^3 * x -> [16,0,0,0] mod 17."""
    g = golden["kernels"]
    assert g["spec_ntt_1px_sq"].tolist() == [1, 2, 1, 0]
    assert g["spec_ntt_x3_x"].tolist() == [16, 0, 0, 0]
    q17 = np.array([17], dtype=np.uint64)
    brv4 = [0, 2, 1, 3]
    psi_brv = np.array([[pow(9, e, 17) for e in brv4]], dtype=np.uint64)
    ipsi = np.array([[pow(9, -e, 17) for e in brv4]], dtype=np.uint64)
    x = np.array([[1, 1, 0, 0]], dtype=np.uint64)
    OK.ntt_forward(x, psi_brv, q17)
    z = np.empty_like(x)
    OK.pw_mul(z, x, x, q17)
    OK.ntt_inverse(z, ipsi, np.array([13], dtype=np.uint64), q17)
    assert z[0].tolist() == [1, 2, 1, 0]


@pytest.mark.parametrize("N,L", [(256, 3), (1024, 7)])
def test_decode_matches_reference(golden, N, L):
    g = golden["kernels"]
    tb = make_params(N, L).tables
    rows = g[f"dec_{N}_{L}_in"]
    d = OK.garner_digits(rows, tb["q"], tb["prefix_inv"])
    assert np.array_equal(d, g[f"dec_{N}_{L}_digits"])
    m = OK.scale_round_digits(d, tb["int_part"], tb["frac_part"], np.uint64((1 << 59) - 1))
    assert np.array_equal(m, g[f"dec_{N}_{L}_m"])
    mb = OK.decode_batch(np.ascontiguousarray(rows[None]), tb["q"], tb["prefix_inv"], tb["int_part"],
                         tb["frac_part"], np.uint64((1 << 59) - 1))
    assert np.array_equal(mb[0], m)


def test_ring_kernels_match_reference(golden):
    g = golden["kernels"]
    assert np.array_equal(OK.negacyclic_mul_wrap(g["negwrap_a"], g["negwrap_b"]), g["negwrap"])
    qm = np.uint64(1073692673)
    assert np.array_equal(OK.negacyclic_mul_mod(g["negwrap_a"] % qm, g["negwrap_b"] % qm, qm), g["negmod"])
    assert np.array_equal(OK.matmul_wrap(g["mm_a"], g["mm_b"]), g["mm"])
    assert np.array_equal(OK.conv2d_wrap(g["conv_x"], g["conv_w"]), g["conv"])
    assert np.array_equal(OK.im2col_wrap(g["conv_x"], 3, 2), g["im2col_s3_st2"])
    cols = OK.im2col_wrap(g["conv_x"], 3, 1)
    assert np.array_equal(OK.col2im_wrap(cols, 2, 3, 7, 6, 3, 1), g["col2im_s3_st1"])


def test_ring_layer_matches_reference(golden):
    g = golden["ring"]
    P = OR.RingParams()
    assert np.array_equal(OR.encode_fixed(g["enc_x"], P), g["enc_f25"])
    assert np.array_equal(OR.encode_fixed(g["enc_x"][:6] / 1024, P, 50), g["enc_f50"])
    assert np.array_equal(OR.decode_fixed(g["enc_f25"], P), g["dec_f25"])
    assert np.array_equal(OR.to_signed(g["enc_f25"], P), g["signed"])
    r = OR.SeededRng(2024, 7)
    assert np.array_equal(r.uniform_ring((5,), P), g["rng_uniform_ring_5"])
    assert np.array_equal(r.uniform_ring((3, 3), P), g["rng_uniform_ring_3x3"])
    assert np.array_equal(r.ternary((33,)), g["rng_ternary"])
    assert np.array_equal(r.uniform_mod((17,), 1073692673), g["rng_uniform_mod"])
    assert np.array_equal(r.uniform_ring((6,), P), g["rng_uniform_ring_after"])
    assert np.array_equal(OR.SeededRng(1, 0).cbd((64,)), g["rng_cbd"])
    x = OR.RingTensor(g["share_x"], 25, P)
    mo, do = OR.share_tensor(x, OR.SeededRng(99, 3))
    assert np.array_equal(mo.value.values, g["share_mo"])
    assert np.array_equal(do.value.values, g["share_do"])
    assert np.array_equal(OR.reconstruct_tensor(mo, do).values, g["share_rec"])
    y = OR.RingTensor(g["shift_in"], 50, P)
    assert np.array_equal(OR.arith_shift(y, 25).values, g["shift_out"])
    e = OR.RingTensor(g["edge_in"], 25, P)
    assert np.array_equal((-e).values, g["edge_neg"])
    for k, want in zip(g["edge_smul_ks"], g["edge_smul"]):
        assert np.array_equal(e.scalar_mul(int(k)).values, want)
    assert np.array_equal(OR.to_signed(g["edge_in"], P), g["edge_signed"])
    assert np.array_equal(OR.decode_fixed(g["edge_in"], P, 50), g["edge_dec_f50"])
    assert np.array_equal(OR.SeededRng(2024, 1000003).normal((16,), 0.5), g["rng_normal"])


def test_spec_ring_kats():
    """SPEC:42-44, 51-53, 60-61, 69-70."""
    P = OR.RingParams()
    assert int(OR.encode_fixed(1.0, P)) == 33554432
    assert int(OR.encode_fixed(0.5, OR.RingParams(59, 2), 2)) == 2
    assert int(OR.encode_fixed(-1.0, P)) == (1 << 59) - (1 << 25)
    assert float(OR.decode_fixed(np.uint64(33554432), P)) == 1.0
    assert float(OR.decode_fixed(np.uint64((1 << 59) - (1 << 25)), P)) == -1.0
    assert float(OR.decode_fixed(np.uint64(6), OR.RingParams(59, 2), 2)) == 1.5
    x = OR.RingTensor([7], 25, P)
    assert (x - OR.RingTensor([3], 25, P)).values.tolist() == [4]
    assert (OR.RingTensor([0], 25, P) - OR.RingTensor([5], 25, P)).values.tolist() == [(1 << 59) - 5]
    assert (OR.RingTensor([(1 << 59) - 1], 25, P) + OR.RingTensor([2], 25, P)).values.tolist() == [1]
    with pytest.raises(OR.EncodeRangeError):
        OR.encode_fixed(2.0**34, P)
