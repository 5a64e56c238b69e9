"""Kernel-level parity: the sm_100a engine vs the CPU oracle (K restated),
bit-exact on identical inputs and tables (SURVEY §8c parity definition i)."""

import numpy as np
import pytest

from oracle import kernels as OK
from oracle.params import make_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kc():
    from paper_2403_11166_b200 import kernels_compat

    return kernels_compat


def _rows(p, P, seed):
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(
        np.stack([np.stack([rng.integers(0, q, size=p.N, dtype=np.uint64) for q in p.moduli]) for _ in range(P)])
        .reshape(P * p.L, p.N)
    )


@pytest.mark.parametrize("N,L", [(16, 2), (64, 3), (1024, 2), (2048, 2), (4096, 3), (8192, 7), (16384, 4), (32768, 8)])
def test_ntt_forward_inverse_bit_exact(kc, N, L):
    p = make_params(N, L)
    tb = p.tables
    P = 3
    rows = _rows(p, P, N + L)
    q = np.tile(tb["q"], P)
    psi = np.ascontiguousarray(np.tile(tb["psi_brv"], (P, 1)))
    ipsi = np.ascontiguousarray(np.tile(tb["ipsi_brv"], (P, 1)))
    ninv = np.tile(tb["n_inv"], P)
    want = rows.copy()
    OK.ntt_forward_cyc(want, tb["psi_brv"], tb["q"])
    got = rows.copy()
    kc.ntt_forward(got, psi, q)
    assert np.array_equal(got, want)
    want_i = rows.copy()
    OK.ntt_inverse_cyc(want_i, tb["ipsi_brv"], tb["n_inv"], tb["q"])
    got_i = rows.copy()
    kc.ntt_inverse(got_i, ipsi, ninv, q)
    assert np.array_equal(got_i, want_i)
    # round trip
    kc.ntt_inverse(got, ipsi, ninv, q)
    assert np.array_equal(got, rows)


def test_ntt_edge_values(kc):
    """All-zero, all-(q-1) and delta rows (maximal lazy-reduction pressure)."""
    p = make_params(8192, 2)
    tb = p.tables
    rows = np.zeros((6, p.N), dtype=np.uint64)
    rows[2] = tb["q"][0] - 1
    rows[3] = tb["q"][1] - 1
    rows[4, 0] = 1
    rows[5, -1] = tb["q"][1] - 1
    q = np.tile(tb["q"], 3)
    want = rows.copy()
    OK.ntt_forward_cyc(want, tb["psi_brv"], tb["q"])
    got = rows.copy()
    kc.ntt_forward(got, np.ascontiguousarray(np.tile(tb["psi_brv"], (3, 1))), q)
    assert np.array_equal(got, want)


def test_spec_ntt_example_small_n(kc, golden):
    g = golden["kernels"]
    for N, L in ((16, 2), (256, 3), (2048, 2), (8192, 1)):
        tb = make_params(N, L).tables
        rows = g[f"ntt_{N}_{L}_in"].copy()
        P = rows.shape[0] // L
        kc.ntt_forward(rows, np.ascontiguousarray(np.tile(tb["psi_brv"], (P, 1))), np.tile(tb["q"], P))
        assert np.array_equal(rows, g[f"ntt_{N}_{L}_fwd"])


@pytest.mark.parametrize("N,L", [(2048, 2), (8192, 7)])
def test_pointwise_bit_exact(kc, N, L):
    p = make_params(N, L)
    tb = p.tables
    P = 2
    a = _rows(p, P, 1)
    b = _rows(p, P, 2)
    o0 = _rows(p, P, 3)
    q = np.tile(tb["q"], P)
    for fn_o, fn_g in ((OK.pw_mul, kc.pw_mul), (OK.pw_mul_acc, kc.pw_mul_acc), (OK.pw_add, kc.pw_add),
                       (OK.pw_sub, kc.pw_sub)):
        w = o0.copy()
        fn_o(w, a, b, q)
        g = o0.copy()
        fn_g(g, a, b, q)
        assert np.array_equal(g, w), fn_o.__name__


@pytest.mark.parametrize("N,L", [(256, 3), (1024, 7)])
def test_decode_bit_exact(kc, golden, N, L):
    g = golden["kernels"]
    tb = make_params(N, L).tables
    d = kc.garner_digits(g[f"dec_{N}_{L}_in"], tb["q"], tb["prefix_inv"])
    assert np.array_equal(d, g[f"dec_{N}_{L}_digits"])
    m = kc.scale_round_digits(d, tb["int_part"], tb["frac_part"], np.uint64((1 << 59) - 1), q=tb["q"])
    assert np.array_equal(m, g[f"dec_{N}_{L}_m"])


def test_ring_kernels_bit_exact(kc, golden):
    g = golden["kernels"]
    assert np.array_equal(kc.negacyclic_mul_wrap(g["negwrap_a"], g["negwrap_b"]), g["negwrap"])
    assert np.array_equal(kc.matmul_wrap(g["mm_a"], g["mm_b"]), g["mm"])
    assert np.array_equal(kc.conv2d_wrap(g["conv_x"], g["conv_w"]), g["conv"])
    assert np.array_equal(kc.im2col_wrap(g["conv_x"], 3, 2), g["im2col_s3_st2"])
    cols = OK.im2col_wrap(g["conv_x"], 3, 1)
    assert np.array_equal(kc.col2im_wrap(cols, 2, 3, 7, 6, 3, 1), g["col2im_s3_st1"])
    qm = np.uint64(1073692673)
    # NTT-based negacyclic product mod q equals the schoolbook oracle
    a, b = g["negwrap_a"] % qm, g["negwrap_b"] % qm
    assert np.array_equal(kc.negacyclic_mul_mod(a, b, int(qm)), g["negmod"])


def test_large_matmul(kc):
    rng = np.random.default_rng(5)
    a = rng.integers(0, 1 << 63, size=(128, 784), dtype=np.uint64)
    b = rng.integers(0, 1 << 63, size=(784, 64), dtype=np.uint64)
    assert np.array_equal(kc.matmul_wrap(a, b), OK.matmul_wrap(a, b))


@pytest.mark.parametrize("n,k,m", [(1, 1, 1), (10, 128, 64), (128, 128, 64), (17, 300, 33), (128, 64, 784),
                                   (5, 7, 3), (64, 129, 16)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_ring_matmul_add_transposes(n, k, m, ta, tb):
    """pb_ring_matmul_add: c +/- (A B) mod 2^ell for every transpose flag, ragged
    tiles and k across the 128-deep slab, against numpy's wrapping u64 GEMM."""
    from paper_2403_11166_b200 import _dev, _lib

    rng = np.random.default_rng(n * 1000 + k * 10 + m + ta * 7 + tb * 3)
    a = rng.integers(0, 1 << 63, size=(n, k), dtype=np.uint64)
    b = rng.integers(0, 1 << 63, size=(k, m), dtype=np.uint64)
    c = rng.integers(0, 1 << 63, size=(n, m), dtype=np.uint64)
    ab = OK.matmul_wrap(a, b)
    mask = np.uint64((1 << 59) - 1)
    da = _dev.u64_to_device(np.ascontiguousarray(a.T) if ta else a)
    db = _dev.u64_to_device(np.ascontiguousarray(b.T) if tb else b)
    dc = _dev.u64_to_device(c)
    for sign, want in ((1, (c + ab) & mask), (-1, (c - ab) & mask), (0, ab & mask)):
        out = _dev.empty_u64(n, m)
        _lib.call("pb_ring_matmul_add", _dev.ptr(da), _dev.ptr(db), n, k, m, ta, tb, _dev.ptr(dc) if sign else None,
                  sign, 59, _dev.ptr(out), _dev.stream())
        assert np.array_equal(_dev.to_numpy_u64(out), want)


@pytest.mark.parametrize("nB,nO,nI,terms", [(4, 3, 1, "A"), (3, 5, 2, "A"), (2, 3, 1, "AB"), (5, 2, 2, "AB"),
                                            (3, 2, 1, "B")])
def test_mask_mac_fused_equals_two_step(nB, nO, nI, terms):
    """pb_mask_mac (mask NTT + streaming MAC in one pass) is bit-identical to
    pb_mask_ntt followed by pb_ctpt_mac_tiled."""
    import torch

    from paper_2403_11166_b200 import _lib
    from paper_2403_11166_b200.params import BfvParams, context

    p = BfvParams()
    h = context(p).handle
    L, N = p.L, p.N
    g = torch.Generator(device="cuda").manual_seed(nB * 100 + nO * 10 + nI)
    q = min(p.moduli)

    def rnd(*shape):
        return torch.randint(0, q, shape, dtype=torch.int32, device="cuda", generator=g)

    ctA = rnd(nB * nI, 2, L, N) if "A" in terms else None
    ptA = rnd(nO * nI, L, N) if "A" in terms else None
    ctB = rnd(nO * nI, 2, L, N) if "B" in terms else None
    ptB = rnd(nB * nI, L, N) if "B" in terms else None
    U = 77
    n_out = nB * nO
    pos = torch.stack([torch.randperm(N, device="cuda", generator=g)[:U] for _ in range(n_out)]).to(torch.int32)
    pos[:, ::7] = -1
    dst = torch.arange(n_out * U, dtype=torch.int64, device="cuda").reshape(n_out, U)
    mask = torch.randint(0, 1 << 59, (n_out * U,), dtype=torch.int64, device="cuda", generator=g)
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    st = torch.cuda.current_stream().cuda_stream
    two = torch.zeros(n_out, 2, L, N, dtype=torch.int32, device="cuda")
    _lib.call("pb_mask_ntt", h, n_out, pos.data_ptr(), dst.data_ptr(), U, mask.data_ptr(), 1, 99, None,
              two.data_ptr(), st)
    _lib.call("pb_ctpt_mac_tiled", h, ptr(ctA), ptr(ptA), ptr(ctB), ptr(ptB), nB, nO, nI, two.data_ptr(), st)
    one = torch.full((n_out, 2, L, N), 7, dtype=torch.int32, device="cuda")
    _lib.call("pb_mask_mac", h, ptr(ctA), ptr(ptA), ptr(ctB), ptr(ptB), nB, nO, nI, pos.data_ptr(), dst.data_ptr(), U,
              mask.data_ptr(), 1, 99, None, one.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(one, two)


@pytest.mark.parametrize("nB,nO,nI,terms", [
    (1, 3, 4, "A"), (1, 3, 4, "AB"),        # one batch block: 1x1 tiles
    (3, 5, 13, "A"),                        # 2x2, 4-deep ring, a fold after 12 k-steps, ragged tile edges
    (3, 5, 7, "AB"), (2, 2, 3, "AB"),       # two cross terms: 2x2, 2-deep ring, a fold after 6
    (2, 3, 16, "B"),                        # the second term alone
    (4, 2, 1, "A"), (3, 3, 2, "AB"),        # streaming shapes (eager kernel)
])
def test_ctpt_mac_tiled_vs_modular_sum(nB, nO, nI, terms):
    """pb_ctpt_mac_tiled against the definition (K:89-95 pw_mul_acc over k):
    c0 = c0_in + sum_k ct0 * pt * 2^-32, c1 = sum_k ct1 * pt * 2^-32 (pt in
    Montgomery form), plus the second cross term, mod each q -- for every
    tile / ring-depth / fold configuration the dispatcher picks."""
    import torch

    from paper_2403_11166_b200 import _lib
    from paper_2403_11166_b200.params import BfvParams, context

    p = BfvParams()
    h = context(p).handle
    L, N = p.L, p.N
    rng = np.random.default_rng(nB * 1000 + nO * 100 + nI * 10 + len(terms))
    qs = np.array(p.moduli, dtype=np.uint64)

    def rnd(*lead):  # residues < q_l along the limb axis (second to last)
        a = rng.integers(0, 1 << 62, size=(*lead, L, N), dtype=np.uint64)
        return a % qs[:, None]

    ctA = rnd(nB * nI, 2) if "A" in terms else None
    ptA = rnd(nO * nI) if "A" in terms else None
    ctB = rnd(nO * nI, 2) if "B" in terms else None
    ptB = rnd(nB * nI) if "B" in terms else None
    out0 = rnd(nB * nO, 2)
    rinv = np.array([pow(1 << 32, -1, int(q)) for q in p.moduli], dtype=np.uint64)[:, None]
    want = np.zeros((nB * nO, 2, L, N), dtype=np.uint64)
    for b in range(nB):
        for o in range(nO):
            acc = np.zeros((2, L, N), dtype=np.uint64)
            for k in range(nI):
                if ctA is not None:
                    w = ptA[o * nI + k] * rinv % qs[:, None]
                    acc = (acc + ctA[b * nI + k] * w % qs[:, None]) % qs[:, None]
                if ctB is not None:
                    w = ptB[b * nI + k] * rinv % qs[:, None]
                    acc = (acc + ctB[o * nI + k] * w % qs[:, None]) % qs[:, None]
            want[b * nO + o, 0] = (acc[0] + out0[b * nO + o, 0]) % qs[:, None]
            want[b * nO + o, 1] = acc[1]
    dev = lambda a: None if a is None else torch.from_numpy(a.astype(np.int32)).cuda()  # noqa: E731
    tA, pA, tB, pB, out = dev(ctA), dev(ptA), dev(ctB), dev(ptB), dev(out0)
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    _lib.call("pb_ctpt_mac_tiled", h, ptr(tA), ptr(pA), ptr(tB), ptr(pB), nB, nO, nI, out.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().astype(np.uint64), want)
