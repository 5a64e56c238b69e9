"""BFV parity on the B200 vs the CPU oracle (oracle/bfv.py, built on K).

* keygen: bit-identical keys (same host draws, GPU NTT/pointwise);
* encrypt with the oracle's noise: bit-identical ciphertexts (pk and sk);
* decrypt: exact plaintext recovery, equal to the oracle's decryption of the
  same ciphertext; ct x pt equals the negacyclic product mod t (centered lift);
* decrypt_to_share gathers exactly the requested coefficients.
"""

import numpy as np
import pytest

from oracle import bfv as OB
from oracle import kernels as OK
from oracle import ring as OR
from oracle.params import make_params

pytestmark = pytest.mark.gpu

T_MASK = np.uint64((1 << 59) - 1)


@pytest.fixture(scope="module", params=[(2048, 8), (8192, 7)])
def setup(request):
    from paper_2403_11166_b200 import bfv, ring
    from paper_2403_11166_b200.params import BfvParams

    N, L = request.param
    op = make_params(N, L)
    pp = BfvParams(N=N, L=L)
    assert pp.digest() == op.digest()
    ar = OB.Arith(op)
    okp = OB.keygen(op, OR.SeededRng(11, 0), ar)
    pkp = bfv.keygen(pp, ring.SeededRng(11, 0))
    return dict(N=N, L=L, op=op, pp=pp, ar=ar, okp=okp, pkp=pkp)


def test_keygen_bit_exact(setup):
    from paper_2403_11166_b200 import bfv

    s = setup
    assert np.array_equal(s["pkp"].sk_coeff, s["okp"].sk_coeff)
    assert np.array_equal(bfv.to_reference_order(s["pp"], s["pkp"].sk_ntt), s["okp"].sk_ntt)
    assert np.array_equal(bfv.to_reference_order(s["pp"], s["pkp"].pk), s["okp"].pk.reshape(2 * s["L"], -1).reshape(2, s["L"], -1))


def test_encrypt_pk_bit_exact_with_oracle_noise(setup):
    from paper_2403_11166_b200 import _dev, bfv

    s = setup
    N, P = s["N"], 3
    m = OR.SeededRng(5, 1).uniform_ring((P, N), OR.RingParams())
    oct_ = OB.encrypt_pk(s["op"], s["okp"], m, OR.SeededRng(6, 0), s["ar"])
    g = OR.SeededRng(6, 0)
    u, e1, e2 = [], [], []
    for _ in range(P):
        u.append(g.ternary((N,)))
        e1.append(g.cbd((N,)))
        e2.append(g.cbd((N,)))
    ct = bfv.encrypt(s["pkp"], _dev.u64_to_device(m), noise=(np.stack(u), np.stack(e1), np.stack(e2)), mode="pk")
    got = bfv.to_reference_order(s["pp"], ct.data).reshape(oct_.shape)
    assert np.array_equal(got, oct_)
    # decrypt on device == plaintext == oracle decrypt
    dm = _dev.to_numpy_u64(bfv.decrypt(s["pkp"], ct))
    assert np.array_equal(dm, m)
    assert np.array_equal(OB.decrypt(s["op"], s["okp"], got, s["ar"]), m)


def test_encrypt_sk_bit_exact_with_oracle_noise(setup):
    from paper_2403_11166_b200 import _dev, bfv

    s = setup
    N, L, P = s["N"], s["L"], 2
    op = s["op"]
    m = OR.SeededRng(7, 1).uniform_ring((P, N), OR.RingParams())
    oct_ = OB.encrypt_sk(op, s["okp"], m, OR.SeededRng(8, 0), s["ar"])
    g = OR.SeededRng(8, 0)
    a, e = [], []
    for _ in range(P):
        a.append(np.stack([g.uniform_mod((N,), q) for q in op.moduli]))
        e.append(g.cbd((N,)))
    ct = bfv.encrypt(s["pkp"], _dev.u64_to_device(m), noise=(np.stack(a), np.stack(e)), mode="sk")
    got = bfv.to_reference_order(s["pp"], ct.data).reshape(oct_.shape)
    assert np.array_equal(got, oct_)
    assert np.array_equal(_dev.to_numpy_u64(bfv.decrypt(s["pkp"], ct)), m)


@pytest.mark.parametrize("mode", ["pk", "sk"])
def test_device_randomness_roundtrip_and_ctpt(setup, mode):
    from paper_2403_11166_b200 import _dev, bfv, ring

    s = setup
    N, P = s["N"], 4
    m = OR.SeededRng(9, 2).uniform_ring((P, N), OR.RingParams())
    w = OR.SeededRng(9, 3).uniform_ring((1, N), OR.RingParams())
    ct = bfv.encrypt(s["pkp"], _dev.u64_to_device(m), ring.SeededRng(10, 0), mode=mode)
    assert np.array_equal(_dev.to_numpy_u64(bfv.decrypt(s["pkp"], ct)), m)
    prod = bfv.he_plain_mul(ct, _dev.u64_to_device(w))
    got = _dev.to_numpy_u64(bfv.decrypt(s["pkp"], prod))
    for i in range(P):
        assert np.array_equal(got[i], OK.negacyclic_mul_wrap(m[i].copy(), w[0].copy()) & T_MASK)
    assert bfv.noise_budget(s["pkp"], prod) > 0
    # two encryptions of the same message differ
    ct2 = bfv.encrypt(s["pkp"], _dev.u64_to_device(m), ring.SeededRng(10, 1), mode=mode)
    assert not np.array_equal(_dev.to_numpy_u32(ct.data), _dev.to_numpy_u32(ct2.data))


def test_split_encrypt_sk(setup):
    """Precomputed (a, -a s, e) + online add (pb_encrypt_sk_zero / _add):
    same a as pb_encrypt_sk under (key, nonce); the ciphertext equals
    pb_encrypt_sk_noise with that (a, e) bit for bit; dense and packed
    sources; decrypts to m; e is a small centred draw."""
    from paper_2403_11166_b200 import _dev, bfv, ring
    from paper_2403_11166_b200.poly_encoding import compact

    s = setup
    N, L, P = s["N"], s["L"], 5
    kp = s["pkp"]
    m = OR.SeededRng(12, 2).uniform_ring((P, N), OR.RingParams())
    md = _dev.u64_to_device(m)
    ref = bfv.encrypt(kp, md, ring.SeededRng(13, 0), mode="sk", nonce=77)
    ct, e = bfv.encrypt_zero(kp, P, ring.SeededRng(13, 0), nonce=77)
    assert np.array_equal(_dev.to_numpy_u32(ct.data[:, 1]), _dev.to_numpy_u32(ref.data[:, 1]))  # same a
    en = e.cpu().numpy()
    assert np.abs(en).max() <= 20 and abs(en.mean()) < 0.1 and 8.0 < en.var() < 12.0  # CBD(20): var 10
    a_ref = bfv.to_reference_order(s["pp"], ct.data[:, 1].contiguous()).reshape(P, L, N)
    want = bfv.encrypt(kp, md, noise=(a_ref, en), mode="sk")
    got = bfv.encrypt_add((ct, e), md)
    assert np.array_equal(_dev.to_numpy_u32(got.data), _dev.to_numpy_u32(want.data))
    assert np.array_equal(_dev.to_numpy_u64(bfv.decrypt(kp, got)), m)
    # packed source: poly p takes flat values at a ragged set of slots
    rs = np.random.default_rng(3)
    flat = OR.SeededRng(12, 3).uniform_ring((300,), OR.RingParams())
    src = np.full((P, N), -1, np.int64)
    for p in range(P):
        k = rs.integers(0, 120)
        src[p, rs.choice(N, size=k, replace=False)] = rs.integers(0, 300, size=k)
    pack = tuple(_dev.i32_to_device(a) for a in compact(src))
    dense = np.where(src >= 0, flat[np.maximum(src, 0)], 0).astype(np.uint64)
    fd = _dev.u64_to_device(flat)
    pre = bfv.encrypt_zero(kp, P, ring.SeededRng(14, 0), nonce=5)
    a_ref = bfv.to_reference_order(s["pp"], pre[0].data[:, 1].contiguous()).reshape(P, L, N)
    want = bfv.encrypt(kp, fd, noise=(a_ref, pre[1].cpu().numpy()), mode="sk", pack=pack)
    got = bfv.encrypt_add(pre, fd, pack=pack)
    assert np.array_equal(_dev.to_numpy_u32(got.data), _dev.to_numpy_u32(want.data))
    assert np.array_equal(_dev.to_numpy_u64(bfv.decrypt(kp, got)), dense)


def test_he_add_and_plain(setup):
    from paper_2403_11166_b200 import _dev, bfv, ring

    s = setup
    N = s["N"]
    a = OR.SeededRng(12, 0).uniform_ring((2, N), OR.RingParams())
    b = OR.SeededRng(12, 1).uniform_ring((2, N), OR.RingParams())
    ca = bfv.encrypt(s["pkp"], _dev.u64_to_device(a), ring.SeededRng(13, 0))
    cb = bfv.encrypt(s["pkp"], _dev.u64_to_device(b), ring.SeededRng(13, 1))
    assert np.array_equal(_dev.to_numpy_u64(bfv.decrypt(s["pkp"], bfv.he_add(ca, cb))), (a + b) & T_MASK)
    assert np.array_equal(_dev.to_numpy_u64(bfv.decrypt(s["pkp"], bfv.he_add(ca, cb, subtract=True))), (a - b) & T_MASK)
    assert np.array_equal(_dev.to_numpy_u64(bfv.decrypt(s["pkp"], bfv.he_add(ca, _dev.u64_to_device(b)))), (a + b) & T_MASK)
    z = bfv.he_add(ca, _dev.u64_to_device(a), subtract=True)  # Enc(m) - m -> 0
    assert not _dev.to_numpy_u64(bfv.decrypt(s["pkp"], z)).any()


def test_noise_budget_matches_oracle(setup):
    from paper_2403_11166_b200 import _dev, bfv, ring

    s = setup
    m = OR.SeededRng(14, 0).uniform_ring((1, s["N"]), OR.RingParams())
    ct = bfv.encrypt(s["pkp"], _dev.u64_to_device(m), ring.SeededRng(15, 0))
    k = bfv.to_reference_order(s["pp"], ct.data).reshape(1, 2, s["L"], s["N"])
    assert bfv.noise_budget(s["pkp"], ct) == OB.noise_budget(s["op"], s["okp"], k, s["ar"]) > 0


def test_decrypt_to_share_gather(setup):
    import torch

    from paper_2403_11166_b200 import _dev, _lib, bfv, ring
    from paper_2403_11166_b200.params import context

    s = setup
    N, P, U = s["N"], 3, 37
    m = OR.SeededRng(16, 0).uniform_ring((P, N), OR.RingParams())
    ct = bfv.encrypt(s["pkp"], _dev.u64_to_device(m), ring.SeededRng(17, 0))
    rng = np.random.default_rng(0)
    pos = np.stack([rng.choice(N, size=U, replace=False) for _ in range(P)]).astype(np.int32)
    pos[1, 5] = -1  # skipped slot
    dst = np.arange(P * U, dtype=np.int64).reshape(P, U)
    share = torch.zeros(P * U, dtype=torch.int64, device="cuda")
    scratch = _dev.empty_u32(P, s["L"], U)
    dpos, ddst = _dev.i32_to_device(pos), _dev.i64_to_device(dst)
    _lib.call("pb_decrypt_to_share", context(s["pp"]).handle, _dev.ptr(s["pkp"].sk_ntt), _dev.ptr(ct.data), P,
              _dev.ptr(dpos), _dev.ptr(ddst), U, _dev.ptr(share), _dev.ptr(scratch), _dev.stream())
    got = _dev.to_numpy_u64(share).reshape(P, U)
    for p in range(P):
        for u in range(U):
            want = 0 if pos[p, u] < 0 else m[p, pos[p, u]]
            assert got[p, u] == want


def test_encrypt_sk_launch_cap(setup):
    """Under a launch cap (background preparation) pb_encrypt_sk's CTAs take
    consecutive polynomial-major rows and draw each polynomial's noise once
    for all limbs: the ciphertext is bit-identical to the uncapped one."""
    from paper_2403_11166_b200 import _dev, _lib, bfv, ring

    s = setup
    N, P = s["N"], 5
    kp = s["pkp"]
    m = OR.SeededRng(12, 4).uniform_ring((P, N), OR.RingParams())
    md = _dev.u64_to_device(m)
    ref = _dev.to_numpy_u32(bfv.encrypt(kp, md, ring.SeededRng(14, 0), mode="sk", nonce=5).data)
    for cap in (1, 3, 8, 34):
        _lib.call("pb_set_launch_cap", cap)
        try:
            got = bfv.encrypt(kp, md, ring.SeededRng(14, 0), mode="sk", nonce=5)
        finally:
            _lib.call("pb_set_launch_cap", 0)
        assert np.array_equal(_dev.to_numpy_u32(got.data), ref), cap
    assert np.array_equal(_dev.to_numpy_u64(bfv.decrypt(kp, got)), m)


@pytest.mark.parametrize("mode", ["pk", "sk"])
def test_encrypt_without_rng_is_randomized(setup, mode):
    """SPEC:139-147's encrypt(pk, m) takes no rng: two default-argument
    encryptions of the same m differ (fresh entropy per call) and both decrypt to m."""
    import torch

    from paper_2403_11166_b200 import bfv

    N = setup["N"]
    m = torch.from_numpy((np.arange(2 * N, dtype=np.uint64) * 977 & T_MASK).view(np.int64)).cuda()
    c1 = bfv.encrypt(setup["pkp"], m, mode=mode)
    c2 = bfv.encrypt(setup["pkp"], m, mode=mode)
    assert not torch.equal(c1.data, c2.data)
    assert not torch.equal(c1.data[:, 1], c2.data[:, 1])
    for c in (c1, c2):
        assert torch.equal(bfv.decrypt(setup["pkp"], c), m.view(2, N))
