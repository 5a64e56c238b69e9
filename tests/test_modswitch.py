"""SPEC:196 response compaction (modulus switch dropping the last RNS limb).

The reference ships no implementation (OFF by default in SPEC), so the
oracle restates the textbook BFV modulus switch (oracle/bfv.py
mod_switch_drop).  GPU: the switched ciphertexts are bit-identical to the
oracle's switch of the oracle's own ciphertexts, decrypt to the original
plaintext under the kept key rows, still decrypt after a ct x pt product,
and their PBFV frames shrink by 1/L.
"""

import numpy as np
import pytest

from oracle import bfv as OB
from oracle import ring as OR
from oracle.params import make_params



@pytest.fixture(scope="module", params=[(2048, 8), (8192, 7), (4096, 4)])
def ms(request):
    from paper_2403_11166_b200 import _dev, bfv, ring
    from paper_2403_11166_b200.params import BfvParams

    N, L = request.param
    op, pp = make_params(N, L), BfvParams(N=N, L=L)
    ar = OB.Arith(op)
    okp = OB.keygen(op, OR.SeededRng(11, 0), ar)
    pkp = bfv.keygen(pp, ring.SeededRng(11, 0))
    P = 3
    m = OR.SeededRng(5, 1).uniform_ring((P, N), OR.RingParams())
    oct_ = OB.encrypt_pk(op, okp, m, OR.SeededRng(6, 0), ar)
    g = OR.SeededRng(6, 0)
    u, e1, e2 = [], [], []
    for _ in range(P):
        u.append(g.ternary((N,)))
        e1.append(g.cbd((N,)))
        e2.append(g.cbd((N,)))
    ct = bfv.encrypt(pkp, _dev.u64_to_device(m), noise=(np.stack(u), np.stack(e1), np.stack(e2)), mode="pk")
    return dict(N=N, L=L, op=op, pp=pp, ct=ct, oct=np.asarray(oct_, dtype=np.uint64), pkp=pkp, m=m)


@pytest.mark.gpu
def test_mod_switch_bit_exact_vs_oracle(ms):
    from paper_2403_11166_b200 import bfv

    lo_o, want = OB.mod_switch_drop(ms["op"], ms["oct"])
    got = bfv.mod_switch_drop(ms["ct"])
    assert got.params.L == ms["L"] - 1 and got.params.moduli == tuple(lo_o.moduli)
    assert np.array_equal(bfv.to_reference_order(got.params, got.data), want)


@pytest.mark.gpu
def test_mod_switch_decrypts(ms):
    from paper_2403_11166_b200 import _dev, bfv

    got = bfv.mod_switch_drop(ms["ct"])
    assert np.array_equal(_dev.to_numpy_u64(bfv.decrypt(bfv.drop_keys(ms["pkp"]), got)), ms["m"])


@pytest.mark.gpu
def test_mod_switch_after_plain_mul(ms):
    """The protocol's use: a masked ct x pt reply, compacted, still decrypts."""
    from paper_2403_11166_b200 import _dev, bfv, wire

    N, t = ms["N"], 1 << 59
    w = OR.SeededRng(9, 0).uniform_ring((1, N), OR.RingParams())
    w = (w % np.uint64(3)).astype(np.uint64)  # small weights keep the noise far from the limit
    prod = bfv.he_plain_mul(ms["ct"], bfv.encode_plain(ms["pp"], _dev.u64_to_device(w)))
    got = bfv.mod_switch_drop(prod)
    want = _dev.to_numpy_u64(bfv.decrypt(ms["pkp"], prod))
    assert np.array_equal(_dev.to_numpy_u64(bfv.decrypt(bfv.drop_keys(ms["pkp"]), got)), want)
    L = ms["L"]
    assert wire.serialize(got).numel() == 3 * (12 + 2 * (L - 1) * N * 8)
    del t


@pytest.mark.parametrize("N,L", [(2048, 8), (4096, 4)])
def test_oracle_mod_switch_decrypts(N, L):
    """CPU: pins the oracle's restatement — the switched ciphertext decrypts
    to the same plaintext under the kept key rows (no GPU involved)."""
    op = make_params(N, L)
    ar = OB.Arith(op)
    kp = OB.keygen(op, OR.SeededRng(1, 0), ar)
    m = OR.SeededRng(5, 1).uniform_ring((2, N), OR.RingParams())
    ct = OB.encrypt_pk(op, kp, m, OR.SeededRng(6, 0), ar)
    lo, c2 = OB.mod_switch_drop(op, ct)
    kp_lo = OB.KeyPair(kp.sk_coeff, np.ascontiguousarray(kp.sk_ntt[: lo.L]), np.ascontiguousarray(kp.pk[:, : lo.L]))
    assert np.array_equal(OB.decrypt(lo, kp_lo, c2, OB.Arith(lo)), m)
