"""PBFV wire format and its census.

CPU: the oracle's frame layout against the SPEC text (header field order and
widths, little-endian u64 rows, c0 then c1), its round trip and every error
class.  GPU: pb_wire_serialize frames byte-identical to the oracle's frames of
the same ciphertexts (NTT form in the reference order, and coefficient form
against the oracle's own inverse NTT), into pinned host memory and into HBM,
at odd frame counts so every 4-byte frame alignment is hit; deserialize round
trips bit-exactly and raises the reference's error classes.
"""

import struct

import numpy as np
import pytest

from oracle import wire as OW


def _rand_rows(rng, P, n_polys, L, N, q):
    return np.stack([rng.integers(0, q[l], size=(P, n_polys, N), dtype=np.uint64) for l in range(L)], axis=2)


def test_oracle_header_is_spec_layout():
    b = OW.serialize(np.zeros((1, 2, 3, 16), np.uint64), 16, 3, OW.FORM_NTT)
    assert b[:12] == b"PBFV" + struct.pack("<H", 1) + struct.pack("<I", 16) + bytes([3, 1])
    assert len(b) == 12 + 2 * 3 * 16 * 8


def test_oracle_census_matches_spec_example():
    # one Alg.-1 FC forward (N=8192, L=3) -> bytes = frames x (header + 2*L*N*8)
    assert OW.frame_bytes(8192, 3, 2) == 12 + 2 * 3 * 8192 * 8
    assert OW.frame_bytes(8192, 7, 1) == 12 + 7 * 8192 * 8


def test_oracle_roundtrip_and_rows_little_endian():
    rng = np.random.default_rng(1)
    q = [97, 193, 257]
    a = _rand_rows(rng, 3, 2, 3, 16, q)
    b = OW.serialize(a, 16, 3, OW.FORM_COEFF)
    assert np.array_equal(OW.deserialize(b, 3, 2, 16, 3, OW.FORM_COEFF, q), a)
    fb = OW.frame_bytes(16, 3, 2)
    # frame 1, c1, limb 2, coefficient 5
    off = fb + 12 + ((1 * 3 + 2) * 16 + 5) * 8
    assert struct.unpack_from("<Q", b, off)[0] == a[1, 1, 2, 5]


@pytest.mark.parametrize("kind", ["header", "params", "form", "residue"])
def test_oracle_rejects(kind):
    q = [97, 193]
    a = np.ones((2, 2, 2, 8), np.uint64)
    b = bytearray(OW.serialize(a, 8, 2, OW.FORM_NTT))
    fb = OW.frame_bytes(8, 2, 2)
    if kind == "header":
        b[fb] = ord("X")
    elif kind == "params":
        b[fb + 10] = 3
    elif kind == "form":
        b[11] = 0
    else:
        struct.pack_into("<Q", b, fb + 12 + 8 * 8 + 8, 193)  # c0 limb 1 coefficient 1 = q_1
    with pytest.raises(OW.WireError) as ei:
        OW.deserialize(bytes(b), 2, 2, 8, 2, OW.FORM_NTT, q)
    assert ei.value.kind == kind


# ------------------------------------------------------------------- GPU --

@pytest.fixture(scope="module", params=[(2048, 8), (8192, 7)])
def gsetup(request):
    from oracle import bfv as OB
    from oracle import ring as OR
    from oracle.params import make_params
    from paper_2403_11166_b200 import _dev, bfv, ring
    from paper_2403_11166_b200.params import BfvParams

    N, L = request.param
    op, pp = make_params(N, L), BfvParams(N=N, L=L)
    ar = OB.Arith(op)
    okp = OB.keygen(op, OR.SeededRng(11, 0), ar)
    pkp = bfv.keygen(pp, ring.SeededRng(11, 0))
    P = 5
    m = OR.SeededRng(5, 1).uniform_ring((P, N), OR.RingParams())
    oct_ = OB.encrypt_pk(op, okp, m, OR.SeededRng(6, 0), ar)
    g = OR.SeededRng(6, 0)
    u, e1, e2 = [], [], []
    for _ in range(P):
        u.append(g.ternary((N,)))
        e1.append(g.cbd((N,)))
        e2.append(g.cbd((N,)))
    ct = bfv.encrypt(pkp, _dev.u64_to_device(m), noise=(np.stack(u), np.stack(e1), np.stack(e2)), mode="pk")
    return dict(N=N, L=L, op=op, pp=pp, ar=ar, ct=ct, oct=np.asarray(oct_, dtype=np.uint64), pkp=pkp, m=m)


@pytest.mark.gpu
def test_gpu_serialize_ntt_bit_exact_vs_oracle(gsetup):
    import torch

    from paper_2403_11166_b200 import wire

    s = gsetup
    want = OW.serialize(s["oct"], s["N"], s["L"], OW.FORM_NTT)
    host = wire.serialize(s["ct"])
    assert host.is_pinned() and host.numel() == len(want) == 5 * wire.frame_bytes(s["pp"])
    assert bytes(host.numpy()) == want
    zc = torch.empty(len(want), dtype=torch.uint8, pin_memory=True)
    assert bytes(wire.serialize(s["ct"], out=zc, stage=False).numpy()) == want  # kernel stores to host
    dev = torch.empty(len(want) + 4, dtype=torch.uint8, device="cuda")
    got = wire.serialize(s["ct"], out=dev[4:])  # frame base 4 mod 16: the other alignment class
    assert bytes(got.cpu().numpy()) == want


@pytest.mark.gpu
def test_gpu_serialize_coeff_bit_exact_vs_oracle(gsetup):
    from paper_2403_11166_b200 import bfv, wire

    s = gsetup
    P, L, N = 5, s["L"], s["N"]
    coeff = s["ar"].ntt_inv(s["oct"].copy().reshape(P * 2, L, N)).reshape(P, 2, L, N)
    want = OW.serialize(coeff, N, L, OW.FORM_COEFF)
    assert bytes(wire.serialize(s["ct"], form=bfv.COEFF).numpy()) == want


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["ntt", "coeff"])
def test_gpu_roundtrip_ct_and_decrypt(gsetup, form):
    import torch

    from paper_2403_11166_b200 import _dev, bfv, wire

    s = gsetup
    buf = wire.serialize(s["ct"], form=form)
    back = wire.deserialize(s["pp"], buf, 5, form=form)
    assert torch.equal(back.data, s["ct"].data)
    assert np.array_equal(_dev.to_numpy_u64(bfv.decrypt(s["pkp"], back)), s["m"])
    back_dev = wire.deserialize(s["pp"], buf.cuda(), 5, form=form)
    assert torch.equal(back_dev.data, s["ct"].data)
    back_zc = wire.deserialize(s["pp"], buf, 5, form=form, stage=False)  # kernel loads from host
    assert torch.equal(back_zc.data, s["ct"].data)
    off = torch.empty(buf.numel() + 4, dtype=torch.uint8, device="cuda")
    off[4:].copy_(buf)
    assert torch.equal(wire.deserialize(s["pp"], off[4:], 5, form=form).data, s["ct"].data)


@pytest.mark.gpu
def test_gpu_roundtrip_plaintext(gsetup):
    import torch

    from paper_2403_11166_b200 import _dev, bfv, wire

    s = gsetup
    pt = bfv.encode_plain(s["pp"], _dev.u64_to_device(s["m"][:3]))
    buf = wire.serialize(pt, s["pp"])
    assert buf.numel() == 3 * wire.frame_bytes(s["pp"], 1)
    back = wire.deserialize(s["pp"], buf, 3, kind="pt")
    assert torch.equal(back.data, pt.data)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["header", "params", "form", "residue"])
def test_gpu_deserialize_rejects(gsetup, kind):
    from paper_2403_11166_b200 import errors, wire

    s = gsetup
    buf = wire.serialize(s["ct"]).clone()
    fb = wire.frame_bytes(s["pp"])
    if kind == "header":
        buf[2 * fb + 1] = ord("X")
    elif kind == "params":
        buf[3 * fb + 10] = s["L"] - 1
    elif kind == "form":
        buf[4 * fb + 11] = 0
    else:
        buf[fb + 12 + 8 * 100 + 4] = 1  # high word of a residue (frame 1: row at 0 mod 8)
    exc = {"header": errors.PencilError, "params": errors.ParamsError, "form": errors.FormError,
           "residue": errors.EncodeRangeError}[kind]
    with pytest.raises(exc):
        wire.deserialize(s["pp"], buf, 5)
    with pytest.raises(exc):
        wire.deserialize(s["pp"], buf, 5, stage=False)


@pytest.mark.gpu
def test_gpu_census_counts_wire_bytes(gsetup):
    from paper_2403_11166_b200 import wire

    s = gsetup
    assert s["ct"].nbytes_wire() == wire.serialize(s["ct"]).numel()


@pytest.mark.gpu
@pytest.mark.parametrize("frame", [0, 1, 2, 3])
def test_gpu_deserialize_range_every_alignment(gsetup, frame):
    """A residue == q_l (low word) or a set high word is caught in rows at
    both 8-byte alignments (even / odd frames) and in the last high word."""
    from paper_2403_11166_b200 import errors, wire

    s = gsetup
    fb, N, L = wire.frame_bytes(s["pp"]), s["N"], s["L"]
    base = wire.serialize(s["ct"]).clone()
    last = frame * fb + 12 + (2 * L * N - 1) * 8  # c1, last limb, last coefficient
    for off, val in [(last, int(s["pp"].moduli[L - 1])), (last + 4, 1)]:
        buf = base.clone()
        buf[off:off + 4] = torch_u32(val)
        with pytest.raises(errors.EncodeRangeError):
            wire.deserialize(s["pp"], buf, 5)


def torch_u32(v):
    import torch

    return torch.tensor(list(int(v).to_bytes(4, "little")), dtype=torch.uint8)
