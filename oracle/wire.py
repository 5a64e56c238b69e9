"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the PBFV wire format ("Ciphertext wire format
(bit-exact)") and of the census arithmetic built on it (SPEC.md:680-688,
example "bytes = frames x (header + 2*L*N*8)").

The reference ships no serializer (SPEC's ``bfv`` module is absent from
/root/reference/pkg), so this row is parity UNPINNED by
reference code: the oracle is pinned by the SPEC text itself — header field
order and widths, little-endian u64 rows, c0 then c1 — and the checks in
tests/test_wire.py restate the SPEC census example.

Conventions fixed here and shared bit-for-bit by pb_wire_serialize:
  * header = struct "<4sHIBB": b"PBFV", version 1, N, L, form (12 bytes, packed);
  * form 0 = coefficient rows, 1 = NTT rows in K:ntt_forward's bit-reversed order;
  * payload = n_polys x L x N residues as little-endian u64 (c0 rows, then c1).
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC = b"PBFV"
VERSION = 1
HEADER = struct.Struct("<4sHIBB")
FORM_COEFF, FORM_NTT = 0, 1


class WireError(ValueError):
    """Malformed frame; ``kind`` is one of header / params / form / residue."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


def frame_bytes(N: int, L: int, n_polys: int) -> int:
    """SPEC:203 frame size; SPEC:680-688 census counts frames x this."""
    return HEADER.size + n_polys * L * N * 8


def serialize(rows, N: int, L: int, form: int) -> bytes:
    """rows: [P][n_polys][L][N] residues (reference order for form=NTT) -> P frames."""
    a = np.asarray(rows)
    assert a.ndim == 4 and a.shape[2:] == (L, N), a.shape
    hdr = HEADER.pack(MAGIC, VERSION, N, L, form)
    out = bytearray()
    for p in range(a.shape[0]):
        out += hdr
        out += a[p].astype("<u8").tobytes()
    return bytes(out)


def deserialize(buf: bytes, P: int, n_polys: int, N: int, L: int, form: int, q) -> np.ndarray:
    """P frames -> [P][n_polys][L][N] uint64, validating header and residue range."""
    fb = frame_bytes(N, L, n_polys)
    if len(buf) < P * fb:
        raise WireError("header", f"{len(buf)} bytes for {P} frames of {fb}")
    out = np.empty((P, n_polys, L, N), dtype=np.uint64)
    qv = np.asarray(q, dtype=np.uint64).reshape(1, L, 1)
    for p in range(P):
        f = buf[p * fb:(p + 1) * fb]
        magic, ver, n, l, fm = HEADER.unpack_from(f, 0)
        if magic != MAGIC or ver != VERSION:
            raise WireError("header", f"bad magic/version {magic!r}/{ver}")
        if n != N or l != L:
            raise WireError("params", f"frame N={n}, L={l}; expected N={N}, L={L}")
        if fm != form:
            raise WireError("form", f"frame form {fm}; expected {form}")
        rows = np.frombuffer(f, dtype="<u8", offset=HEADER.size).reshape(n_polys, L, N)
        if np.any(rows >= qv):
            raise WireError("residue", "residue >= q_i")
        out[p] = rows
    return out
