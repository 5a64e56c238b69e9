"""PBFV wire format — serialize / deserialize ciphertexts and
plaintext polynomials at the transport boundary, on the device.

SPEC:194 keeps ciphertexts in NTT form internally and converts "at
encode/serialize boundaries"; the frame payload is what the two-party census
counts (bytes = frames x (header + 2 L N 8) per ciphertext).

``serialize`` runs one kernel (pb_wire_serialize): the device-order ->
reference-order conversion, the u32 -> little-endian u64 widening and the
headers in one pass over HBM; a host destination (pinned, the default) is
then filled by the copy engine, or — ``stage=False`` — by the kernel's own
stores over the host link.  Pass ``out=`` a CUDA uint8 tensor to keep the
frames in HBM.
``deserialize`` validates every header and residue on the device
(pb_wire_deserialize) and raises the reference's error classes (E:4-41).
Coefficient-form frames (``form=COEFF``) go through the engine's inverse /
forward NTT on either side.
"""

from __future__ import annotations

import torch

from . import _dev, _lib
from .bfv import COEFF, NTT, Ciphertext, RnsPoly
from .errors import EncodeRangeError, FormError, ParamsError, PencilError, ShapeError
from .params import BfvParams, context

WIRE_VERSION = 1
HEADER_BYTES = 12
_FORM = {COEFF: 0, NTT: 1}
BAD_HEADER, BAD_PARAMS, BAD_FORM, BAD_RESIDUE = 1, 2, 4, 8


def frame_bytes(params: BfvParams, n_polys: int = 2) -> int:
    """Bytes of one PBFV frame: 2 polynomials per ciphertext, 1 per plaintext."""
    return HEADER_BYTES + n_polys * params.L * params.N * 8


def _rows(obj, params):
    if isinstance(obj, Ciphertext):
        return obj.data, obj.params, 2, NTT
    if isinstance(obj, RnsPoly):
        if params is None:
            raise ParamsError("serializing an RnsPoly needs params")
        d = obj.data.reshape(-1, params.L, params.N)
        return d, params, 1, obj.form
    raise ShapeError(f"cannot serialize {type(obj).__name__}")


def serialize(obj, params: BfvParams | None = None, *, form: str = NTT, out: torch.Tensor | None = None,
              stage: bool = True) -> torch.Tensor:
    """Ciphertext [P,2,L,N] / RnsPoly [P,L,N] -> P frames in a uint8 tensor
    (pinned host memory unless ``out`` is given).  ``stage=False`` lets the
    kernel store into a host ``out`` directly (zero-copy over the link)."""
    data, params, n_polys, have = _rows(obj, params)
    if form not in _FORM:
        raise FormError(f"unknown wire form {form!r}")
    data = data.contiguous()
    P = data.numel() // (n_polys * params.L * params.N)
    if have != form:  # convert on a scratch copy (at the boundary)
        data = data.clone()
        fn = "pb_ntt_inverse" if form == COEFF else "pb_ntt_forward"
        _lib.call(fn, context(params).handle, _dev.ptr(data), data.numel() // params.N, None, _dev.stream())
    nbytes = P * frame_bytes(params, n_polys)
    if out is None:
        out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    elif out.numel() < nbytes or out.dtype != torch.uint8:
        raise ShapeError(f"wire buffer holds {out.numel()} bytes, {P} frames need {nbytes}")
    if not out.is_cuda and not stage and not out.is_pinned():
        # the kernel would store straight into pageable memory: an illegal address
        raise ShapeError("serialize(stage=False) needs a CUDA or pinned host `out`")
    # A host destination is staged in HBM and moved by the copy engine: on
    # B200 the DMA beats the kernel's own zero-copy stores over the host link
    # (profiles/r01_wire_bench.jsonl: 54.6 vs 50.3 GB/s of frames).
    dst = out if out.is_cuda or not stage else torch.empty(nbytes, dtype=torch.uint8, device=_dev.device())
    _lib.call("pb_wire_serialize", context(params).handle, _dev.ptr(data), P, n_polys, _FORM[form],
              dst.data_ptr(), _dev.stream())
    if not out.is_cuda:
        if dst is not out:
            out[:nbytes].copy_(dst, non_blocking=True)
        torch.cuda.current_stream().synchronize()  # frames are host-visible on return
    return out[:nbytes]


def deserialize(params: BfvParams, buf: torch.Tensor, count: int, *, kind: str = "ct", form: str = NTT,
                stage: bool = True):
    """``count`` frames (uint8 tensor, pinned host or CUDA) -> Ciphertext or
    RnsPoly in NTT form, device order."""
    n_polys = {"ct": 2, "pt": 1}[kind]
    if form not in _FORM:
        raise FormError(f"unknown wire form {form!r}")
    nbytes = count * frame_bytes(params, n_polys)
    if buf.dtype != torch.uint8 or buf.numel() < nbytes:
        raise ShapeError(f"{buf.numel()} wire bytes for {count} frames of {frame_bytes(params, n_polys)}")
    if not buf.is_cuda:
        if stage:  # the copy engine brings the frames into HBM (see serialize)
            buf = buf[:nbytes].to(_dev.device(), non_blocking=buf.is_pinned())
        elif not buf.is_pinned():
            buf = buf.pin_memory()
    data = _dev.empty_u32(count, n_polys, params.L, params.N) if kind == "ct" else _dev.empty_u32(count, params.L, params.N)
    bad = torch.empty(1, dtype=torch.int32, device=_dev.device())
    _lib.call("pb_wire_deserialize", context(params).handle, buf.data_ptr(), count, n_polys, _FORM[form],
              _dev.ptr(data), _dev.ptr(bad), _dev.stream())
    flags = int(bad.item())
    if flags & BAD_HEADER:
        raise PencilError("PBFV frame: bad magic or version")
    if flags & BAD_PARAMS:
        raise ParamsError("PBFV frame: N / L differ from the session parameters")
    if flags & BAD_FORM:
        raise FormError(f"PBFV frame: form is not {form}")
    if flags & BAD_RESIDUE:
        raise EncodeRangeError("PBFV frame: residue >= q_i or high word set")
    if form == COEFF:
        _lib.call("pb_ntt_forward", context(params).handle, _dev.ptr(data), data.numel() // params.N, None,
                  _dev.stream())
    return Ciphertext(data, params) if kind == "ct" else RnsPoly(data, NTT)
