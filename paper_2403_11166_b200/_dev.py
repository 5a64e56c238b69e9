"""Device plumbing: torch CUDA tensors as raw buffers for the C ABI.

PyTorch supplies device memory, the caching allocator and streams; every
arithmetic step is a call into libpencil_b200.so.  Residues are stored as
torch.int32 (bit pattern of u32), Z_{2^ell} elements as torch.int64 (bit
pattern of u64).
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import DeviceError, ShapeError

U32 = torch.int32  # storage dtype for uint32 residues
U64 = torch.int64  # storage dtype for uint64 ring elements


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("a CUDA device is required (the engine has no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def device() -> torch.device:
    return require_cuda()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise DeviceError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ShapeError("expected a contiguous tensor")
    return t.data_ptr()


def empty_u32(*shape) -> torch.Tensor:
    return torch.empty(shape, dtype=U32, device=device())


def empty_u64(*shape) -> torch.Tensor:
    return torch.empty(shape, dtype=U64, device=device())


def zeros_u64(*shape) -> torch.Tensor:
    return torch.zeros(shape, dtype=U64, device=device())


def u64_to_device(a) -> torch.Tensor:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    return torch.from_numpy(a.view(np.int64)).to(device())


def u32_to_device(a) -> torch.Tensor:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint32))
    return torch.from_numpy(a.view(np.int32)).to(device())


def i64_to_device(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.int64))).to(device())


def i32_to_device(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.int32))).to(device())


def to_numpy_u64(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)


def to_numpy_u32(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint32)
