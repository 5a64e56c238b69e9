"""ncu driver for the round-2 kernels (one call each, run a few times):
  tc     tcgen05 ring GEMM: CIFAR conv2 forward (B=64, 64->64, 5x5, 16x16) and a 4096^3 matmul
  nl     OT non-linear ReLU + truncation over the CIFAR conv1 activations (64 x 64 x 32 x 32)
  ntt32k the two-CTA cluster NTT at N=32768 (forward + inverse over 1 GiB)
  maskmac the fused mask NTT + K=1 MAC (B_ct=64, O_pt=13)
usage: python scripts/prof_round2.py <what>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib  # noqa: E402
from paper_2403_11166_b200.params import BfvParams, context  # noqa: E402

what = sys.argv[1]
st = _dev.stream()
rng = np.random.default_rng(0)
if what == "tc":
    B, ci, co, H, s, p = 64, 64, 64, 16, 5, 2
    x = _dev.u64_to_device(rng.integers(0, 1 << 59, size=(B, ci, H, H), dtype=np.uint64))
    w = _dev.u64_to_device(rng.integers(0, 1 << 59, size=(co, ci, s, s), dtype=np.uint64))
    y = _dev.empty_u64(B, co, H, H)
    a = _dev.u64_to_device(rng.integers(0, 1 << 59, size=(4096, 4096), dtype=np.uint64))
    c = _dev.empty_u64(4096, 4096)
    for _ in range(2):
        _lib.call("pb_ring_conv_ex", _lib.CONV_FWD, _dev.ptr(x), _dev.ptr(w), B, ci, co, H, H, s, p, 1, 59, _dev.ptr(y),
                  _lib.BACKEND_TENSOR, st)
        _lib.call("pb_ring_matmul_ex", _dev.ptr(a), _dev.ptr(a), 4096, 4096, 4096, 0, 0, 59, _dev.ptr(c),
                  _lib.BACKEND_TENSOR, st)
elif what == "nl":
    n = 64 * 64 * 32 * 32
    x0 = _dev.u64_to_device(rng.integers(0, 1 << 59, size=n, dtype=np.uint64))
    x1 = _dev.u64_to_device(rng.integers(0, 1 << 59, size=n, dtype=np.uint64))
    y0, y1 = _dev.empty_u64(n), _dev.empty_u64(n)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for i in range(2):
        _lib.call("pb_nl_op", _lib.NL_RELU_TRUNC, _dev.ptr(x0), _dev.ptr(x1), n, 59, 25, None, d.data_ptr(), 7, None,
                  1_000_000 + i, 0, _dev.ptr(y0), _dev.ptr(y1), st)
elif what == "ntt32k":
    p = BfvParams(N=32768, L=8)
    ctx = context(p)
    rows = (1 << 30) // (4 * 32768)
    x = torch.randint(0, p.moduli[-1], (rows, 32768), dtype=torch.int32, device="cuda")
    for _ in range(2):
        _lib.call("pb_ntt_forward", ctx.handle, x.data_ptr(), rows, None, st)
        _lib.call("pb_ntt_inverse", ctx.handle, x.data_ptr(), rows, None, st)
elif what == "maskmac":
    p = BfvParams()
    ctx = context(p)
    L, N, nB, nO, U = p.L, p.N, 64, 13, 128
    ct = torch.randint(0, p.moduli[-1], (nB, 2, L, N), dtype=torch.int32, device="cuda")
    pt = torch.randint(0, p.moduli[-1], (nO, L, N), dtype=torch.int32, device="cuda")
    o = torch.empty((nB * nO, 2, L, N), dtype=torch.int32, device="cuda")
    pos = (torch.arange(U, dtype=torch.int32, device="cuda") * 61 % N).repeat(nB * nO, 1).contiguous()
    dst = torch.arange(nB * nO * U, dtype=torch.int64, device="cuda")
    mask = torch.randint(0, 1 << 59, (nB * nO * U,), dtype=torch.int64, device="cuda")
    for _ in range(2):
        _lib.call("pb_mask_mac", ctx.handle, ct.data_ptr(), pt.data_ptr(), None, None, nB, nO, 1, pos.data_ptr(),
                  dst.data_ptr(), U, mask.data_ptr(), 1, 7, None, o.data_ptr(), st)
torch.cuda.synchronize()
print("ok")
