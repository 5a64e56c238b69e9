"""Tiny driver for ncu: a few NTT launches over 1 GiB of residues (N=8192, L=7)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib  # noqa: E402
from paper_2403_11166_b200.params import BfvParams, context  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
p = BfvParams(N=N, L=7)
ctx = context(p)
rows = (1 << 30) // (4 * N)
x = torch.randint(0, p.moduli[-1], (rows, N), dtype=torch.int32, device="cuda")
for _ in range(2):
    _lib.call("pb_ntt_forward", ctx.handle, x.data_ptr(), rows, None, _dev.stream())
    _lib.call("pb_ntt_inverse", ctx.handle, x.data_ptr(), rows, None, _dev.stream())
torch.cuda.synchronize()
print("ok")
