"""ncu driver: the ct x pt MAC at the conv-like (B_ct=64, O_pt=13, K=16) and FC-like (K=1) shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib  # noqa: E402
from paper_2403_11166_b200.params import BfvParams, context  # noqa: E402

p = BfvParams()
ctx = context(p)
L, N = p.L, p.N
for nB, nO, nI in ((64, 13, 16), (64, 13, 1), (8, 8, 13)):
    ct = torch.randint(0, p.moduli[-1], (nB * nI, 2, L, N), dtype=torch.int32, device="cuda")
    pt = torch.randint(0, p.moduli[-1], (nO * nI, L, N), dtype=torch.int32, device="cuda")
    out = torch.zeros((nB * nO, 2, L, N), dtype=torch.int32, device="cuda")
    for _ in range(2):
        _lib.call("pb_ctpt_mac_tiled", ctx.handle, ct.data_ptr(), pt.data_ptr(), None, None, nB, nO, nI,
                  out.data_ptr(), _dev.stream())
torch.cuda.synchronize()
print("ok")
