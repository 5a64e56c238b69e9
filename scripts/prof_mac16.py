"""ncu driver: the tiled ct x pt MAC (k_mac_ws) at the conv-like shape B_ct=64, O_pt=13, K=16, twice."""
import os, sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2403_11166_b200 import _dev, _lib
from paper_2403_11166_b200.params import BfvParams, context
p = BfvParams(); ctx = context(p); L, N = p.L, p.N
nB, nO, nI = 64, 13, 16
ct = torch.randint(0, p.moduli[-1], (nB * nI, 2, L, N), dtype=torch.int32, device="cuda")
pt = torch.randint(0, p.moduli[-1], (nO * nI, L, N), dtype=torch.int32, device="cuda")
out = torch.zeros((nB * nO, 2, L, N), dtype=torch.int32, device="cuda")
for _ in range(2):
    _lib.call("pb_ctpt_mac_tiled", ctx.handle, ct.data_ptr(), pt.data_ptr(), None, None, nB, nO, nI, out.data_ptr(), _dev.stream())
torch.cuda.synchronize(); print("ok")
