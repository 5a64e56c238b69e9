"""ncu driver: pb_decrypt_to_share at the MLP step's FC-784 forward (32 cts)
and layer-0 weight-gradient (50 cts, 2041 useful slots each) shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib, bfv  # noqa: E402
from paper_2403_11166_b200.linear_protocols import _Shard  # noqa: E402
from paper_2403_11166_b200.params import BfvParams, context  # noqa: E402
from paper_2403_11166_b200.poly_encoding import MatmulGeometry, plan_matmul  # noqa: E402
from paper_2403_11166_b200.ring import SeededRng  # noqa: E402

p = BfvParams()
kp = bfv.keygen(p, SeededRng(1, 0))
h = context(p).handle
for g, vs in ((MatmulGeometry(784, 128, 64), None), (MatmulGeometry(64, 128, 784), (1, 64))):
    plan = plan_matmul(g, p.N, vs, None, None)
    sh = _Shard(plan, 0, 1)
    ct = torch.randint(0, p.moduli[-1], (sh.n_out, 2, p.L, p.N), dtype=torch.int32, device="cuda")
    share = _dev.empty_u64(g.n_o * g.B)
    scratch = _dev.empty_u32(sh.n_out, p.L, sh.U)
    for _ in range(3):
        _lib.call("pb_decrypt_to_share", h, _dev.ptr(kp.sk_ntt), _dev.ptr(ct), sh.n_out, _dev.ptr(sh.out_pos),
                  _dev.ptr(sh.out_dst), sh.U, _dev.ptr(share), _dev.ptr(scratch), _dev.stream())
    torch.cuda.synchronize()
    print("n_out", sh.n_out, "U", sh.U)
