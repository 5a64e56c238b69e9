"""ncu driver: pb_encrypt_sk (k_enc_noise + k_encrypt_sk) at the MLP step's
FC-784 forward input size (the plan's 100 input polynomials), twice."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib, bfv  # noqa: E402
from paper_2403_11166_b200.linear_protocols import _pk, _Shard  # noqa: E402
from paper_2403_11166_b200.params import BfvParams, context  # noqa: E402
from paper_2403_11166_b200.poly_encoding import MatmulGeometry, plan_matmul  # noqa: E402
from paper_2403_11166_b200.ring import SeededRng  # noqa: E402

p = BfvParams()
kp = bfv.keygen(p, SeededRng(1, 0))
h = context(p).handle
plan = plan_matmul(MatmulGeometry(784, 128, 64), p.N)
sh = _Shard(plan, 0, 1)
vals = _dev.u64_to_device(np.random.default_rng(0).integers(0, 1 << 59, size=784 * 64, dtype=np.uint64))
ct = _dev.empty_u32(sh.n_in, 2, p.L, p.N)
for i in range(2):
    _lib.call("pb_encrypt_sk", h, _dev.ptr(kp.sk_ntt), _dev.ptr(kp.sk_sh), _dev.ptr(vals), *_pk(sh.in_pack), sh.n_in, 5 + i, None, 0,
              _dev.ptr(ct), _dev.stream())
torch.cuda.synchronize()
print("ok", sh.n_in)
