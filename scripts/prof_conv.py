"""ncu driver: the local ring-conv operators at CIFAR conv2 size (B=64, 64->64, 5x5, 16x16, pad 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib  # noqa: E402
from paper_2403_11166_b200.linear_protocols import _ring_conv  # noqa: E402

B, ci, co, H, W, s, p, st = 64, 64, 64, 16, 16, 5, 2, 1
rng = np.random.default_rng(0)
x = _dev.u64_to_device(rng.integers(0, 1 << 59, size=(B, ci, H, W), dtype=np.uint64))
w = _dev.u64_to_device(rng.integers(0, 1 << 59, size=(co, ci, s, s), dtype=np.uint64))
gy = _dev.u64_to_device(rng.integers(0, 1 << 59, size=(B, co, H, W), dtype=np.uint64))
args = (B, ci, co, H, W, s, p, st, 59)
for _ in range(2):
    _ring_conv(_lib.CONV_FWD, x, w, *args, (B, co, H, W))
    _ring_conv(_lib.CONV_BWDX, gy, w, *args, (B, ci, H, W))
    _ring_conv(_lib.CONV_GRADW, x, gy, *args, (co, ci, s, s))
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
ev[0].record()
_ring_conv(_lib.CONV_FWD, x, w, *args, (B, co, H, W))
ev[1].record()
_ring_conv(_lib.CONV_BWDX, gy, w, *args, (B, ci, H, W))
ev[2].record()
_ring_conv(_lib.CONV_GRADW, x, gy, *args, (co, ci, s, s))
ev[3].record()
torch.cuda.synchronize()
macs = B * co * ci * s * s * H * W
print("fwd/bwdx/gradw ms", [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(3)], "MAC/s",
      [f"{macs / (ev[i].elapsed_time(ev[i + 1]) / 1e3):.3e}" for i in range(3)])
# per-operator timing loop (10 reps each) for steadier numbers
for kind, shp, xa, xb in ((_lib.CONV_FWD, (B, co, H, W), x, w), (_lib.CONV_BWDX, (B, ci, H, W), gy, w),
                          (_lib.CONV_GRADW, (co, ci, s, s), x, gy)):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(10):
        _ring_conv(kind, xa, xb, *args, shp)
    s1.record()
    torch.cuda.synchronize()
    print("kind", kind, "ms", round(s0.elapsed_time(s1) / 10, 3))
