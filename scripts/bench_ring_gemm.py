"""Ring-GEMM backends side by side (CUDA events, warm, best of 5): the CIFAR
CNN's local-term convolutions at batch 64 and large FC-style matmuls, each
on the CUDA-core u64 kernels and on the tcgen05 int8 tensor-core path.
Prints one JSON line per (operator, backend) with u64 MAC/s."""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_11166_b200 import _dev as D  # noqa: E402
from paper_2403_11166_b200 import _lib  # noqa: E402

CONVS = {  # name: B, c_i, c_o, H, W, s, pad, stride (oracle/nn.py MODELS["cifar_cnn"], B = 64)
    "cifar_conv1": (64, 3, 64, 32, 32, 5, 2, 1), "cifar_conv2": (64, 64, 64, 16, 16, 5, 2, 1),
    "cifar_conv3": (64, 64, 64, 8, 8, 3, 1, 1), "cifar_conv4": (64, 64, 64, 8, 8, 1, 0, 1),
    "cifar_conv5": (64, 64, 16, 8, 8, 1, 0, 1),
    # MNIST CNNs (configs[2]): few channels -- skinny GEMMs
    "mnist_conv1": (64, 1, 5, 28, 28, 5, 2, 2), "mnist_conv2": (64, 5, 5, 14, 14, 5, 2, 1),
}
MATMULS = {"mm_1024x1600x512": (1024, 1600, 512), "mm_4096x4096x4096": (4096, 4096, 4096),
           "mm_128x784x64": (128, 784, 64)}


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main():
    rng = np.random.default_rng(0)
    st = D.stream()
    only = sys.argv[1] if len(sys.argv) > 1 else ""
    for name, (B, ci, co, H, W, s, p, stv) in CONVS.items():
        if only and not name.startswith(only):
            continue
        oh = (H + 2 * p - s) // stv + 1
        x = D.u64_to_device(rng.integers(0, 1 << 59, size=(B, ci, H, W), dtype=np.uint64))
        w = D.u64_to_device(rng.integers(0, 1 << 59, size=(co, ci, s, s), dtype=np.uint64))
        gy = D.u64_to_device(rng.integers(0, 1 << 59, size=(B, co, oh, oh), dtype=np.uint64))
        macs = B * co * ci * s * s * oh * oh
        for kind, a, b, shp in ((_lib.CONV_FWD, x, w, (B, co, oh, oh)), (_lib.CONV_BWDX, gy, w, (B, ci, H, W)),
                                (_lib.CONV_GRADW, x, gy, (co, ci, s, s))):
            out = D.empty_u64(*shp)
            for be in (1, 2):
                ms = timeit(lambda: _lib.call("pb_ring_conv_ex", kind, D.ptr(a), D.ptr(b), B, ci, co, H, W, s, p, stv,
                                              59, D.ptr(out), be, st))
                print(json.dumps({"op": f"{name}/{['fwd', 'bwdx', 'gradw'][kind]}", "backend": ["", "cuda_core",
                                  "tensor"][be], "ms": ms, "u64_macs": macs, "macs_per_s": macs / ms * 1e3}),
                      flush=True)
    for name, (n, k, m) in MATMULS.items():
        if only:
            continue
        a = D.u64_to_device(rng.integers(0, 1 << 59, size=(n, k), dtype=np.uint64))
        b = D.u64_to_device(rng.integers(0, 1 << 59, size=(k, m), dtype=np.uint64))
        out = D.empty_u64(n, m)
        for be in (1, 2):
            ms = timeit(lambda: _lib.call("pb_ring_matmul_ex", D.ptr(a), D.ptr(b), n, k, m, 0, 0, 59, D.ptr(out), be,
                                          st))
            print(json.dumps({"op": name, "backend": ["", "cuda_core", "tensor"][be], "ms": ms, "u64_macs": n * k * m,
                              "macs_per_s": n * k * m / ms * 1e3}), flush=True)


if __name__ == "__main__":
    main()
