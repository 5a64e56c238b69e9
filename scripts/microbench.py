"""Kernel microbenchmarks (CUDA events): NTT fwd/inv over >= 1 GiB of residues."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2403_11166_b200 import _dev, _lib
from paper_2403_11166_b200.params import BfvParams, context


def time_it(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3


def main():
    res = []
    for N, L in ((4096, 7), (8192, 7), (16384, 7), (32768, 8), (8192, 2)):
        p = BfvParams(N=N, L=L)
        ctx = context(p)
        rows = (1 << 30) // (4 * N)
        rows -= rows % L
        x = torch.randint(0, p.moduli[-1], (rows, N), dtype=torch.int32, device="cuda")
        st = _dev.stream()
        tf = time_it(lambda: _lib.call("pb_ntt_forward", ctx.handle, x.data_ptr(), rows, None, st))
        x = torch.randint(0, p.moduli[-1], (rows, N), dtype=torch.int32, device="cuda")
        ti = time_it(lambda: _lib.call("pb_ntt_inverse", ctx.handle, x.data_ptr(), rows, None, st))
        by = rows * N * 4 * 2
        res.append(dict(N=N, L=L, rows=rows, fwd_ms=tf * 1e3, inv_ms=ti * 1e3, fwd_GBs=by / tf / 1e9, inv_GBs=by / ti / 1e9,
                        fwd_rows_per_s=rows / tf, inv_rows_per_s=rows / ti))
        print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__":
    main()
