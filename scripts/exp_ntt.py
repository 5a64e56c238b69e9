"""Drive scripts/exp_ntt.cu variants on the B200: correctness vs the product
NTT and CUDA-event throughput over 1 GiB of residues (N=8192, L=7)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib  # noqa: E402
from paper_2403_11166_b200.params import BfvParams, context  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libexp_ntt.so"))
lib.exp_ntt_fwd.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                            ctypes.c_int, ctypes.c_void_p]
lib.exp_occupancy.argtypes = [ctypes.c_int, ctypes.c_int]


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    p = BfvParams(N=8192, L=7)
    ctx = context(p)
    rows = (1 << 30) // (4 * 8192)
    rows -= rows % 7
    x0 = torch.randint(0, p.moduli[-1], (rows, 8192), dtype=torch.int32, device="cuda")
    st = _dev.stream()
    want = x0.clone()
    _lib.call("pb_ntt_forward", ctx.handle, want.data_ptr(), rows, None, st)
    x = torch.empty_like(x0)
    by = rows * 8192 * 8
    base = timeit(lambda: _lib.call("pb_ntt_forward", ctx.handle, x.data_ptr(), rows, None, st))
    print(json.dumps({"variant": "product", "ms": base, "GB_s": by / base / 1e6}), flush=True)
    combos = [tuple(int(t) for t in a.split(",")) for a in sys.argv[1:]] or [(5, 4, 0)]
    for v, minb, cps in combos:
        x.copy_(x0)
        rc = lib.exp_ntt_fwd(ctx.handle, v, minb, x.data_ptr(), rows, cps, st)
        torch.cuda.synchronize()
        ok = rc == 0 and torch.equal(x, want)
        t = timeit(lambda: lib.exp_ntt_fwd(ctx.handle, v, minb, x.data_ptr(), rows, cps, st))
        print(json.dumps({"variant": v, "minb": minb, "ctas_per_sm_cap": cps, "occ": lib.exp_occupancy(v, minb),
                          "ok": bool(ok), "rc": rc, "ms": t, "GB_s": by / t / 1e6}), flush=True)


if __name__ == "__main__":
    main()
