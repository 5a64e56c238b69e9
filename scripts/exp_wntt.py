"""Wide-NTT experiment: correctness vs the product NTT and single-row latency /
throughput of NttW<13, LOGV> (scripts/exp_ntt.cu) vs the product kernel."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib  # noqa: E402
from paper_2403_11166_b200.params import BfvParams, context  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libexp_ntt.so"))
lib.exp_wntt.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]


def tgraph(fn, iters=30):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


p = BfvParams()
ctx = context(p)
for rows in (7, 14, 70, 448, 32767):
    x0 = torch.randint(0, p.moduli[-1], (rows, 8192), dtype=torch.int32, device="cuda")
    want = x0.clone()
    _lib.call("pb_ntt_forward", ctx.handle, want.data_ptr(), rows, None, _dev.stream())
    res = {"rows": rows}
    x = x0.clone()
    res["product_fwd"] = round(tgraph(lambda: _lib.call("pb_ntt_forward", ctx.handle, x.data_ptr(), rows, None,
                                                       _dev.stream())), 2)
    res["product_inv"] = round(tgraph(lambda: _lib.call("pb_ntt_inverse", ctx.handle, x.data_ptr(), rows, None,
                                                       _dev.stream())), 2)
    for logv in (3, 4):
        x = x0.clone()
        lib.exp_wntt(ctx.handle, logv, 0, x.data_ptr(), rows, _dev.stream())
        ok_f = torch.equal(x, want)
        lib.exp_wntt(ctx.handle, logv, 1, x.data_ptr(), rows, _dev.stream())
        torch.cuda.synchronize()
        ok_i = torch.equal(x, x0)
        res[f"w{logv}_ok"] = [ok_f, ok_i]
        res[f"w{logv}_fwd"] = round(tgraph(lambda: lib.exp_wntt(ctx.handle, logv, 0, x.data_ptr(), rows, _dev.stream())), 2)
        res[f"w{logv}_inv"] = round(tgraph(lambda: lib.exp_wntt(ctx.handle, logv, 1, x.data_ptr(), rows, _dev.stream())), 2)
    print(json.dumps(res), flush=True)
