"""Graph-timed latency of pb_ring_matmul_add at the MLP step's local-term shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib  # noqa: E402


def t_graph(fn, iters=50):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
    torch.cuda.current_stream().wait_stream(st)
    g = torch.cuda.CUDAGraph()
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


rng = np.random.default_rng(0)
res = {}
for n, k, m, ta, tb in ((128, 128, 64, 0, 0), (10, 128, 64, 0, 0), (128, 10, 64, 1, 0), (10, 64, 128, 0, 1),
                        (128, 64, 128, 0, 1), (128, 64, 784, 0, 1), (1, 1, 1, 0, 0)):
    a = _dev.u64_to_device(rng.integers(0, 1 << 63, size=(n * k,), dtype=np.uint64))
    b = _dev.u64_to_device(rng.integers(0, 1 << 63, size=(k * m,), dtype=np.uint64))
    c = _dev.u64_to_device(rng.integers(0, 1 << 63, size=(n * m,), dtype=np.uint64))
    out = _dev.empty_u64(n * m)
    f = lambda: _lib.call("pb_ring_matmul_add", _dev.ptr(a), _dev.ptr(b), n, k, m, ta, tb, _dev.ptr(c), -1, 59,
                          _dev.ptr(out), _dev.stream())
    res[f"{n}x{k}x{m}"] = round(t_graph(f), 2)
x = _dev.empty_u64(16)
res["ring_binary_16"] = round(t_graph(lambda: _lib.call("pb_ring_binary", 0, _dev.ptr(x), _dev.ptr(x), _dev.ptr(x), 16,
                                                        16, 59, _dev.stream())), 2)
print(json.dumps(res))
