"""Warm per-launch latency of the fused protocol kernels at the MLP step's
plan sizes (back-to-back launches on one stream, CUDA events, L2 warm):
how long ONE small launch takes when the GPU is otherwise idle."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib, bfv  # noqa: E402
from paper_2403_11166_b200.linear_protocols import _Shard, _pk  # noqa: E402
from paper_2403_11166_b200.params import BfvParams  # noqa: E402
from paper_2403_11166_b200.poly_encoding import MatmulGeometry, plan_matmul  # noqa: E402
from paper_2403_11166_b200.ring import SeededRng  # noqa: E402


def t_launch(fn, iters=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us


def t_graph(fn, iters=50):
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


def main():
    p = BfvParams()
    kp = bfv.keygen(p, SeededRng(1, 0))
    h = kp.ctx.handle if hasattr(kp, "ctx") else None
    from paper_2403_11166_b200.params import context

    h = context(p).handle
    L, N = p.L, p.N
    st = _dev.stream()
    vals = _dev.u64_to_device(np.random.default_rng(0).integers(0, 1 << 59, size=784 * 784, dtype=np.uint64))
    for nm, g in [("fwd0", (784, 128, 64)), ("fwd1", (128, 128, 64)), ("fwd2", (128, 10, 64)),
                  ("bx2", (10, 128, 64)), ("gw0", (64, 128, 784))]:
        plan = plan_matmul(MatmulGeometry(*g), N)
        sh = _Shard(plan, 0, 1)
        ct = _dev.empty_u32(sh.n_in, 2, L, N)
        ebuf = torch.zeros(sh.n_in, N, dtype=torch.int8, device=ct.device)
        pt = _dev.empty_u32(sh.n_pt, L, N)
        out = _dev.empty_u32(sh.n_out, 2, L, N)
        share = _dev.empty_u64(g[1] * g[2])
        scratch = _dev.empty_u32(sh.n_out, L, sh.U)
        mask = _dev.u64_to_device(np.zeros(g[1] * g[2], dtype=np.uint64))
        fns = {
            "encrypt_sk": lambda: _lib.call("pb_encrypt_sk", h, _dev.ptr(kp.sk_ntt), _dev.ptr(kp.sk_sh), _dev.ptr(vals), *_pk(sh.in_pack),
                                            sh.n_in, 5, None, 0, _dev.ptr(ct), _dev.stream()),
            "encrypt_add": lambda: _lib.call("pb_encrypt_sk_add", h, _dev.ptr(vals), *_pk(sh.in_pack), sh.n_in,
                                             _dev.ptr(ebuf), _dev.ptr(ct), _dev.stream()),
            "encrypt_zero": lambda: _lib.call("pb_encrypt_sk_zero", h, _dev.ptr(kp.sk_ntt), sh.n_in, 5, None, 0,
                                              _dev.ptr(ct), _dev.ptr(ebuf), _dev.stream()),
            "encode_mont": lambda: _lib.call("pb_encode_plain_mont", h, _dev.ptr(vals), *_pk(sh.pt_pack), sh.n_pt,
                                             _dev.ptr(pt), _dev.stream()),
            "mask_ntt": lambda: _lib.call("pb_mask_ntt", h, sh.n_out, _dev.ptr(sh.out_pos), _dev.ptr(sh.out_dst), sh.U,
                                          _dev.ptr(mask), 1, 7, None, _dev.ptr(out), _dev.stream()),
            "mac_tiled": lambda: _lib.call("pb_ctpt_mac_tiled", h, _dev.ptr(ct), _dev.ptr(pt), None, None, sh.nb,
                                           sh.no, sh.nI, _dev.ptr(out), _dev.stream()),
            "decrypt_to_share": lambda: _lib.call("pb_decrypt_to_share", h, _dev.ptr(kp.sk_ntt), _dev.ptr(out),
                                                  sh.n_out, _dev.ptr(sh.out_pos), _dev.ptr(sh.out_dst), sh.U,
                                                  _dev.ptr(share), _dev.ptr(scratch), _dev.stream()),
        }
        res = {"plan": nm, "n_in": sh.n_in, "n_pt": sh.n_pt, "n_out": sh.n_out, "nI": sh.nI}
        for k, f in fns.items():
            res[k] = [round(t_launch(f), 2), round(t_graph(f), 2)]
        print(json.dumps(res), flush=True)
    # empty-kernel floor
    x = _dev.empty_u64(16)
    res = {"ring_binary_16": [round(t_launch(lambda: _lib.call("pb_ring_binary", 0, _dev.ptr(x), _dev.ptr(x), _dev.ptr(x),
                                                                16, 16, 59, st)), 2)]}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
