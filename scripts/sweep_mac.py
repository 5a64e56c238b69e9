"""MAC tile-variant sweep (PB_MAC_VARIANT, read once per process): CUDA-graph
timing of pb_ctpt_mac_tiled at the MLP step's plan shapes and the conv-like
K=16 shape, with a checksum of the output so variants can be compared for
bit-identity.  usage: PB_MAC_VARIANT=k python scripts/sweep_mac.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib  # noqa: E402
from paper_2403_11166_b200.params import BfvParams, context  # noqa: E402


def main():
    p = BfvParams()
    h = context(p).handle
    L, N = p.L, p.N
    g = torch.Generator(device="cuda").manual_seed(0)
    res = {"variant": int(os.environ.get("PB_MAC_VARIANT", "0"))}
    # (name, nB, nO, nI, two_terms)
    for name, nB, nO, nI, two in (("fwd0", 4, 8, 25, False), ("gw0", 5, 10, 16, False), ("fwd1", 2, 8, 8, False),
                                  ("gw1", 4, 8, 8, True), ("conv", 64, 13, 16, False), ("cifar", 16, 16, 9, True),
                                  ("cifar_gw2", 13, 32, 32, True)):
        q = p.moduli[-1]
        ctA = torch.randint(0, q, (nB * nI, 2, L, N), dtype=torch.int32, device="cuda", generator=g)
        ptA = torch.randint(0, q, (nO * nI, L, N), dtype=torch.int32, device="cuda", generator=g)
        ctB = torch.randint(0, q, (nO * nI, 2, L, N), dtype=torch.int32, device="cuda", generator=g) if two else None
        ptB = torch.randint(0, q, (nB * nI, L, N), dtype=torch.int32, device="cuda", generator=g) if two else None
        out = torch.zeros((nB * nO, 2, L, N), dtype=torch.int32, device="cuda")

        def f():
            _lib.call("pb_ctpt_mac_tiled", h, _dev.ptr(ctA), _dev.ptr(ptA), _dev.ptr(ctB) if two else None,
                      _dev.ptr(ptB) if two else None, nB, nO, nI, _dev.ptr(out), _dev.stream())

        f()
        torch.cuda.synchronize()
        chk = int(out.to(torch.int64).sum().item())
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            for _ in range(2):
                f()
        torch.cuda.current_stream().wait_stream(st)
        gr = torch.cuda.CUDAGraph()
        iters = 20
        with torch.cuda.graph(gr):
            for _ in range(iters):
                f()
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / iters * 1e3
        macs = nB * nO * nI * (2 if two else 1) * 2 * L * N
        res[name] = {"us": round(us, 2), "mod_macs_per_s": macs / (us * 1e-6), "chk": chk}
        del ctA, ptA, ctB, ptB, out
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
