"""pb_encrypt_sk under a launch cap (the background operand preparation) vs
uncapped: CUDA-graph time per call and bit-identity of the ciphertexts.
usage: python scripts/enc_cap.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib, bfv  # noqa: E402
from paper_2403_11166_b200.params import BfvParams, context  # noqa: E402
from paper_2403_11166_b200.ring import SeededRng  # noqa: E402


def main():
    p = BfvParams()
    h = context(p).handle
    kp = bfv.keygen(p, SeededRng(1, 0))
    out = {}
    for nP in (16, 80, 100):
        m = torch.randint(0, 1 << 40, (nP, p.N), dtype=torch.int64, device="cuda")
        res = {}
        for cap in (0, 148):
            ct = torch.empty((nP, 2, p.L, p.N), dtype=torch.int32, device="cuda")

            def f():
                _lib.call("pb_set_launch_cap", cap)
                _lib.call("pb_encrypt_sk", h, _dev.ptr(kp.sk_ntt), _dev.ptr(kp.sk_sh), _dev.ptr(m), None, None, 0, nP, 1234, None, 7,
                          _dev.ptr(ct), _dev.stream())
                _lib.call("pb_set_launch_cap", 0)

            f()
            torch.cuda.synchronize()
            ref = ct.clone()
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                f()
            torch.cuda.current_stream().wait_stream(st)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(10):
                    f()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            res[f"cap{cap}_us"] = round(e0.elapsed_time(e1) / 10 * 1e3, 2)
            res[f"cap{cap}"] = ref
        res["identical"] = bool(torch.equal(res.pop("cap0"), res.pop("cap148")))
        out[nP] = res
    print(json.dumps(out))


if __name__ == "__main__":
    main()
