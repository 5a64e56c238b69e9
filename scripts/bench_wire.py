"""PBFV wire kernels on one B200: pb_wire_serialize /
pb_wire_deserialize over P ciphertexts at N=8192, L=7, into / out of HBM
and pinned host memory (the kernel moves the bytes over the host link
itself), against the unfused alternative (reorder + widen in HBM, then a
cudaMemcpy D2H of the frames).

Algorithmic bytes per residue: serialize 4 read + 8 written, deserialize 8
read + 4 written; the frame headers are noise.  L2 is flushed (256 MiB
write) before every timed launch.  One JSON line per case.

    python scripts/bench_wire.py [P ...]
"""

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2403_11166_b200 import _dev, _lib, bfv, ring, wire  # noqa: E402
from paper_2403_11166_b200.params import BfvParams, context  # noqa: E402


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 7700.0, "nominal"


def timed(fn, reps=10):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    ts = []
    for i in range(reps + 2):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main(Ps):
    pp = BfvParams(N=8192, L=7)
    h = context(pp).handle
    kp = bfv.keygen(pp, ring.SeededRng(1, 0))
    pk, kind = peak()
    for P in Ps:
        m = torch.zeros(P, pp.N, dtype=torch.int64, device="cuda")
        ct = bfv.encrypt(kp, m, ring.SeededRng(2, 0), mode="sk")
        res = P * 2 * pp.L * pp.N
        fb = wire.frame_bytes(pp)
        dev = torch.empty(P * fb, dtype=torch.uint8, device="cuda")
        host = torch.empty(P * fb, dtype=torch.uint8, pin_memory=True)
        back = _dev.empty_u32(P, 2, pp.L, pp.N)
        bad = torch.empty(1, dtype=torch.int32, device="cuda")
        s = _dev.stream()

        def ser(out):
            _lib.call("pb_wire_serialize", h, _dev.ptr(ct.data), P, 2, 1, out.data_ptr(), s)

        def des(src):
            _lib.call("pb_wire_deserialize", h, src.data_ptr(), P, 2, 1, _dev.ptr(back), _dev.ptr(bad), s)

        def unfused():  # what a non-fused path does: reorder + widen in HBM, then D2H
            t = ct.data.clone()
            _lib.call("pb_ntt_reorder", h, _dev.ptr(t), t.numel() // pp.N, 0, s)
            host[: res * 8].copy_(t.view(torch.int32).to(torch.int64).view(torch.uint8).view(-1), non_blocking=True)

        def staged():  # wire.serialize's default for a host destination
            ser(dev)
            host.copy_(dev, non_blocking=True)

        cases = [
            ("serialize_staged_to_pinned_host", staged, 12),
            ("serialize_to_hbm", lambda: ser(dev), 12),
            ("serialize_to_pinned_host", lambda: ser(host), 12),
            ("deserialize_from_hbm", lambda: des(dev), 12),
            ("deserialize_from_pinned_host", lambda: des(host), 12),
            ("unfused_reorder_widen_d2h", unfused, 12),
        ]
        ser(dev)
        ser(host)
        for name, fn, bpr in cases:
            ms = timed(fn)
            gbs = res * bpr / (ms * 1e-3) / 1e9
            line = {"kernel": name, "N": pp.N, "L": pp.L, "ciphertexts": P, "frame_bytes": fb, "ms": ms,
                    "alg_GB_s": gbs, "wire_GB_s": P * fb / (ms * 1e-3) / 1e9, "ct_per_s": P / (ms * 1e-3)}
            if "hbm" in name:
                line.update(frac_hbm=gbs / pk, peak_kind=kind)
            print(json.dumps(line), flush=True)
        assert torch.equal(back, ct.data) and int(bad.item()) == 0
        # SPEC:196 response compaction on the same ciphertexts: L rows read, L-1 written per polynomial
        ms = timed(lambda: bfv.mod_switch_drop(ct))
        alg = P * 2 * pp.N * 4 * (2 * pp.L - 1)
        print(json.dumps({"kernel": "mod_switch_drop", "N": pp.N, "L": pp.L, "ciphertexts": P, "ms": ms,
                          "alg_GB_s": alg / (ms * 1e-3) / 1e9, "frac_hbm": alg / (ms * 1e-3) / 1e9 / pk,
                          "peak_kind": kind, "ct_per_s": P / (ms * 1e-3),
                          "note": "memcpy2D + 1-limb INTT + lift + (L-1)-limb NTT + finish; includes allocation"}),
              flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [64, 1024])
