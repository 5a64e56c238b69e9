"""Where the MLP private step's time goes (graph replay, warm L2): forward
graph, host loss (D2H logits, float64 softmax-CE, H2D gradient), backward
graph; and the same with the L2 flushed before the step (bench.py's rule)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11166_b200 import bfv  # noqa: E402
from paper_2403_11166_b200 import nn as PN  # noqa: E402
from paper_2403_11166_b200.linear_protocols import Session  # noqa: E402
from paper_2403_11166_b200.params import BfvParams  # noqa: E402
from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main(name="mnist_mlp", B=64, iters=20):
    ring, params = RingParams(), BfvParams()
    sess = Session(params, ring, bfv.keygen(params, SeededRng(1, 0)), seed=1)
    model = PN.Model(name, ring, seed=1)
    if len(model.in_shape) == 1:
        xh, labels = PN.synthetic_mnist(1, B, ring)
    else:
        xh, labels = PN.synthetic_images(1, B, model.in_shape, ring)
    x = RingTensor(encode_fixed(xh, ring), ring.f, ring, _canonical=True)
    r = PN.GraphStep(sess, model, x)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.int64, device="cuda")
    for i in range(5):
        r.step(100 + i, labels)
    torch.cuda.synchronize()
    for flushed in (False, True):
        acc = {"fwd": 0.0, "host": 0.0, "bwd": 0.0, "step": 0.0}
        for i in range(iters):
            if flushed:
                flush.zero_()
            e0, e1, e2, e3 = ev(), ev(), ev(), ev()
            r.sess.reseed(500 + i)
            main = torch.cuda.current_stream()
            e0.record()
            r.g_fwd.replay()
            e1.record()
            r._pre_stream.wait_stream(main)
            with torch.cuda.stream(r._pre_stream):
                r.g_pre.replay()
            r.logits_host.copy_(r.logits.values, non_blocking=True)
            main.synchronize()
            t0 = time.perf_counter()
            loss, _ = r._loss(labels)
            acc["host"] += (time.perf_counter() - t0) * 1e3
            r.g_do.copy_(r.g_host, non_blocking=True)
            e2.record()
            main.wait_stream(r._pre_stream)
            r.g_bwd.replay()
            e3.record()
            torch.cuda.synchronize()
            acc["fwd"] += e0.elapsed_time(e1)
            acc["bwd"] += e2.elapsed_time(e3)
            acc["step"] += e0.elapsed_time(e3)
        print(json.dumps({"model": name, "l2_flushed": flushed, **{k: round(v / iters, 4) for k, v in acc.items()}}),
              flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["mnist_mlp"]))
