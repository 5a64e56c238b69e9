"""Where the private step's time goes (graph replay through GraphStep.step,
prefetched input encryption as in bench.py) -- CUDA events at the phase
boundaries (GraphStep.timing), with and without an L2 flush before the step.
With the device-side host handoff (default, PB_HANDOFF=1) the phases are the
forward graph and the backward graph, whose chain waits on the device for the
host's float64 softmax-CE (so "bwd" includes the host loss); with
PB_HANDOFF=0 also the host round trip ("host": logits D2H, loss, gradient
H2D) and the wait for the separately replayed operand-preparation graph ("pre")."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_11166_b200 import bfv  # noqa: E402
from paper_2403_11166_b200 import nn as PN  # noqa: E402
from paper_2403_11166_b200.linear_protocols import Session  # noqa: E402
from paper_2403_11166_b200.params import BfvParams  # noqa: E402
from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed  # noqa: E402


def main(name="mnist_mlp", B=64, iters=20):
    ring, params = RingParams(), BfvParams()
    sess = Session(params, ring, bfv.keygen(params, SeededRng(1, 0)), seed=1)
    model = PN.Model(name, ring, seed=1)
    if len(model.in_shape) == 1:
        xh, labels = PN.synthetic_mnist(1, B, ring)
    else:
        xh, labels = PN.synthetic_images(1, B, model.in_shape, ring)
    x = RingTensor(encode_fixed(xh, ring), ring.f, ring, _canonical=True)
    r = PN.GraphStep(sess, model, x, prefetch_input=True)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.int64, device="cuda")
    for i in range(5):
        r.step(100 + i, labels)
    torch.cuda.synchronize()
    for flushed in (False, True):
        acc = {}
        for i in range(iters):
            if flushed:
                flush.zero_()
            r.timing = []
            r.step(500 + i, labels)
            torch.cuda.synchronize()
            ev = r.timing
            r.timing = None
            for (a, ea), (b, eb) in zip(ev, ev[1:]):
                acc[b] = acc.get(b, 0.0) + ea.elapsed_time(eb)
            acc["step"] = acc.get("step", 0.0) + ev[0][1].elapsed_time(ev[-1][1])
        print(json.dumps({"model": name, "l2_flushed": flushed, **{k: round(v / iters, 4) for k, v in acc.items()}}),
              flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["mnist_mlp"]))
