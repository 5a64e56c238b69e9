"""Device timeline of graph-replayed private steps (CUPTI through
torch.profiler): every kernel's start/end/stream, the per-stream busy time,
the SM-idle gaps, and a critical-path estimate -- what the serialised ncu
launch list cannot show.  Writes gpurun_out/timeline_<model>.json (compact
per-kernel list of one step) and prints a summary.

usage: python scripts/timeline.py [model] [B]
"""
import collections
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2403_11166_b200 import bfv  # noqa: E402
from paper_2403_11166_b200 import nn as PN  # noqa: E402
from paper_2403_11166_b200.linear_protocols import Session  # noqa: E402
from paper_2403_11166_b200.params import BfvParams  # noqa: E402
from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed  # noqa: E402


def short(name):
    n = re.sub(r"^void ", "", name.strip()).replace("(anonymous namespace)::", "")
    n = re.sub(r"<.*", "", n)
    n = re.sub(r"\(.*", "", n)
    return n.split("::")[-1].strip() or name[:40]


def main(name="mnist_mlp", B=64, steps=3):
    ring, params = RingParams(), BfvParams()
    sess = Session(params, ring, bfv.keygen(params, SeededRng(1, 0)), seed=1)
    model = PN.Model(name, ring, seed=1)
    if len(model.in_shape) == 1:
        xh, labels = PN.synthetic_mnist(1, B, ring)
    else:
        xh, labels = PN.synthetic_images(1, B, model.in_shape, ring)
    x = RingTensor(encode_fixed(xh, ring), ring.f, ring, _canonical=True)
    r = PN.GraphStep(sess, model, x, prefetch_input=True)
    for i in range(5):
        r.step(100 + i, labels)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for i in range(steps):
            r.step(200 + i, labels)
        torch.cuda.synchronize()
    os.makedirs("gpurun_out", exist_ok=True)
    trace = f"gpurun_out/trace_{name}.json"
    prof.export_chrome_trace(trace)
    with open(trace) as f:
        ev = json.load(f)["traceEvents"]
    ks = [e for e in ev if e.get("cat") == "kernel"]
    ks.sort(key=lambda e: e["ts"])
    if not ks:
        print("no kernel events (CUPTI unavailable?)")
        return
    # split into steps at the largest gaps (host loss between fwd and bwd, and between steps)
    t0, t1 = ks[0]["ts"], ks[-1]["ts"] + ks[-1]["dur"]
    # per-step: take the last step's kernels = those after the (2*steps-1)-th largest gap
    gaps = []
    end = ks[0]["ts"] + ks[0]["dur"]
    for a, b in zip(ks, ks[1:]):
        end = max(end, a["ts"] + a["dur"])
        if b["ts"] > end:
            gaps.append((b["ts"] - end, b["ts"]))
    big = sorted(gaps, reverse=True)[: 2 * steps - 1]
    cuts = sorted(t for _, t in big)
    # start of the last step's backward (cuts[-2]) or, with PB_TIMELINE_FULL=1, its forward (cuts[-3])
    back = 3 if os.environ.get("PB_TIMELINE_FULL") == "1" else 2
    last_start = cuts[-back] if len(cuts) >= back else t0
    step_ks = [k for k in ks if k["ts"] >= last_start]
    s0 = step_ks[0]["ts"]
    s1 = max(k["ts"] + k["dur"] for k in step_ks)
    busy = collections.Counter()
    per_kernel = collections.defaultdict(lambda: [0.0, 0])
    streams = collections.defaultdict(list)
    for k in step_ks:
        nm = short(k["name"])
        per_kernel[nm][0] += k["dur"]
        per_kernel[nm][1] += 1
        st = k.get("args", {}).get("stream", k.get("tid"))
        streams[st].append(k)
        busy[st] += k["dur"]
    # union of busy intervals (any stream) and idle gaps inside the step
    iv = sorted((k["ts"], k["ts"] + k["dur"]) for k in step_ks)
    union, cur = 0.0, list(iv[0])
    idle = []
    for a, b in iv[1:]:
        if a > cur[1]:
            union += cur[1] - cur[0]
            idle.append((cur[1] - s0, a - cur[1]))
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    union += cur[1] - cur[0]
    out = {
        "model": name, "B": B, "step_span_us": s1 - s0, "gpu_busy_union_us": union,
        "sum_kernel_us": sum(v[0] for v in per_kernel.values()), "kernels": len(step_ks),
        "streams": {str(s): {"busy_us": round(busy[s], 1), "kernels": len(v)} for s, v in streams.items()},
        "idle_gaps_us": [(round(a, 1), round(d, 1)) for a, d in idle if d > 2.0],
        "per_kernel": {k: {"us": round(v[0], 1), "n": v[1]} for k, v in
                       sorted(per_kernel.items(), key=lambda kv: -kv[1][0])},
        "launches": [(round(k["ts"] - s0, 1), round(k["dur"], 1), str(k.get("args", {}).get("stream", k.get("tid"))),
                      short(k["name"]), k.get("args", {}).get("grid")) for k in step_ks],
    }
    with open(f"gpurun_out/timeline_{name}.json", "w") as f:
        json.dump(out, f, indent=0)
    os.remove(trace)
    print(json.dumps({k: v for k, v in out.items() if k != "launches"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "mnist_mlp", int(sys.argv[2]) if len(sys.argv) > 2 else 64)
