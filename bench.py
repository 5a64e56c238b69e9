"""Benchmark: Pencil private training step on the B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload: one private training step of the MNIST MLP
784-128-128-10, batch 64, synthetic MNIST-shaped data, BFV N=8192, t=2^59,
7 x 30-bit RNS limbs, f=25: per FC layer Alg.1 forward, Alg.2 weight
gradient, bias reveal and (layers 2-3) the input gradient, all through the
B200 engine; ReLU/truncation via the SPEC's dealer backend; softmax-CE and
SGD-momentum exactly as the reference engine.  A "step" therefore performs
~2000 ciphertext x plaintext products, ~2000 decryptions and ~900
encryptions (see DESIGN.md for the block plan).

Prints ONE JSON line on rank 0.  ``value`` is samples/s with the batch
resident in HBM; ``e2e`` is the same metric through the public API with the
batch copied from pinned host memory every step and the loss read back;
``roofline`` is the dominant kernel's algorithmic HBM bytes / its CUDA-event
time; ``cpu_baseline`` is the oracle (the reference's CPU algorithm restated
in C + numpy) timed on this host's cores on one step of the same workload.
``--impl reference`` times that CPU path alone on the same config.

Multi-GPU (torchrun, N>1): every he-matmul's output ciphertext blocks are
sharded round-robin over the ranks (each rank encrypts only the input
ciphertexts its blocks need) and the decrypted share tiles are summed with
one NCCL all-reduce (exact: every element comes from exactly one rank);
the batch is fixed, so scaling is "strong".
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "private-training samples/sec; HE linear-layer ct-pt MACs/sec + NTT GB/s vs roofline"
SIZES = [784, 128, 128, 10]
BATCH = 64
SEED = 2024


# entry point -> device kernels it launches (for the ncu DRAM-traffic lookup)
ENTRY_KERNELS = {
    "pb_encrypt_sk": ("k_encrypt_sk",), "pb_encrypt_sk_zero": ("k_encrypt_sk",),
    "pb_encrypt_sk_add": ("k_encrypt_add",), "pb_encode_plain_mont": ("k_encode_plain_mont",),
    "pb_mask_ntt": ("k_mask_ntt",), "pb_ctpt_mac_tiled": ("k_mac_ws", "k_mac_pipe", "k_mac_eager"),
    "pb_decrypt_to_share": ("k_decrypt_share_cluster", "k_decrypt_inv", "k_decode_gather"),
}


def _traffic(entry):
    """DRAM bytes per launch of an entry point's kernels from the committed ncu
    capture of the same step (profiles/r01_step_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_step_traffic.json")) as f:
            ks = json.load(f)["kernels"]
    except Exception:
        return None
    names = [k for k in ENTRY_KERNELS.get(entry, ()) if k in ks]
    if not names:
        return None
    # kernels of one entry point launch once per call each (k_mac_pipe / k_mac_eager: either)
    if entry == "pb_ctpt_mac_tiled":
        tot = sum(ks[k]["dram_bytes_per_launch"] * ks[k]["launches"] for k in names)
        return tot / max(1, sum(ks[k]["launches"] for k in names))
    return float(sum(ks[k]["dram_bytes_per_launch"] for k in names))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.samples = []
        self.idx = gpu_index
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    f = [x.strip() for x in line.split(",")]
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and "Active" in s[3 + i]
                          and "Not" not in s[3 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------- CPU legs ---

def cpu_oracle_step_time(steps=1, warmup=1):
    """Time the oracle (reference CPU algorithm) on one private step of the workload."""
    from oracle import bfv as OB
    from oracle import kernels as OK
    from oracle import nn as ON
    from oracle import protocols as OPR
    from oracle import ring as OR
    from oracle.params import make_params

    ncores = os.cpu_count() or 1
    OK.set_threads(ncores)
    ring = OR.RingParams()
    p = make_params(8192, 7)
    ar = OB.Arith(p)
    kp = OB.keygen(p, OR.SeededRng(SEED, 0), ar)
    model = ON.Model(SIZES, ring, seed=SEED)
    x, labels = ON.synthetic_mnist(SEED, BATCH, ring)
    ctx = OPR.Ctx(p, ring, kp, seed=SEED, ar=ar)
    for _ in range(warmup):
        ON.private_train_step(ctx, model, x, labels)
    t0 = time.perf_counter()
    for i in range(steps):
        ctx.seed = SEED + 1 + i
        ON.private_train_step(ctx, model, x, labels)
    dt = (time.perf_counter() - t0) / steps
    return dt, OK.get_threads()


def run_reference(args, rank, world):
    if rank != 0:
        return
    steps = max(1, args.steps)
    warm = max(0, args.warmup)
    # bounded sample: one oracle step is several seconds; cap the run to a few minutes
    t_first, cores = cpu_oracle_step_time(steps=1, warmup=min(warm, 1))
    budget = 240.0
    steps_run = max(1, min(steps, int(budget / max(t_first, 1e-3))))
    dt, cores = cpu_oracle_step_time(steps=steps_run, warmup=0) if steps_run > 1 else (t_first, cores)
    v = BATCH / dt
    sample = (f"{steps_run} private training step(s) of the MNIST MLP 784-128-128-10, B={BATCH}, N=8192, L=7 "
              f"(oracle = reference kernel algorithms restated in C/OpenMP + numpy), after in-process warm-up")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world,
        "steps": steps_run, "warmup": min(warm, 1), "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32-rns/u64-ring", "data": "synthetic",
        "config": {"workload": "configs[1]: MNIST MLP 784-128-128-10 private training step", "global_batch": BATCH,
                   "bfv": "N=8192, t=2^59, L=7x30-bit", "f": 25},
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU leg ----

def run_ours(args, rank, world):
    import torch

    from paper_2403_11166_b200 import _dev, _lib, bfv
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.linear_protocols import Session
    from paper_2403_11166_b200.params import BfvParams
    from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed

    dev = _dev.device()
    ring = RingParams()
    params = BfvParams()
    kp = bfv.keygen(params, SeededRng(SEED, 0))
    group = None
    if world > 1:
        import torch.distributed as dist

        group = dist.group.WORLD
    sess = Session(params, ring, kp, seed=SEED, shard=(rank, world, group))
    model = PN.Model(SIZES, ring, seed=SEED)
    xh, labels = PN.synthetic_mnist(SEED, BATCH, ring)
    x_dev = RingTensor(encode_fixed(xh, ring), ring.f, ring, _canonical=True)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.int64, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    def eager_step(i, x):
        sess.reseed(SEED + 10 + i)
        return PN.private_train_step(sess, model, x, labels, check=False)

    for i in range(max(3, args.warmup)):
        eager_step(i, x_dev)
    torch.cuda.synchronize()

    # ---- kernel profile pass (eager, CUDA events around every fused entry point):
    #      per-kernel durations + algorithmic bytes, kernel launches per step
    prof_steps = 3
    stats = _lib.CallStats(timed=("pb_ctpt_mac_tiled", "pb_mask_ntt", "pb_decrypt_to_share", "pb_encrypt_sk",
                                  "pb_encrypt_sk_add", "pb_encrypt_sk_zero", "pb_encode_plain_mont"))
    sess.alg_bytes.clear()
    _lib.STATS = stats
    for i in range(prof_steps):
        flush.zero_()
        eager_step(500 + i, x_dev)
    _lib.STATS = None
    torch.cuda.synchronize()
    launches_per_step = stats.launches / prof_steps
    per = {}
    for name, s, e, _tag in stats.events:
        acc = per.setdefault(name, [0.0, 0])
        acc[0] += s.elapsed_time(e)
        acc[1] += 1
    alg = dict(sess.alg_bytes)
    census_per_step = sess.channel.total_bytes() / max(1, sess.steps_seen)

    # ---- timed region: the same step replayed from CUDA graphs (GraphStep),
    #      batch resident in HBM, per-step CUDA events, L2 flushed between steps
    try:
        runner = PN.GraphStep(sess, model, x_dev, prefetch_input=True)
        replay = "CUDA graphs"
    except Exception as exc:  # e.g. a collective backend that cannot be captured
        if world == 1:
            raise
        torch.cuda.synchronize()
        runner = _EagerStep(sess, model, x_dev)
        replay = f"eager launches (graph capture failed: {type(exc).__name__})"
    for i in range(3):
        runner.step(SEED + 100 + i, labels)
    torch.cuda.synchronize()
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    evs = []
    loss = None
    for i in range(args.steps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        loss = runner.step(SEED + 1000 + i, labels)
        if hasattr(runner, "join_prefetch"):
            runner.join_prefetch()  # the next step's prefetched input encryption is inside this window
        e.record()
        evs.append((s, e))
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    t_ms = _max_over_ranks(sum(s.elapsed_time(e) for s, e in evs), world)
    value = args.steps * BATCH / (t_ms / 1e3)

    dom = max(per, key=lambda k: per[k][0])
    tot_ms, n_launch = per[dom]
    peak, peak_kind = _peaks()
    bytes_per_launch = alg.get(dom, 0.0) / max(1, n_launch)
    achieved = bytes_per_launch / (tot_ms / n_launch / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_kind": peak_kind, "traffic": _traffic(dom),
                "traffic_note": "ncu dram__bytes_read+write per launch (profiles/r01_step_traffic.json); far below "
                                "the algorithmic bytes because the step's working set is L2-resident",
                "bytes_per_launch": bytes_per_launch, "launches": n_launch,
                "ms_per_launch": tot_ms / n_launch, "share_of_step": (tot_ms / prof_steps) / (t_ms / args.steps)}
    kernels = {k: {"ms_per_step": v[0] / prof_steps, "calls_per_step": v[1] / prof_steps,
                   "alg_GBs": (alg.get(k, 0.0) / (v[0] / 1e3) / 1e9) if v[0] else None} for k, v in per.items()}

    # ---- e2e through the public API: host batch (pinned) -> device every step, loss back on the host
    x_pin = torch.from_numpy(np.ascontiguousarray(xh)).pin_memory()
    torch.cuda.synchronize()
    barrier()
    evs = []
    h2d = x_pin.numel() * 8
    for i in range(args.steps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        if hasattr(runner, "load_batch"):
            runner.load_batch(x_pin)  # H2D + device encode, range flag checked at the step's sync
        else:
            x_dev.values.copy_(encode_fixed(x_pin.to(dev, non_blocking=True), ring))
        loss = runner.step(SEED + 2000 + i, labels)
        if hasattr(runner, "join_prefetch"):
            runner.join_prefetch()
        e.record()
        evs.append((s, e))
    torch.cuda.synchronize()
    barrier()
    te_ms = _max_over_ranks(sum(s.elapsed_time(e) for s, e in evs), world)
    e2e = {"value": args.steps * BATCH / (te_ms / 1e3), "unit": "samples/s",
           # per step: batch H2D + DO loss-gradient H2D; logits D2H (DO reconstructs) + encode range flag
           "h2d_bytes_per_step": h2d + 10 * BATCH * 8, "d2h_bytes_per_step": 10 * BATCH * 8 + 4}

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu and world == 1:
        dt, cores = cpu_oracle_step_time(steps=1, warmup=1)
        cpu = {"value": BATCH / dt, "unit": "samples/s", "cores": cores, "kind": "port",
               "sample": "1 private training step (MNIST MLP 784-128-128-10, B=64, N=8192, L=7) of the oracle "
                         "(reference kernel algorithms restated in C/OpenMP + numpy), after an in-process warm-up step"}
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": t_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32-rns/u64-ring", "data": "synthetic",
        "config": {"workload": "configs[1]: MNIST MLP 784-128-128-10 private training step", "global_batch": BATCH,
                   "bfv": "N=8192, t=2^59, L=7x30-bit (log2 Q = 210)", "f": 25,
                   "parallelism": f"ct-block shards x{world}" if world > 1 else "single GPU",
                   "l2": "flushed (256 MiB write) between timed steps"},
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
        "gpu_launches": int(round(launches_per_step * args.steps)), "kernels": kernels, "loss": loss,
        "census_bytes_per_step": census_per_step,
        "timing": f"value/e2e: K steps replayed from {replay} (same kernels); per-kernel times from an "
                  "instrumented eager pass of the same step",
    }
    print(json.dumps(line), flush=True)


class _EagerStep:
    """GraphStep's interface over plain eager launches (multi-rank fallback)."""

    def __init__(self, sess, model, x):
        self.sess, self.model, self.x = sess, model, x

    def step(self, seed, labels):
        from paper_2403_11166_b200 import nn as PN

        self.sess.reseed(seed)
        loss, _, _ = PN.private_train_step(self.sess, self.model, self.x, labels, check=False)
        return loss


def _max_over_ranks(v, world):
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
