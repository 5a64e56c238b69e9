"""Benchmark: Pencil private training on the B200 (BASELINE.json configs[1]
headline, configs[3] and configs[4] beside it).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-cpu] [--no-configs]

Headline workload (configs[1]): one private training step of
the MNIST MLP 784-128-128-10, batch 64 per GPU, synthetic MNIST-shaped data,
BFV N=8192, t=2^59, 7 x 30-bit RNS limbs, f=25: per FC layer Alg.1 forward,
Alg.2 weight gradient, bias reveal and (layers 2-3) the input gradient, all
through the B200 engine; ReLU / truncation by the SPEC:479 dealer backend
(stated in the line: "nonlinear"); softmax-CE and SGD-momentum exactly as
the reference engine.

ONE JSON line on rank 0:
  value      samples/s, batch resident in HBM, steps replayed from CUDA graphs,
             CUDA events on the launching stream, L2 flushed (256 MiB write)
             before every timed step, max over ranks
  e2e        the same through the public API (GraphStep.load_batch + step):
             the float64 batch copied from pinned host memory every step, the
             logits read back for the DO's loss, the loss gradient copied in
  roofline   the step's dominant entry point by CUPTI device time over
             graph-replayed steps (torch.profiler): algorithmic HBM bytes
              / its device time, plus the integer-pipe fraction
             (NTT butterflies x 4 IMAD issue slots, lazy mod-MACs x 1
             IMAD.WIDE) against the measured B200 integer peaks
  kernels    per entry point: CUPTI ms per step, launches, HBM and int fractions
  configs    c4: CIFAR-10 CNN private step (PAPER Fig. 7, B=64), c5: NTT and
             ct x pt MAC / decrypt sweep points -- each with the CPU oracle
             beside it
  cpu_baseline  the oracle (the reference's kernels K:31-278 restated in
             C/OpenMP + numpy glue) on this host's cores, one warm MLP step

``--impl reference`` times that CPU path alone on the same config dict.

Multi-GPU (torchrun, N>1): data-parallel private training -- every rank
trains on its own batch of 64 (weak scaling); the loss gradients are scaled
by the global batch and the MO's revealed gradients are summed over ranks
with one NCCL all-reduce per layer before SGD (exact mod 2^59), which is
bit-identical to reference_train_step at batch 64 N.
"""

from __future__ import annotations

import argparse
import json
import os
import re
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
NONLINEAR = "dealer backend (SPEC:479: reconstruct, apply, reshare) for ReLU / truncation; no OT"
LAN_BPS = 384e6  # PAPER:777 LAN, for the census' wire-time estimate

# CUPTI kernel name -> the C-ABI entry point that launches it
KERNEL_ENTRY = {
    "k_enc_noise": "pb_encrypt_sk", "k_encrypt_sk": "pb_encrypt_sk", "k_encrypt_pre": "pb_encrypt_sk",
    "k_encrypt_add": "pb_encrypt_sk", "k_encode_plain_mont": "pb_encode_plain_mont",
    "k_mask_ntt": "pb_mask_ntt", "k_mac_ws": "pb_ctpt_mac_tiled", "k_mac_eager": "pb_ctpt_mac_tiled",
    "k_mask_mac": "pb_mask_mac", "k_nl": "pb_nl_op", "k_dealer": "pb_dealer_op_out",
    "k_decrypt_share_cluster": "pb_decrypt_to_share", "k_decrypt_inv": "pb_decrypt_to_share",
    "k_decode_gather": "pb_decrypt_to_share",
}


def _config(world):
    """The config dict both arms print."""
    return {"workload": "configs[1]: MNIST MLP 784-128-128-10 private training step", "global_batch": BATCH * world,
            "batch_per_gpu": BATCH, "bfv": "N=8192, t=2^59, L=7x30-bit (log2 Q = 210)", "f": 25,
            "parallelism": f"data-parallel x{world} (revealed-gradient all-reduce)" if world > 1 else "single GPU",
            "l2": "flushed (256 MiB write) between timed steps"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        hbm = (float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)")
    except Exception:
        hbm = (6650.0, "fallback (B200_PROFILING.md)")
    try:
        with open(os.path.join(ROOT, "profiles", "r01_int_peak.json")) as f:
            d = json.load(f)
        ip = {"imad": d["IMAD"]["ops_per_s"], "imad_wide": d["IMAD.WIDE.U32"]["ops_per_s"],
              "kind": "measured on B200 (scripts/int_peak.py -> profiles/r01_int_peak.json)"}
    except Exception:
        ip = {"imad": 128 * 148 * 1.965e9 / 2, "imad_wide": 24 * 148 * 1.965e9, "kind": "nominal"}
    return hbm, ip


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
                    self.samples.append([x.strip() for x in line.split(",")])
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
# The oracle: the reference's numeric kernels (K:31-278) restated in C/OpenMP
# (oracle/kernels.c) + numpy glue for the SPEC-only layers -- test / baseline
# infrastructure, executed only here and in tests/.

def _oracle_ctx(seed=SEED):
    from oracle import bfv as OB
    from oracle import kernels as OK
    from oracle import protocols as OPR
    from oracle import ring as OR
    from oracle.params import make_params

    OK.set_threads(os.cpu_count() or 1)
    ring = OR.RingParams()
    p = make_params(8192, 7)
    ar = OB.Arith(p)
    kp = OB.keygen(p, OR.SeededRng(seed, 0), ar)
    return OPR.Ctx(p, ring, kp, seed=seed, ar=ar), OK.get_threads()


def cpu_model_steps(name, B, steps, warmup):
    """Seconds per oracle private step of model ``name`` at batch B (after warm-up)."""
    from oracle import nn as ON

    ctx, cores = _oracle_ctx()
    model = ON.Model(name, ctx.ring, seed=SEED)
    if len(model.in_shape) == 1:
        x, labels = ON.synthetic_mnist(SEED, B, ctx.ring)
    else:
        x, labels = ON.synthetic_images(SEED, B, model.in_shape, ctx.ring)
    for i in range(warmup):
        ctx.seed = SEED + 100 + i
        ON.private_train_step(ctx, model, x, labels)
    t0 = time.perf_counter()
    for i in range(steps):
        ctx.seed = SEED + 1 + i
        ON.private_train_step(ctx, model, x, labels)
    return (time.perf_counter() - t0) / steps, cores


def cpu_c5():
    """The oracle's C5 primitives on the host (N=8192, L=7): NTT rows/s, ct x pt
    MACs/s (K:89-95 pw_mul_acc over both ciphertext polys), decrypt
    ciphertexts/s (c0 + c1 s, INTT, Garner + scale-round, K:53-77, 158-199)."""
    from oracle import kernels as OK

    ctx, cores = _oracle_ctx()
    p, ar = ctx.p, ctx.ar
    L, N = 7, 8192
    rng = np.random.default_rng(0)
    q = p.tables["q"]
    out = {"cores": cores, "kind": "port"}
    rows = rng.integers(0, 1 << 62, size=(L * 128, N), dtype=np.uint64) % np.tile(q, 128)[:, None]
    OK.ntt_forward_cyc(rows[:L].copy(), p.tables["psi_brv"], q)  # warm-up
    t0 = time.perf_counter()
    OK.ntt_forward_cyc(rows, p.tables["psi_brv"], q)
    dt = time.perf_counter() - t0
    out["ntt_fwd"] = {"rows_per_s": rows.shape[0] / dt, "GB_s": rows.shape[0] * N * 8 / dt / 1e9,
                      "sample": f"{rows.shape[0]} rows, N={N} (GB/s at 4 B/residue read + write)"}
    nct, nI = 16, 8
    ct = rows[: 2 * L * nct].reshape(nct, 2, L, N)
    pt = rows[2 * L * nct: 2 * L * nct + L * nI].reshape(nI, L, N)
    acc = np.zeros((nct, L, N), dtype=np.uint64)
    t0 = time.perf_counter()
    for k in range(nI):  # out[b] += ct[b] (*) pt[k] for both polys: nct * nI ct x pt MACs
        for c in range(2):
            ar.mac(acc, np.ascontiguousarray(ct[:, c]), pt[k])
    dt = time.perf_counter() - t0
    out["ctpt_mac"] = {"ctpt_macs_per_s": nct * nI / dt, "mod_macs_per_s": nct * nI * 2 * L * N / dt,
                       "sample": f"{nct * nI} ct x pt MACs (K:89-95 pw_mul_acc)"}
    sk = ctx.kp.sk_ntt if hasattr(ctx.kp, "sk_ntt") else ctx.kp.s_ntt
    t0 = time.perf_counter()
    m = ar.mul(np.ascontiguousarray(ct[:8, 1]), np.asarray(sk).reshape(L, N))
    m = ar.add(m, np.ascontiguousarray(ct[:8, 0]))
    ar.ntt_inv(m)
    ar.decode(m)
    dt = time.perf_counter() - t0
    out["decrypt"] = {"ct_per_s": 8 / dt, "sample": "8 ciphertexts: c0 + c1 s, INTT, Garner + scale-round"}
    return out


def run_reference(args, rank, world):
    """--impl reference: the oracle private MLP step on this host's cores."""
    if rank != 0:
        return
    warm = max(3, args.warmup)
    t1, cores = cpu_model_steps("mnist_mlp", BATCH, 1, 1)
    budget = 240.0  # bound the run to a few minutes
    steps_run = max(1, min(args.steps, int(budget / max(t1, 1e-3)) - warm))
    dt, cores = cpu_model_steps("mnist_mlp", BATCH, steps_run, warm - 1)
    v = BATCH / dt
    sample = (f"{steps_run} oracle private training step(s) of the MNIST MLP 784-128-128-10, B={BATCH}, N=8192, "
              f"L=7, after {warm} in-process warm-up steps (oracle = reference kernels restated in C/OpenMP + numpy)"
              + (f"; rank 0 of {world} alone, one host process" if world > 1 else ""))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world,
        "steps": steps_run, "warmup": warm, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak" if world > 1 else "n/a", "vs_baseline": None, "dtype": "u32-rns/u64-ring",
        "data": "synthetic", "config": _config(world), "nonlinear": NONLINEAR,  # the GPU arm's config
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU leg ----

def _short(name):
    n = re.sub(r"^void ", "", name.strip()).replace("(anonymous namespace)::", "")
    n = re.sub(r"<.*", "", n)
    n = re.sub(r"\(.*", "", n)
    return n.split("::")[-1].strip()


def cupti_kernels(fn, n):
    """Device time (ms) and launches per call of ``fn`` for every engine kernel,
    from CUPTI activity records (torch.profiler) over n calls."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(n):
            fn(i)
        torch.cuda.synchronize()
    per = {}
    for ev in prof.key_averages():
        t = getattr(ev, "device_time_total", None)
        if t is None:
            t = getattr(ev, "cuda_time_total", 0.0)
        nm = _short(ev.key)
        if not nm.startswith("k_") or ev.count == 0:
            continue
        acc = per.setdefault(nm, [0.0, 0.0])
        acc[0] += t / 1e3 / n
        acc[1] += ev.count / n
    return per


def _time_steps(fn, steps, flush, join=None):
    import torch

    evs = []
    for i in range(steps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn(i)
        if join is not None:
            join()
        e.record()
        evs.append((s, e))
    torch.cuda.synchronize()
    return sum(s.elapsed_time(e) for s, e in evs)  # ms


def _max_over_ranks(v, world):
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _roofline(name, ms, launches, nbytes, work, hbm, ip):
    """HBM and integer-pipe fractions of one entry point per step."""
    ntt_rows, mod_macs = work
    d = {"kernel": name, "ms_per_step": ms, "launches_per_step": launches, "ms_per_launch": ms / max(launches, 1e-9)}
    ach = nbytes / (ms / 1e3) / 1e9 if ms else 0.0
    d.update({"hbm_GBs": ach, "hbm_frac": ach / hbm[0], "alg_bytes_per_step": nbytes})
    slots = ntt_rows * (8192 // 2) * 13 * 4  # Harvey butterflies x (2 IMAD + IMAD.HI = 4 issue slots)
    if slots and ms:
        d["int_ops_per_s"] = slots / (ms / 1e3)
        d["int_frac"] = d["int_ops_per_s"] / ip["imad"]
        d["int_model"] = "NTT butterflies x 4 IMAD issue slots / measured IMAD peak (RNG, gathers not counted)"
    elif mod_macs and ms:
        d["int_ops_per_s"] = mod_macs / (ms / 1e3)
        d["int_frac"] = d["int_ops_per_s"] / ip["imad_wide"]
        d["int_model"] = "lazy mod-MACs (1 IMAD.WIDE.U32 each) / measured IMAD.WIDE.U32 peak"
    return d


def run_ours(args, rank, world):
    import torch

    from paper_2403_11166_b200 import _dev, _lib, bfv
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.linear_protocols import Session
    from paper_2403_11166_b200.params import BfvParams
    from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed

    dev = _dev.device()
    hbm, ip = _peaks()
    ring = RingParams()
    params = BfvParams()
    kp = bfv.keygen(params, SeededRng(SEED, 0))
    sess = Session(params, ring, kp, seed=SEED)
    model = PN.Model(SIZES, ring, seed=SEED)
    if world > 1:
        import torch.distributed as dist

        model.set_data_parallel(dist.group.WORLD, world)  # revealed gradients summed over ranks before SGD
    xh, labels = PN.synthetic_mnist(SEED + rank, BATCH, ring)  # every rank its own batch
    x_dev = RingTensor(encode_fixed(xh, ring), ring.f, ring, _canonical=True)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.int64, device=dev)  # > 126 MB L2
    warm = max(3, args.warmup)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    # ---- one instrumented eager step: algorithmic bytes / work per entry point
    for i in range(2):
        sess.reseed(SEED + 10 + i)
        PN.private_train_step(sess, model, x_dev, labels, check=False)
    torch.cuda.synchronize()
    sess.alg_bytes.clear()
    sess.alg_work.clear()
    _lib.STATS = _lib.CallStats()
    sess.reseed(SEED + 500)
    PN.private_train_step(sess, model, x_dev, labels, check=False)
    torch.cuda.synchronize()
    _lib.STATS = None
    alg, work = dict(sess.alg_bytes), {k: list(v) for k, v in sess.alg_work.items()}
    census_per_step = sess.channel.total_bytes() / max(1, sess.steps_seen)

    # ---- the step replayed from CUDA graphs (GraphStep): what `value` times
    runner = PN.GraphStep(sess, model, x_dev, prefetch_input=True)
    for i in range(warm):
        runner.step(SEED + 100 + i, labels)
    torch.cuda.synchronize()
    # per-kernel device times from CUPTI over graph replays (outside the timed region)
    per = cupti_kernels(lambda i: (runner.step(SEED + 300 + i, labels), runner.join_prefetch()), 3)
    launches_per_step = sum(v[1] for v in per.values())

    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    t_ms = _time_steps(lambda i: runner.step(SEED + 1000 + i, labels), args.steps, flush, runner.join_prefetch)
    barrier()
    clk = clocks.stop()
    t_ms = _max_over_ranks(t_ms, world)
    value = world * args.steps * BATCH / (t_ms / 1e3)

    # ---- e2e through the public API: host batch (pinned) -> device every step, loss back on the host
    x_pin = torch.from_numpy(np.ascontiguousarray(xh)).pin_memory()
    torch.cuda.synchronize()
    barrier()

    # pipelined data loading through the public API: every timed step runs the
    # step on the staged batch and stages the next one (pinned H2D + device
    # encode + the DO's input encryption, overlapping this step's backward);
    # the first batch is staged before the timed region
    runner.load_batch(x_pin)

    def e2e_step(i):
        runner.step(SEED + 2000 + i, labels, next_batch=x_pin)

    te_ms = _max_over_ranks(_time_steps(e2e_step, args.steps, flush, runner.join_prefetch), world)
    e2e = {"value": world * args.steps * BATCH / (te_ms / 1e3), "unit": "samples/s",
           # per step: batch H2D + DO loss-gradient H2D; logits D2H (DO reconstructs) + encode range flag
           "h2d_bytes_per_step": x_pin.numel() * 8 + 10 * BATCH * 8, "d2h_bytes_per_step": 10 * BATCH * 8 + 4}

    # ---- kernels grouped by entry point; the dominant one carries the roofline
    entries = {}
    for k, (ms, n) in per.items():
        e = KERNEL_ENTRY.get(k, k)
        acc = entries.setdefault(e, [0.0, 0.0])
        acc[0] += ms
        acc[1] += n
    kernels = {e: _roofline(e, ms, n, alg.get(e, 0.0), work.get(e, [0.0, 0.0]), hbm, ip)
               for e, (ms, n) in sorted(entries.items(), key=lambda kv: -kv[1][0])}
    dom = next(iter(kernels))
    r = kernels[dom]
    calls = max(1.0, r["launches_per_step"] / (2.0 if dom == "pb_encrypt_sk" else 1.0))
    roofline = {"bound": "hbm", "kernel": dom, "achieved": r["hbm_GBs"], "peak": hbm[0], "unit": "GB/s",
                "frac": r["hbm_frac"], "peak_kind": hbm[1], "traffic": None,
                "traffic_note": "the step's working set is L2-resident: ncu DRAM bytes per launch are far below "
                                "the algorithmic bytes (profiles/r02_*)",
                "bytes_per_launch": r["alg_bytes_per_step"] / calls, "ms_per_launch": r["ms_per_step"] / calls,
                "share_of_step": r["ms_per_step"] / (t_ms / args.steps),
                "timing": "CUPTI device time over 3 graph-replayed steps (torch.profiler)"}
    if "int_frac" in r:
        roofline["int_pipe"] = {"achieved": r["int_ops_per_s"], "unit": "ops/s", "frac": r["int_frac"],
                                "peak": ip["imad"] if "NTT" in r["int_model"] else ip["imad_wide"],
                                "model": r["int_model"], "peak_kind": ip["kind"]}

    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if world > 1 else "n/a", "vs_baseline": None, "dtype": "u32-rns/u64-ring",
        "data": "synthetic", "config": _config(world), "nonlinear": NONLINEAR,
        "e2e": e2e, "roofline": roofline, "clocks": clk,
        "gpu_launches": int(round(launches_per_step * args.steps)), "kernels": kernels,
        "census_bytes_per_step": census_per_step,
        "census_wire_s_at_384MBps": census_per_step / LAN_BPS,
        "timing": "value/e2e: K graph-replayed steps (CUDA events, max over ranks), each joined with the next "
                  "step's prefetched input encryption; per-kernel: CUPTI",
    }
    del runner
    torch.cuda.empty_cache()
    if not args.no_configs:
        line["configs"] = {"c1": bench_c1(args) if world == 1 else None,
                           "c3": bench_c4(args, rank, world, "mnist_cnn2"),
                           "c4": bench_c4(args, rank, world), "c5": bench_c5(args),
                           "c2_ot_nonlinear": bench_c4(args, rank, world, "mnist_mlp", "ot"),
                           "c4_ot_nonlinear": bench_c4(args, rank, world, "cifar_cnn", "ot"),
                           "c2_prep_online": bench_c4(args, rank, world, "mnist_mlp", prep_m=8),
                           "c4_prep_online": bench_c4(args, rank, world, "cifar_cnn", prep_m=8)}
    if rank != 0:
        return
    if not args.no_cpu and world == 1:
        dt, cores = cpu_model_steps("mnist_mlp", BATCH, 1, 1)
        line["cpu_baseline"] = {
            "value": BATCH / dt, "unit": "samples/s", "cores": cores, "kind": "port",
            "sample": "1 oracle private training step (MNIST MLP, B=64, N=8192, L=7) after 1 warm-up step "
                      "(the reference kernels restated in C/OpenMP + numpy glue)"}
        if "configs" in line:
            dt4, cores4 = cpu_model_steps("cifar_cnn", 4, 1, 0)
            line["configs"]["c4"]["cpu"] = {
                "value": 4 / dt4, "unit": "samples/s", "cores": cores4, "kind": "port",
                "sample": "1 oracle private CIFAR-CNN step at B=4 (bounded sample of configs[3]; B=64 takes minutes)"}
            line["configs"]["c5"]["cpu"] = cpu_c5()
            line["configs"]["c1"]["cpu"] = cpu_c1()
    else:
        line["cpu_baseline"] = None
    print(json.dumps(line), flush=True)


def bench_c4(args, rank, world, name="cifar_cnn", nonlinear="dealer", prep_m=0):
    """configs[3]: CIFAR-10 CNN (PAPER Fig. 7) private step, B=64 per GPU, graph
    replay; ``nonlinear="ot"``: ReLU / truncation / pooling through the
    OT-based protocols (dealer OT functionality) instead of the
    dealer's reconstruct-reshare; ``prep_m``: SPEC mode "prep" (Pencil+,
    PAPER Alg. 3/4) -- the offline mask banks (m^2 HE evaluations per
    operator) built first and timed separately, the step is the HE-free
    online phase."""
    import torch

    from paper_2403_11166_b200 import bfv
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.linear_protocols import Session
    from paper_2403_11166_b200.params import BfvParams
    from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed

    ring, params = RingParams(), BfvParams()
    sess = Session(params, ring, bfv.keygen(params, SeededRng(SEED, 0)), seed=SEED)
    sess.nonlinear = nonlinear
    model = PN.Model(name, ring, seed=SEED)
    if world > 1:
        import torch.distributed as dist

        model.set_data_parallel(dist.group.WORLD, world)
    if len(model.in_shape) == 1:
        xh, labels = PN.synthetic_mnist(SEED + rank, BATCH, ring)
    else:
        xh, labels = PN.synthetic_images(SEED + rank, BATCH, model.in_shape, ring)
    x = RingTensor(encode_fixed(xh, ring), ring.f, ring, _canonical=True)
    prep, bank_s = None, None
    if prep_m:
        from paper_2403_11166_b200 import preprocessing as PP

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prep = PP.PrepState(sess, model, BATCH, m=prep_m, bank_seed=SEED)
        torch.cuda.synchronize()
        bank_s = time.perf_counter() - t0
    runner = PN.GraphStep(sess, model, x, prep=prep)
    for i in range(3):
        runner.step(SEED + i, labels)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.int64, device="cuda")
    steps = max(3, min(args.steps, 10))
    torch.cuda.synchronize()
    ms = _max_over_ranks(_time_steps(lambda i: runner.step(SEED + 50 + i, labels), steps, flush), world) / steps
    per = cupti_kernels(lambda i: runner.step(SEED + 80 + i, labels), 1)
    agg = {}
    for k, v in per.items():
        e = KERNEL_ENTRY.get(k, k)
        agg[e] = agg.get(e, 0.0) + v[0]
    del runner
    torch.cuda.empty_cache()
    wl = {"cifar_cnn": "configs[3]: CIFAR-10 CNN (5 conv + FC, PAPER Fig. 7) private training step",
          "mnist_mlp": "configs[1]: MNIST MLP 784-128-128-10 private training step",
          "mnist_cnn2": "configs[2]: MNIST CNN (2 x conv5x5 + FC) private training step",
          "mnist_cnn": "configs[2] (PAPER Fig. 6 variant): MNIST CNN (conv5x5 + 2 FC) private training step"}[name]
    extra = {"mode": f"prep (Pencil+, m={prep_m})", "offline_bank_build_s": bank_s} if prep_m else {"mode": "fullhe"}
    return {"workload": wl, "nonlinear": nonlinear, **extra, "batch_per_gpu": BATCH, "value": world * BATCH / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms,
            "steps": steps, "kernels_ms_per_step": {k: round(v, 4) for k, v in
                                                    sorted(agg.items(), key=lambda kv: -kv[1])[:10]}}


def _fc_round_parts(B):
    """configs[0] operands: W (128x784), b, two-sided shares of x (784xB) and gy (128xB)."""
    rng = np.random.default_rng(1)
    W = rng.uniform(-0.03, 0.03, (128, 784))
    b = rng.uniform(-0.03, 0.03, 128)
    x = rng.uniform(-1, 1, (784, B))
    gy = rng.normal(0, 0.01, (128, B))
    return W, b, x, gy


def bench_c1(args):
    """configs[0]: one FC layer 784->128 private round -- linear_forward,
    reveal_grad_bias, grad_weight (Alg. 2) and linear_backward_input on
    two-sided shares, B=64 -- replayed from one CUDA graph, with the oracle's
    same round on the host cores beside it."""
    import torch

    from paper_2403_11166_b200 import bfv
    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200.linear_protocols import Session
    from paper_2403_11166_b200.params import BfvParams
    from paper_2403_11166_b200.ring import DO, MO, RingParams, RingTensor, SeededRng, ShareTensor, encode_fixed

    ring, params = RingParams(), BfvParams()
    sess = Session(params, ring, bfv.keygen(params, SeededRng(SEED, 0)), seed=SEED)
    Wf, bf, xf, gf = _fc_round_parts(BATCH)

    def enc(a, sc=25):
        return RingTensor(encode_fixed(a, ring, sc), sc, ring, _canonical=True)

    W, b = enc(Wf), enc(bf, 50)
    x, gy = encode_fixed(xf, ring), encode_fixed(gf, ring)
    xm = SeededRng(5, 1).uniform_ring(x.shape, ring)
    gm = SeededRng(5, 2).uniform_ring(gy.shape, ring)
    m = (1 << ring.ell) - 1
    xs = (ShareTensor(MO, RingTensor(xm, 25, ring, _canonical=True)),
          ShareTensor(DO, RingTensor((x - xm) & m, 25, ring, _canonical=True)))
    gs = (ShareTensor(MO, RingTensor(gm, 25, ring, _canonical=True)),
          ShareTensor(DO, RingTensor((gy - gm) & m, 25, ring, _canonical=True)))

    def rnd(i):
        sess.reseed(SEED + 50 + i)
        LP.linear_forward(sess, 1, W, b, *xs)
        LP.reveal_grad_bias(sess, 1, *gs)
        LP.grad_weight(sess, 1, *xs, *gs)
        LP.linear_backward_input(sess, 1, W, *gs)
        sess.join_side()

    sess.enable_graph_mode()
    for i in range(3):
        rnd(100 + i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        rnd(200)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.int64, device="cuda")
    for i in range(3):
        g.replay()
    steps = max(3, min(args.steps, 20))

    def replay(i):
        sess.reseed(SEED + 300 + i)
        g.replay()

    torch.cuda.synchronize()
    ms = _time_steps(replay, steps, flush) / steps
    del g, flush
    torch.cuda.empty_cache()
    return {"workload": "configs[0]: one FC layer 784->128 private round (forward, bias reveal, Alg. 2 weight "
                        "gradient, input gradient) on two-sided shares, B=64", "batch": BATCH,
            "value": BATCH / (ms / 1e3), "unit": "samples/s", "ms_per_round": ms, "steps": steps,
            "timing": "one CUDA graph per round, L2 flushed between rounds"}


def cpu_c1():
    """The oracle's configs[0] round on the host cores (one round after one warm-up)."""
    from oracle import bfv as OB
    from oracle import kernels as OK
    from oracle import protocols as OPR
    from oracle import ring as OR
    from oracle.params import make_params

    OK.set_threads(os.cpu_count() or 1)
    R = OR.RingParams()
    p = make_params(8192, 7)
    ar = OB.Arith(p)
    ctx = OPR.Ctx(p, R, OB.keygen(p, OR.SeededRng(SEED, 0), ar), seed=SEED, ar=ar)
    Wf, bf, xf, gf = _fc_round_parts(BATCH)
    W, b = OR.encode_fixed(Wf, R), OR.encode_fixed(bf, R, 50)
    x, gy = OR.encode_fixed(xf, R), OR.encode_fixed(gf, R)
    xm, gm = OR.SeededRng(5, 1).uniform_ring(x.shape, R), OR.SeededRng(5, 2).uniform_ring(gy.shape, R)
    xd, gd = (x - xm) & R.mask, (gy - gm) & R.mask

    def rnd():
        OPR.linear_forward(ctx, 1, W, b, xm, xd)
        OPR.reveal_grad_bias(ctx, 1, gm, gd)
        OPR.grad_weight(ctx, 1, xm, xd, gm, gd)
        OPR.linear_backward_input(ctx, 1, W, gm, gd)

    rnd()
    t0 = time.perf_counter()
    rnd()
    dt = time.perf_counter() - t0
    return {"value": BATCH / dt, "unit": "samples/s", "s_per_round": dt, "cores": OK.get_threads(), "kind": "port",
            "sample": "1 oracle round of configs[0] after 1 warm-up round"}


def bench_c5(args):
    """configs[4] points at N=8192, L=7: NTT fwd / inv over 1 GiB of residues,
    ct x pt MAC (FC-like K=1, conv-like K=16), decrypt-to-share of 1024 cts."""
    import torch

    from paper_2403_11166_b200 import _dev, _lib, bfv
    from paper_2403_11166_b200.params import BfvParams, context
    from paper_2403_11166_b200.ring import SeededRng

    hbm, ip = _peaks()
    p = BfvParams()
    ctx = context(p)
    L, N = p.L, p.N
    st = _dev.stream()
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.int64, device="cuda")

    def t(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        return _time_steps(lambda i: fn(), reps, flush) / reps

    out = {"workload": "configs[4] points: N=8192, L=7 (set A); L2 flushed before every timed launch"}
    rows = (1 << 30) // (4 * N)
    rows -= rows % L
    x = torch.randint(0, p.moduli[-1], (rows, N), dtype=torch.int32, device="cuda")
    for nm, fn in (("ntt_fwd", "pb_ntt_forward"), ("ntt_inv", "pb_ntt_inverse")):
        ms = t(lambda: _lib.call(fn, ctx.handle, x.data_ptr(), rows, None, st))
        by = rows * N * 8
        bf = rows * (N // 2) * 13 * 4
        out[nm] = {"rows": rows, "ms": ms, "rows_per_s": rows / (ms / 1e3), "GB_s": by / ms / 1e6,
                   "hbm_frac": by / ms / 1e6 / hbm[0], "int_frac": bf / (ms / 1e3) / ip["imad"]}
    del x
    for tag, (nB, nO, nI) in (("mac_fc_k1", (64, 13, 1)), ("mac_conv_k16", (64, 13, 16))):
        ct = torch.randint(0, p.moduli[-1], (nB * nI, 2, L, N), dtype=torch.int32, device="cuda")
        pt = torch.randint(0, p.moduli[-1], (nO * nI, L, N), dtype=torch.int32, device="cuda")
        o = torch.empty((nB * nO, 2, L, N), dtype=torch.int32, device="cuda")
        ms = t(lambda: _lib.call("pb_ctpt_mac_tiled", ctx.handle, ct.data_ptr(), pt.data_ptr(), None, None, nB, nO,
                                 nI, o.data_ptr(), st))
        by = 4 * L * N * (2 * nB * nI + nO * nI + 2 * nB * nO)
        mm = nB * nO * nI * 2 * L * N
        out[tag] = {"B_ct": nB, "O_pt": nO, "K": nI, "ms": ms, "ctpt_macs_per_s": nB * nO * nI / (ms / 1e3),
                    "GB_s": by / ms / 1e6, "hbm_frac": by / ms / 1e6 / hbm[0],
                    "int_frac": mm / (ms / 1e3) / ip["imad_wide"]}
        if nI == 1:  # the MO's whole K=1 evaluation fused with the mask NTT (pb_mask_mac)
            U = 128
            pos = (torch.arange(U, dtype=torch.int32, device="cuda") * 61 % N).repeat(nB * nO, 1).contiguous()
            dst = torch.arange(nB * nO * U, dtype=torch.int64, device="cuda")
            mask = torch.randint(0, 1 << 59, (nB * nO * U,), dtype=torch.int64, device="cuda")
            ms = t(lambda: _lib.call("pb_mask_mac", ctx.handle, ct.data_ptr(), pt.data_ptr(), None, None, nB, nO, nI,
                                     pos.data_ptr(), dst.data_ptr(), U, mask.data_ptr(), 1, 7, None, o.data_ptr(), st))
            by2 = by + 8 * nB * nO * U
            out["mask_mac_fc_k1"] = {"B_ct": nB, "O_pt": nO, "K": nI, "ms": ms,
                                     "ctpt_macs_per_s": nB * nO * nI / (ms / 1e3), "GB_s": by2 / ms / 1e6,
                                     "hbm_frac": by2 / ms / 1e6 / hbm[0],
                                     "note": "mask NTT (-Delta NTT(mask + filler)) + K=1 MAC in one pass"}
            del pos, dst, mask
        del ct, pt, o
    kp = bfv.keygen(p, SeededRng(SEED, 0))
    n, U = 1024, 128
    ct = torch.randint(0, p.moduli[-1], (n, 2, L, N), dtype=torch.int32, device="cuda")
    pos = (torch.arange(U, dtype=torch.int32, device="cuda") * 61 % N).repeat(n, 1).contiguous()
    dst = torch.arange(n * U, dtype=torch.int64, device="cuda")
    share = torch.empty(n * U, dtype=torch.int64, device="cuda")
    scratch = torch.empty((n, L, U), dtype=torch.int32, device="cuda")
    ms = t(lambda: _lib.call("pb_decrypt_to_share", ctx.handle, _dev.ptr(kp.sk_ntt), ct.data_ptr(), n,
                             pos.data_ptr(), dst.data_ptr(), U, share.data_ptr(), scratch.data_ptr(), st))
    by = n * (2 * L * N * 4 + 8 * U)
    out["decrypt_to_share"] = {"cts": n, "useful_slots": U, "ms": ms, "ct_per_s": n / (ms / 1e3),
                               "GB_s": by / ms / 1e6, "hbm_frac": by / ms / 1e6 / hbm[0]}
    del ct, share, scratch
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--no-configs", action="store_true", help="headline only (no c4 / c5 objects)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        if args.impl == "ours":  # the reference arm is host-only (gloo): no device needed
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
