"""Throughput of every BASELINE.json config on one B200 (bench.py times
configs[1] only; this script covers the rest and writes one JSON line per
measurement).

    python scripts/bench_configs.py [c1 c2 c3 c4 c5] [--steps K] [--cpu]

c1  single FC layer 784->128, B=64: one private fwd + bwd round
    (linear_forward, reveal_grad_bias, grad_weight, linear_backward_input)
c2  MNIST MLP 784-128-128-10 private training step, B=64
c3  MNIST CNN (2 x conv5x5 + FC, "mnist_cnn2") private training step, B=64
    (also the paper's 1-conv "mnist_cnn")
c4  CIFAR-10 CNN (PAPER Fig. 7, 5 conv + FC) private training step, B=64
c2p/c3p/c4p  the same models in SPEC mode "prep" (Pencil+, Alg. 3/4, m=8):
    offline bank build time and the HE-free online step
c5  NTT fwd/inv sweep N=4096..32768, L=2..8 over >= 1 GiB of residues, and
    the ct x pt MAC operator (pb_ctpt_mac_tiled) at FC-like (B_ct=64, O_pt=13,
    K=1) and conv-like (K=16) shapes

Timing: CUDA events on the launching stream, >= 3 warm-up steps, the L2
flushed (256 MiB write) before every timed step, steps replayed from CUDA
graphs (nn.GraphStep) -- the same kernels as the eager path.  --cpu adds the
oracle (the reference's CPU algorithm, C/OpenMP + numpy) on this host for
c1-c3 (c4's oracle step takes minutes and is skipped).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2403_11166_b200 import _dev, _lib, bfv  # noqa: E402
from paper_2403_11166_b200 import nn as PN  # noqa: E402
from paper_2403_11166_b200.linear_protocols import Session  # noqa: E402
from paper_2403_11166_b200.params import BfvParams, context  # noqa: E402
from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed  # noqa: E402

SEED, B = 2024, 64
HBM = 6551.0


def _peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def _flush_buf():
    return torch.empty(256 * 1024 * 1024 // 8, dtype=torch.int64, device="cuda")


def time_steps(fn, steps, warm=3, flush=None):
    for _ in range(warm):
        fn(-1)
    torch.cuda.synchronize()
    tot = 0.0
    for i in range(steps):
        if flush is not None:
            flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn(i)
        e.record()
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    return tot / steps  # ms


def model_step(name, steps, cpu, prep_m=0):
    ring, params = RingParams(), BfvParams()
    sess = Session(params, ring, bfv.keygen(params, SeededRng(SEED, 0)), seed=SEED)
    model = PN.Model(name, ring, seed=SEED)
    if len(model.in_shape) == 1:
        xh, labels = PN.synthetic_mnist(SEED, B, ring)
    else:
        xh, labels = PN.synthetic_images(SEED, B, model.in_shape, ring)
    x = RingTensor(encode_fixed(xh, ring), ring.f, ring, _canonical=True)
    flush = _flush_buf()
    prep, prep_s = None, None
    if prep_m:
        from paper_2403_11166_b200 import preprocessing as PP

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prep = PP.PrepState(sess, model, B, m=prep_m, bank_seed=SEED)
        torch.cuda.synchronize()
        prep_s = time.perf_counter() - t0
    # eager (kernel-time breakdown + launch count)
    stats = _lib.CallStats(timed=("pb_ctpt_mac_tiled", "pb_mask_ntt", "pb_decrypt_to_share", "pb_encrypt_sk",
                                  "pb_encrypt_sk_add", "pb_encrypt_sk_zero", "pb_encode_plain_mont", "pb_ring_conv"))
    for i in range(2):
        sess.reseed(SEED + i)
        PN.private_train_step(sess, model, x, labels, check=False, prep=prep)
    torch.cuda.synchronize()
    _lib.STATS = stats
    flush.zero_()
    sess.reseed(SEED + 7)
    t0 = time.perf_counter()
    PN.private_train_step(sess, model, x, labels, check=False, prep=prep)
    torch.cuda.synchronize()
    eager_s = time.perf_counter() - t0
    _lib.STATS = None
    per = {}
    for nm, s, e, _ in stats.events:
        per[nm] = per.get(nm, 0.0) + s.elapsed_time(e)
    runner = PN.GraphStep(sess, model, x, prep=prep, prefetch_input=prep is None)  # as bench.py
    ms = time_steps(lambda i: runner.step(SEED + 100 + i, labels), steps, flush=flush)
    out = {"config": name + (f"+prep(m={prep_m})" if prep_m else ""), "batch": B, "ms_per_step": ms, "samples_per_s": B / (ms / 1e3),
           "eager_wall_ms": eager_s * 1e3, "launches_per_step": stats.launches,
           "kernel_ms": {k: round(v, 4) for k, v in sorted(per.items(), key=lambda kv: -kv[1])}}
    if prep_m:
        out["offline_bank_build_s"] = prep_s
        out["online_census_bytes_per_step"] = sum(v[1] for k, v in sess.channel.census.items() if k in (0x42, 0x43)) / 4
    if cpu:
        out["cpu"] = cpu_model_step(name)
    return out


def cpu_model_step(name):
    from oracle import bfv as OB
    from oracle import kernels as OK
    from oracle import nn as ON
    from oracle import protocols as OPR
    from oracle import ring as OR
    from oracle.params import make_params

    OK.set_threads(os.cpu_count() or 1)
    ring = OR.RingParams()
    p = make_params(8192, 7)
    ar = OB.Arith(p)
    ctx = OPR.Ctx(p, ring, OB.keygen(p, OR.SeededRng(SEED, 0), ar), seed=SEED, ar=ar)
    model = ON.Model(name, ring, seed=SEED)
    if len(model.in_shape) == 1:
        x, labels = ON.synthetic_mnist(SEED, B, ring)
    else:
        x, labels = ON.synthetic_images(SEED, B, model.in_shape, ring)
    ON.private_train_step(ctx, model, x, labels)  # warm-up
    t0 = time.perf_counter()
    ctx.seed = SEED + 1
    ON.private_train_step(ctx, model, x, labels)
    dt = time.perf_counter() - t0
    return {"s_per_step": dt, "samples_per_s": B / dt, "cores": OK.get_threads(), "kind": "port"}


def fc_round(steps, cpu):
    """c1: one FC layer 784->128 private fwd + bwd round with two-sided shares."""
    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200.ring import DO, MO, ShareTensor

    ring, params = RingParams(), BfvParams()
    sess = Session(params, ring, bfv.keygen(params, SeededRng(SEED, 0)), seed=SEED)
    rng = np.random.default_rng(1)
    n_i, n_o = 784, 128

    def enc(a, sc=25):
        return RingTensor(encode_fixed(a, ring, sc), sc, ring, _canonical=True)

    W, b = enc(rng.uniform(-0.03, 0.03, (n_o, n_i))), enc(rng.uniform(-0.03, 0.03, n_o), 50)
    x = encode_fixed(rng.uniform(-1, 1, (n_i, B)), ring)
    gy = encode_fixed(rng.normal(0, 0.01, (n_o, B)), ring)
    xm = SeededRng(5, 1).uniform_ring((n_i, B), ring)
    gm = SeededRng(5, 2).uniform_ring((n_o, B), ring)
    xs = (ShareTensor(MO, RingTensor(xm, 25, ring, _canonical=True)),
          ShareTensor(DO, RingTensor((x - xm) & ((1 << 59) - 1), 25, ring, _canonical=True)))
    gs = (ShareTensor(MO, RingTensor(gm, 25, ring, _canonical=True)),
          ShareTensor(DO, RingTensor((gy - gm) & ((1 << 59) - 1), 25, ring, _canonical=True)))

    def rnd(i):
        sess.reseed(SEED + 50 + i)
        LP.linear_forward(sess, 1, W, b, *xs)
        LP.reveal_grad_bias(sess, 1, *gs)
        LP.grad_weight(sess, 1, *xs, *gs)
        LP.linear_backward_input(sess, 1, W, *gs)

    ms_eager = time_steps(rnd, steps, flush=_flush_buf())
    # the same round replayed from one CUDA graph (seed indirection re-keys it per replay)
    sess.enable_graph_mode()
    for i in range(2):
        rnd(100 + i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        rnd(200)

    def replay(i):
        sess.reseed(SEED + 300 + i)
        g.replay()

    ms = time_steps(replay, steps, flush=_flush_buf())
    out = {"config": "fc784x128_round", "batch": B, "ms_per_round": ms, "samples_per_s": B / (ms / 1e3),
           "eager_ms_per_round": ms_eager, "note": "graph replay; eager_ms_per_round: the same calls launched eagerly"}
    if cpu:
        out["cpu"] = cpu_fc_round()
    return out


def cpu_fc_round():
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
    rng = np.random.default_rng(1)
    W = OR.encode_fixed(rng.uniform(-0.03, 0.03, (128, 784)), R)
    b = OR.encode_fixed(rng.uniform(-0.03, 0.03, 128), R, 50)
    x = OR.encode_fixed(rng.uniform(-1, 1, (784, B)), R)
    gy = OR.encode_fixed(rng.normal(0, 0.01, (128, B)), R)
    xm, gm = OR.SeededRng(5, 1).uniform_ring((784, B), R), OR.SeededRng(5, 2).uniform_ring((128, B), R)
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
    return {"s_per_round": dt, "samples_per_s": B / dt, "cores": OK.get_threads(), "kind": "port"}


def sweep(steps):
    """c5: NTT fwd/inv and ct x pt MAC throughput vs the HBM roofline."""
    peak = _peak()
    res = []
    st = _dev.stream()
    for N, L in ((4096, 2), (4096, 7), (8192, 2), (8192, 7), (16384, 4), (16384, 7), (32768, 8)):
        p = BfvParams(N=N, L=L)
        ctx = context(p)
        rows = (1 << 30) // (4 * N)
        rows -= rows % L
        x = torch.randint(0, p.moduli[-1], (rows, N), dtype=torch.int32, device="cuda")
        tf = time_steps(lambda i: _lib.call("pb_ntt_forward", ctx.handle, x.data_ptr(), rows, None, st), steps)
        ti = time_steps(lambda i: _lib.call("pb_ntt_inverse", ctx.handle, x.data_ptr(), rows, None, st), steps)
        by = rows * N * 4 * 2
        for nm, t in (("ntt_fwd", tf), ("ntt_inv", ti)):
            res.append({"kernel": nm, "N": N, "L": L, "rows": rows, "ms": t, "GB_s": by / t / 1e6,
                        "frac_hbm": by / t / 1e6 / peak, "rows_per_s": rows / (t / 1e3)})
        del x
        torch.cuda.empty_cache()
    for N, L in ((8192, 7), (4096, 4), (16384, 7)):
        p = BfvParams(N=N, L=L)
        ctx = context(p)
        for nB, nO, nI in ((64, 13, 1), (64, 13, 16)):
            ct = torch.randint(0, p.moduli[-1], (nB * nI, 2, L, N), dtype=torch.int32, device="cuda")
            pt = torch.randint(0, p.moduli[-1], (nO * nI, L, N), dtype=torch.int32, device="cuda")
            out = torch.empty((nB * nO, 2, L, N), dtype=torch.int32, device="cuda")
            t = time_steps(lambda i: _lib.call("pb_ctpt_mac_tiled", ctx.handle, ct.data_ptr(), pt.data_ptr(), None,
                                               None, nB, nO, nI, out.data_ptr(), st), steps, flush=_flush_buf())
            by = 4 * L * N * (2 * nB * nI + nO * nI + 2 * nB * nO)
            macs = nB * nO * nI
            res.append({"kernel": "ctpt_mac_tiled", "N": N, "L": L, "B_ct": nB, "O_pt": nO, "K": nI, "ms": t,
                        "ctpt_macs_per_s": macs / (t / 1e3), "mod_macs_per_s": macs * 2 * L * N / (t / 1e3),
                        "GB_s": by / t / 1e6, "frac_hbm": by / t / 1e6 / peak})
            del ct, pt, out
            torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="*", default=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--cpu", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for w in a.which:
        if w == "c1":
            print(json.dumps(fc_round(a.steps, a.cpu)), flush=True)
        elif w == "c2":
            print(json.dumps(model_step("mnist_mlp", a.steps, a.cpu)), flush=True)
        elif w == "c3":
            print(json.dumps(model_step("mnist_cnn2", a.steps, a.cpu)), flush=True)
            print(json.dumps(model_step("mnist_cnn", a.steps, a.cpu)), flush=True)
        elif w == "c4":
            print(json.dumps(model_step("cifar_cnn", a.steps, False)), flush=True)
        elif w == "c2p":
            print(json.dumps(model_step("mnist_mlp", a.steps, False, prep_m=8)), flush=True)
        elif w == "c3p":
            print(json.dumps(model_step("mnist_cnn2", a.steps, False, prep_m=8)), flush=True)
        elif w == "c4p":
            print(json.dumps(model_step("cifar_cnn", a.steps, False, prep_m=8)), flush=True)
        elif w == "c5":
            for r in sweep(a.steps):
                print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
