"""Multi-rank host logic on the CPU: the ciphertext-block
sharding of an HE matmul / conv over ``world`` ranks and the combine step.

* every output ciphertext of a block plan is owned by exactly one rank, and
  each rank's input / plaintext polynomial lists are exactly the ones its
  rectangle's MAC terms reference;
* world_size-2 ``gloo`` run: each rank evaluates its rectangle of the packed
  product in the clear (negacyclic products mod 2^64 of the packed
  polynomials -- the plaintext shadow of the ct x pt MAC), writes its useful
  slots into a compact tile, the ranks all-gather the tiles and scatter them
  through ``gather_maps`` -- the same combine the engine does with NCCL; the
  result must equal ``matmul_wrap`` / ``conv2d_wrap`` bit-for-bit;
* world_size-2 data-parallel private training (the oracle step with the
  revealed gradients summed over ranks, loss gradients over the global batch)
  equals ``reference_train_step`` on the concatenated batch.
"""

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import kernels as OK
from paper_2403_11166_b200.linear_protocols import gather_maps, shard_grid, shard_maps
from paper_2403_11166_b200.poly_encoding import ConvGeometry, MatmulGeometry, plan_conv, plan_matmul

MASK59 = np.uint64((1 << 59) - 1)


@pytest.mark.parametrize("nB,nO", [(1, 1), (1, 13), (64, 13), (3, 5), (8, 1), (2, 7)])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_grid_partitions(nB, nO, world):
    seen = np.zeros((nB, nO), dtype=int)
    for r in range(world):
        b0, b1, o0, o1 = shard_grid(nB, nO, r, world)
        assert 0 <= b0 <= b1 <= nB and 0 <= o0 <= o1 <= nO
        seen[b0:b1, o0:o1] += 1
    assert (seen == 1).all()


def _plans():
    return [
        plan_matmul(MatmulGeometry(40, 12, 9), 256),
        plan_matmul(MatmulGeometry(300, 7, 3), 256),
        plan_conv(ConvGeometry(3, 2, 3, 6, 6, 3), 256),
    ]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_maps_cover_outputs_once(world):
    for plan in _plans():
        owned = []
        for r in range(world):
            m = shard_maps(plan, r, world)
            nI = m["nI"]
            assert m["n_in"] == m["nb"] * nI and m["n_pt"] == m["no"] * nI
            assert m["in_src"].shape[0] == m["n_in"] and m["pt_src"].shape[0] == m["n_pt"]
            dst = m["out_dst"][m["out_pos"] >= 0]
            owned.append(dst)
        owned = np.concatenate(owned)
        full = plan.out_dst[plan.out_pos >= 0]
        assert len(owned) == len(full) and np.array_equal(np.sort(owned), np.sort(full))


def _packed(src_rows, vals, N):
    out = np.zeros((src_rows.shape[0], N), dtype=np.uint64)
    ok = src_rows >= 0
    out[ok] = vals[src_rows[ok]]
    return out


def eval_shard(plan, v, W, rank, world):
    """Rank's compact tile [n_max][U]: the useful slots of its output
    ciphertexts of sum_k pi_v(v) * pi_W(W) (gather_maps layout)."""
    m = shard_maps(plan, rank, world)
    n_max, _ = gather_maps(plan, world)
    N = plan.N
    vin = _packed(m["in_src"], v.ravel(), N)
    wpt = _packed(m["pt_src"], W.ravel(), N)
    tile = np.zeros((n_max, plan.U), dtype=np.uint64)
    for r in range(m["n_out"]):
        bi, oi = divmod(r, m["no"])
        acc = np.zeros(N, dtype=np.uint64)
        for k in range(m["nI"]):
            acc += OK.negacyclic_mul_wrap(vin[bi * m["nI"] + k], wpt[oi * m["nI"] + k])
        ok = m["out_pos"][r] >= 0
        tile[r, ok] = acc[m["out_pos"][r][ok]] & MASK59
    return tile.reshape(-1)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        res = []
        for plan in _plans():
            g = plan.geometry
            if plan.kind == "matmul":
                v = rng.integers(0, 1 << 59, size=(g.n_i, g.B), dtype=np.uint64)
                W = rng.integers(0, 1 << 59, size=(g.n_o, g.n_i), dtype=np.uint64)
                want = OK.matmul_wrap(W, v) & MASK59
            else:
                v = rng.integers(0, 1 << 59, size=(g.B, g.c_i, g.h, g.w), dtype=np.uint64)
                W = rng.integers(0, 1 << 59, size=(g.c_o, g.c_i, g.s, g.s), dtype=np.uint64)
                want = OK.conv2d_wrap(v, W) & MASK59
            tile = torch.from_numpy(eval_shard(plan, v, W, rank, world).view(np.int64).copy())
            parts = [torch.empty_like(tile) for _ in range(world)]
            dist.all_gather(parts, tile)
            _, gdst = gather_maps(plan, world)
            out = np.zeros(want.size, dtype=np.uint64)
            src = torch.cat(parts).numpy().view(np.uint64)
            out[gdst[gdst >= 0]] = src[gdst >= 0]  # pb_scatter_u64
            res.append(bool(np.array_equal(out.reshape(want.shape), want)))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_products_combine_exactly():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 2000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0] == out[1] and all(out[0]), out


def _dp_worker(rank, world, port, q):
    import copy

    import torch.distributed as dist

    from oracle import bfv as OB
    from oracle import nn as ON
    from oracle import protocols as PR
    from oracle import ring as OR
    from oracle.params import make_params

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        R = OR.RingParams()
        p = make_params(8192, 7)
        ar = OB.Arith(p)
        ctx = PR.Ctx(p, R, OB.keygen(p, OR.SeededRng(1, 0), ar), seed=31 + rank, ar=ar)
        m = ON.Model([784, 8, 10], R, seed=3)
        ref = copy.deepcopy(m)
        x, labels = ON.synthetic_mnist(9, 4 * world, R)  # the global batch; rank r trains on its quarter
        xs, ls = x[:, 4 * rank:4 * rank + 4], labels[4 * rank:4 * rank + 4]
        ok = True
        for step in range(2):
            _, gw, gb = ON.private_train_step(ctx, m, np.ascontiguousarray(xs), ls, dp_group=dist.group.WORLD)
            _, rgw, rgb = ON.reference_train_step(ref, x, labels)
            ok &= all(np.array_equal(a, b) for a, b in zip(gw, rgw)) and all(np.array_equal(a, b) for a, b in
                                                                                zip(gb, rgb))
            ok &= all(np.array_equal(a, b) for a, b in zip(m.w, ref.w))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_data_parallel_step_equals_reference_on_global_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + os.getpid() % 2000
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out == {0: True, 1: True}
