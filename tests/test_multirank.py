"""Multi-rank host logic on the CPU: the ciphertext-block
sharding of an HE matmul / conv over ``world`` ranks and the combine step.

* every output ciphertext of a block plan is owned by exactly one rank, and
  each rank's input / plaintext polynomial lists are exactly the ones its
  rectangle's MAC terms reference;
* world_size-2 ``gloo`` run: each rank evaluates its rectangle of the packed
  product in the clear (negacyclic products mod 2^64 of the packed
  polynomials -- the plaintext shadow of the ct x pt MAC), scatters its
  decoded outputs into a zero tile and the ranks all-reduce (SUM) -- the same
  combine the engine does with NCCL; the result must equal ``matmul_wrap`` /
  ``conv2d_wrap`` bit-for-bit.
"""

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import kernels as OK
from paper_2403_11166_b200.linear_protocols import shard_grid, shard_maps
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


def eval_shard(plan, v, W, rank, world, out_size):
    """Rank's decoded tile of pi_y^-1( sum_k pi_v(v) * pi_W(W) ), zero elsewhere."""
    m = shard_maps(plan, rank, world)
    N = plan.N
    vin = _packed(m["in_src"], v.ravel(), N)
    wpt = _packed(m["pt_src"], W.ravel(), N)
    tile = np.zeros(out_size, dtype=np.uint64)
    for r in range(m["n_out"]):
        bi, oi = divmod(r, m["no"])
        acc = np.zeros(N, dtype=np.uint64)
        for k in range(m["nI"]):
            acc += OK.negacyclic_mul_wrap(vin[bi * m["nI"] + k], wpt[oi * m["nI"] + k])
        ok = m["out_pos"][r] >= 0
        tile[m["out_dst"][r][ok]] = acc[m["out_pos"][r][ok]] & MASK59
    return tile


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
            tile = eval_shard(plan, v, W, rank, world, want.size)
            t = torch.from_numpy(tile.view(np.int64).copy())
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            res.append(bool(np.array_equal(t.numpy().view(np.uint64).reshape(want.shape), want)))
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
