"""Multi-rank engine paths on the GPU.

* Sharding: two ranks split every HE matmul / conv's output-ciphertext grid
  (Session(shard=...)) and combine the decrypted useful slots with an
  all-gather of compact tiles + pb_scatter_u64.  The box has one GPU, so both
  ranks share cuda:0 and the collective runs over gloo (host-staged -- no
  kernel waits on another rank's kernel); NCCL takes the same call.  The
  sharded shares and a full private training step equal the single-rank run.
* Data parallelism under NCCL inside CUDA graphs: a world-1 NCCL group drives
  Model.set_data_parallel (the revealed-gradient all-reduce) through
  GraphStep capture + replay; the steps equal the eager engine and the
  oracle.  (Two NCCL ranks cannot share one GPU: the sharded all-gather's
  NCCL form is the same torch call as the gloo one tested above.)"""

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _run(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2403_11166_b200 import bfv
    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.params import BfvParams
    from paper_2403_11166_b200.ring import DO, MO, RingParams, RingTensor, SeededRng, ShareTensor, encode_fixed

    torch.cuda.set_device(0)
    group = None
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        group = dist.group.WORLD
    try:
        ring, params = RingParams(), BfvParams()
        sess = LP.Session(params, ring, bfv.keygen(params, SeededRng(3, 0)), seed=11, shard=(rank, world, group))
        out = {}
        rng = np.random.default_rng(5)
        W = RingTensor(encode_fixed(rng.uniform(-0.1, 0.1, (48, 200)), ring), 25, ring)
        b = RingTensor(encode_fixed(rng.uniform(-0.1, 0.1, 48), ring, 50), 50, ring)
        x = encode_fixed(rng.uniform(-1, 1, (200, 16)), ring)
        xm = SeededRng(9, 1).uniform_ring((200, 16), ring)
        xs = (ShareTensor(MO, RingTensor(xm, 25, ring)), ShareTensor(DO, RingTensor(x - xm, 25, ring)))
        y = LP.linear_forward(sess, 1, W, b, *xs)
        out["fc_fwd"] = (y[0].value.numpy(), y[1].value.numpy())
        Wc = RingTensor(encode_fixed(rng.uniform(-0.2, 0.2, (6, 3, 3, 3)), ring), 25, ring)
        bc = RingTensor(encode_fixed(rng.uniform(-0.2, 0.2, 6), ring, 50), 50, ring)
        xc = encode_fixed(rng.uniform(-1, 1, (4, 3, 10, 10)), ring)
        xcm = SeededRng(9, 2).uniform_ring((4, 3, 10, 10), ring)
        xcs = (ShareTensor(MO, RingTensor(xcm, 25, ring)), ShareTensor(DO, RingTensor(xc - xcm, 25, ring)))
        yc = LP.conv_forward(sess, 2, Wc, bc, *xcs, 1, 2)
        out["conv_fwd"] = (yc[0].value.numpy(), yc[1].value.numpy())
        model = PN.Model([784, 32, 10], ring, seed=4)
        xh, labels = PN.synthetic_mnist(6, 8, ring)
        sess.reseed(77)
        loss, gw, gb = PN.private_train_step(sess, model, RingTensor(encode_fixed(xh, ring), 25, ring), labels)
        out["step"] = (loss, [g.numpy() for g in gw], [g.numpy() for g in gb])
        torch.cuda.synchronize()
        q.put((rank, out))
    finally:
        if world > 1:
            dist.destroy_process_group()


def _collect(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000 + world
    procs = [ctx.Process(target=_run, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_two_rank_sharding_matches_single_rank():
    one = _collect(1)[0]
    two = _collect(2)
    for r in (0, 1):
        got = two[r]
        for k in ("fc_fwd", "conv_fwd"):
            assert np.array_equal(got[k][0], one[k][0]) and np.array_equal(got[k][1], one[k][1]), (r, k)
        assert got["step"][0] == one["step"][0]
        for a, b in zip(got["step"][1] + got["step"][2], one["step"][1] + one["step"][2]):
            assert np.array_equal(a, b), r


def _nccl_graph(rank, port, q):
    import torch
    import torch.distributed as dist

    from oracle import nn as ON
    from oracle import ring as OR
    from paper_2403_11166_b200 import bfv
    from paper_2403_11166_b200 import linear_protocols as LP
    from paper_2403_11166_b200 import nn as PN
    from paper_2403_11166_b200.params import BfvParams
    from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed

    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        ring, params = RingParams(), BfvParams()
        kp = bfv.keygen(params, SeededRng(3, 0))
        sizes, B = [784, 32, 10], 8
        xh, labels = PN.synthetic_mnist(7, B, ring)
        g = dist.group.WORLD
        s_eager = LP.Session(params, ring, kp, seed=1)
        m_eager = PN.Model(sizes, ring, seed=4)
        s_graph = LP.Session(params, ring, kp, seed=1)
        m_graph = PN.Model(sizes, ring, seed=4)
        m_graph.set_data_parallel(g, 1)  # NCCL all-reduce of the revealed gradients, captured
        runner = PN.GraphStep(s_graph, m_graph, RingTensor(encode_fixed(xh, ring), 25, ring, _canonical=True))
        om = ON.Model(sizes, OR.RingParams(), seed=4)
        xo, _ = ON.synthetic_mnist(7, B, OR.RingParams())
        x1 = RingTensor(encode_fixed(xh, ring), 25, ring, _canonical=True)
        ok = True
        for step in range(3):
            s_eager.reseed(400 + step)
            l1, _, _ = PN.private_train_step(s_eager, m_eager, x1, labels)
            l2 = runner.step(400 + step, labels)
            l3, _, _ = ON.reference_train_step(om, xo, labels)
            ok &= l1 == l2 == l3
            for l in range(len(sizes) - 1):
                ok &= np.array_equal(m1 := m_eager.W[l].numpy(), m_graph.W[l].numpy())
                ok &= np.array_equal(m1, om.W(l))
        q.put(bool(ok))
    finally:
        dist.destroy_process_group()


def test_nccl_data_parallel_graph_capture_matches_eager_and_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_graph, args=(0, 29900 + os.getpid() % 500, q))
    p.start()
    ok = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0 and ok
