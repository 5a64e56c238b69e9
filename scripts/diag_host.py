import os, sys, time, json
sys.path.insert(0, '/root/repo')
import torch, numpy as np
from paper_2403_11166_b200 import bfv, nn as PN
from paper_2403_11166_b200.linear_protocols import Session
from paper_2403_11166_b200.params import BfvParams
from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed
ring, params = RingParams(), BfvParams()
sess = Session(params, ring, bfv.keygen(params, SeededRng(1, 0)), seed=1)
model = PN.Model("mnist_mlp", ring, seed=1)
xh, labels = PN.synthetic_mnist(1, 64, ring)
x = RingTensor(encode_fixed(xh, ring), ring.f, ring, _canonical=True)
r = PN.GraphStep(sess, model, x, prefetch_input=True)
for i in range(5): r.step(100+i, labels)
torch.cuda.synchronize()
# instrumented copy of step
import paper_2403_11166_b200.nn as N
T = []
def t(label): T.append((label, time.perf_counter()))
for it in range(20):
    T.clear()
    self = r
    t('begin')
    self.sess.reseed(900+it)
    main = torch.cuda.current_stream()
    main.wait_event(self._ev_ready); self.x.values.copy_(self._x_next)
    t('pre-fwd')
    self.g_fwd.replay(); t('fwd launched')
    self._ev_fwd.record(main)
    self._pre_stream.wait_stream(main)
    with torch.cuda.stream(self._pre_stream): self.g_pre.replay(); self._ev_pre.record()
    t('pre launched')
    self.logits_host.copy_(self.logits.values, non_blocking=True)
    self._ev_logits.record(main)
    while not self._ev_logits.query(): pass
    t('logits ready')
    loss, _ = self._loss(labels); t('loss')
    from paper_2403_11166_b200 import _lib
    _lib.load().pb_copy_async(self._g_dev_ptr, self._g_host_ptr, self._g_bytes, main.cuda_stream)
    main.wait_event(self._ev_pre)
    self.g_bwd.replay(); t('bwd launched')
    self._copy_stream.wait_event(self._ev_fwd); self._schedule_encrypt(); t('enc sched')
    torch.cuda.synchronize(); t('end')
    if it == 19:
        base = T[0][1]
        print([(l, round((v-base)*1e6,1)) for l, v in T])
