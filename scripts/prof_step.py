"""One private MLP training step (the bench workload) for ncu: warm-up steps
run unprofiled, then exactly one eager step runs between cudaProfilerStart/Stop
(use ncu --profile-from-start off)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_11166_b200 import bfv  # noqa: E402
from paper_2403_11166_b200 import nn as PN  # noqa: E402
from paper_2403_11166_b200.linear_protocols import Session  # noqa: E402
from paper_2403_11166_b200.params import BfvParams  # noqa: E402
from paper_2403_11166_b200.ring import RingParams, RingTensor, SeededRng, encode_fixed  # noqa: E402

ring, params = RingParams(), BfvParams()
kp = bfv.keygen(params, SeededRng(2024, 0))
sess = Session(params, ring, kp, seed=2024)
model = PN.Model([784, 128, 128, 10], ring, seed=2024)
xh, labels = PN.synthetic_mnist(2024, 64, ring)
x = RingTensor(encode_fixed(xh, ring), 25, ring, _canonical=True)
for i in range(3):
    sess.reseed(10 + i)
    PN.private_train_step(sess, model, x, labels, check=False)
torch.cuda.synchronize()
torch.cuda.profiler.start()
sess.reseed(99)
PN.private_train_step(sess, model, x, labels, check=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
