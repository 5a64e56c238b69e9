"""Print the worst useful-slot noise budget of the guard cases (tests/test_gpu_noise.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gpu_noise import _min_budget, _shares  # noqa: E402

from paper_2403_11166_b200 import bfv, ring  # noqa: E402
from paper_2403_11166_b200 import linear_protocols as LP  # noqa: E402
from paper_2403_11166_b200 import preprocessing as PP  # noqa: E402
from paper_2403_11166_b200.params import BfvParams  # noqa: E402

pp = BfvParams()
s = LP.Session(pp, ring.RingParams(), bfv.keygen(pp, ring.SeededRng(5, 0)), seed=3)
s.capture = []
LP.grad_weight(s, 0, *_shares(s, (784, 64), 1), *_shares(s, (128, 64), 2))
print("FC 784x128 weight gradient (dense share x share):", _min_budget(s, s.capture, 4), "bits")
s.capture = []
LP.conv_grad_weight(s, 0, *_shares(s, (64, 3, 32, 32), 3), *_shares(s, (64, 64, 32, 32), 4), 5, 2, 1)
print("CIFAR conv1 weight gradient (65536-term accumulation):", _min_budget(s, s.capture, 4), "bits")
s.capture = []
PP.prep_operator(s, 0, PP.Operator(("fc", 784, 128), PP.GRADW, 64), 1, bank_seed=2)
print("Pencil+ bank, FC gradW operator:", _min_budget(s, s.capture, 4), "bits")
