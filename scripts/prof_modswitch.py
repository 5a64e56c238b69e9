import torch, sys
sys.path.insert(0, '.')
from paper_2403_11166_b200 import bfv, ring
from paper_2403_11166_b200.params import BfvParams
pp = BfvParams(N=8192, L=7)
kp = bfv.keygen(pp, ring.SeededRng(1, 0))
ct = bfv.encrypt(kp, torch.zeros(1024, 8192, dtype=torch.int64, device="cuda"), ring.SeededRng(2, 0), mode="sk")
for _ in range(3):
    bfv.mod_switch_drop(ct)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
bfv.mod_switch_drop(ct)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
