import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import bfv as OB, ring as OR, kernels as OK
from oracle.params import make_params
from paper_2403_11166_b200 import bfv, ring, _dev
from paper_2403_11166_b200.params import BfvParams
for N, L in ((2048, 8), (4096, 8), (8192, 7), (16384, 8)):
    op = make_params(N, L); ar = OB.Arith(op); pp = BfvParams(N=N, L=L)
    okp = OB.keygen(op, OR.SeededRng(11, 0), ar); pkp = bfv.keygen(pp, ring.SeededRng(11, 0))
    w = OR.SeededRng(9, 3).uniform_ring((1, N), OR.RingParams())
    opt = OB.encode_plain(op, w, ar)
    ppt = bfv.encode_plain(pp, _dev.u64_to_device(w))
    got = bfv.to_reference_order(pp, ppt.data)
    print(N, L, 'encode_plain eq', np.array_equal(got.reshape(opt.shape), opt))
    m = OR.SeededRng(9, 2).uniform_ring((1, N), OR.RingParams())
    ct = bfv.encrypt(pkp, _dev.u64_to_device(m), ring.SeededRng(10, 0))
    k = bfv.to_reference_order(pp, ct.data).reshape(1, 2, L, N)
    oprod = OB.he_plain_mul(k.copy(), opt, ar)
    pprod = bfv.he_plain_mul(ct, ppt)
    gp = bfv.to_reference_order(pp, pprod.data).reshape(oprod.shape)
    print(' he_plain_mul eq', np.array_equal(gp, oprod), 'odec ok', np.array_equal(OB.decrypt(op, okp, oprod, ar)[0], OK.negacyclic_mul_wrap(m[0].copy(), w[0].copy()) & np.uint64((1<<59)-1)), 'budget', OB.noise_budget(op, okp, oprod, ar))
