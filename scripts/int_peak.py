"""Measure the B200 integer-pipe peaks (ops/s, whole GPU) with scripts/int_peak.cu."""
import ctypes
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libint_peak.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", os.path.join(HERE, "int_peak.cu"), "-o", so])
lib = ctypes.CDLL(so)
lib.int_peak.restype = ctypes.c_float
blocks, iters = 148 * 8, 2000
ops_per_launch = blocks * 256 * iters * 16 * 8
res = {}
for op, name in enumerate(("IMAD", "IMAD.HI", "IMAD.WIDE.U32", "IADD3")):
    ms = lib.int_peak(op, blocks, iters)
    res[name] = {"ms": round(ms, 3), "ops_per_s": ops_per_launch / (ms / 1e3),
                 "per_sm_per_clk_at_1965MHz": ops_per_launch / (ms / 1e3) / 148 / 1.965e9}
print(json.dumps(res))
