"""Generate the golden vectors that pin the CPU oracle to the reference.

Run in the build container, where the reference package is importable:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

It imports the UNMODIFIED reference (``pencil._kernels`` = K, ``pencil.ring`` = R)
and records its outputs on seeded inputs into tests/golden/kernels.npz and
tests/golden/ring.npz.  tests/test_oracle_golden.py then checks that the
oracle restatement (oracle/kernels.c, oracle/ring.py) reproduces every vector
bit-for-bit.  The GPU box never reads /root/reference: only these committed
fixtures travel.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from pencil import _kernels as K  # noqa: E402  (the reference)
from pencil import ring as R  # noqa: E402

from oracle.params import make_params  # noqa: E402


def kernels_vectors() -> dict:
    out = {}
    rng = np.random.default_rng(20240318)
    # --- NTT forward / inverse on real tables, several (N, L) ---
    for N, L in ((16, 2), (256, 3), (2048, 2), (8192, 1)):
        p = make_params(N, L)
        tb = p.tables
        P = 2
        rows = np.concatenate([rng.integers(0, q, size=(P, N), dtype=np.uint64) for q in p.moduli]).reshape(L, P, N)
        rows = np.ascontiguousarray(rows.transpose(1, 0, 2).reshape(P * L, N))
        q = np.tile(tb["q"], P)
        psi = np.ascontiguousarray(np.tile(tb["psi_brv"], (P, 1)))
        ipsi = np.ascontiguousarray(np.tile(tb["ipsi_brv"], (P, 1)))
        ninv = np.tile(tb["n_inv"], P)
        fwd = rows.copy()
        K.ntt_forward(fwd, psi, q)
        inv = rows.copy()
        K.ntt_inverse(inv, ipsi, ninv, q)
        out[f"ntt_{N}_{L}_in"] = rows
        out[f"ntt_{N}_{L}_fwd"] = fwd
        out[f"ntt_{N}_{L}_inv"] = inv
        # pointwise ops on the same rows
        b = np.ascontiguousarray(np.roll(rows, 1, axis=1))
        for name, fn in (("mul", K.pw_mul), ("mac", K.pw_mul_acc), ("add", K.pw_add), ("sub", K.pw_sub)):
            o = fwd.copy()
            fn(o, rows, b, q)
            out[f"pw_{name}_{N}_{L}"] = o
    # --- SPEC:127-129 NTT examples (N=4, q=17) ---
    q17 = np.array([17], dtype=np.uint64)
    psi = 9  # smallest generator-derived primitive 8th root of unity mod 17
    brv4 = [0, 2, 1, 3]
    psi_brv = np.array([[pow(psi, e, 17) for e in brv4]], dtype=np.uint64)
    ipsi_brv = np.array([[pow(psi, -e, 17) for e in brv4]], dtype=np.uint64)
    ninv = np.array([pow(4, -1, 17)], dtype=np.uint64)

    def spec_mul(a, b):
        x = np.array([a], dtype=np.uint64)
        y = np.array([b], dtype=np.uint64)
        K.ntt_forward(x, psi_brv, q17)
        K.ntt_forward(y, psi_brv, q17)
        z = np.empty_like(x)
        K.pw_mul(z, x, y, q17)
        K.ntt_inverse(z, ipsi_brv, ninv, q17)
        return z[0]

    out["spec_ntt_1px_sq"] = spec_mul([1, 1, 0, 0], [1, 1, 0, 0])
    out["spec_ntt_x3_x"] = spec_mul([0, 0, 0, 1], [0, 1, 0, 0])
    # --- decode (Garner + scale-round) on random residues ---
    for N, L in ((256, 3), (1024, 7)):
        p = make_params(N, L)
        tb = p.tables
        rows = np.stack([rng.integers(0, q, size=N, dtype=np.uint64) for q in p.moduli])
        d = K.garner_digits(rows, tb["q"], tb["prefix_inv"])
        m = K.scale_round_digits(d, tb["int_part"], tb["frac_part"], np.uint64(p.t - 1))
        out[f"dec_{N}_{L}_in"] = rows
        out[f"dec_{N}_{L}_digits"] = d
        out[f"dec_{N}_{L}_m"] = m
    # --- negacyclic oracles ---
    a = rng.integers(0, 1 << 63, size=64, dtype=np.uint64)
    b = rng.integers(0, 1 << 63, size=64, dtype=np.uint64)
    out["negwrap_a"], out["negwrap_b"] = a, b
    out["negwrap"] = K.negacyclic_mul_wrap(a, b)
    qm = 1073692673
    am, bm = a % np.uint64(qm), b % np.uint64(qm)
    out["negmod"] = K.negacyclic_mul_mod(am, bm, np.uint64(qm))
    # --- ring GEMM / conv / im2col / col2im ---
    A = rng.integers(0, 1 << 63, size=(7, 13), dtype=np.uint64)
    Bm = rng.integers(0, 1 << 63, size=(13, 5), dtype=np.uint64)
    out["mm_a"], out["mm_b"], out["mm"] = A, Bm, K.matmul_wrap(A, Bm)
    X = rng.integers(0, 1 << 63, size=(2, 3, 7, 6), dtype=np.uint64)
    Wc = rng.integers(0, 1 << 63, size=(4, 3, 3, 3), dtype=np.uint64)
    out["conv_x"], out["conv_w"], out["conv"] = X, Wc, K.conv2d_wrap(X, Wc)
    out["im2col_s3_st2"] = K.im2col_wrap(X, 3, 2)
    cols = K.im2col_wrap(X, 3, 1)
    out["col2im_s3_st1"] = K.col2im_wrap(cols, 2, 3, 7, 6, 3, 1)
    return out


def ring_vectors() -> dict:
    out = {}
    P = R.RingParams()
    xs = np.array([1.0, 0.5, -1.0, -0.25, 3.14159, -2.71828, 1e-8, -1e-8, 255.99, -255.99])
    out["enc_x"] = xs
    out["enc_f25"] = R.encode_fixed(xs, P)
    out["enc_f50"] = R.encode_fixed(xs[:6] / 1024, P, 50)
    out["dec_f25"] = R.decode_fixed(out["enc_f25"], P)
    out["signed"] = R.to_signed(out["enc_f25"], P)
    g = R.SeededRng(2024, 7)
    out["rng_uniform_ring_5"] = g.uniform_ring((5,), P)
    out["rng_uniform_ring_3x3"] = g.uniform_ring((3, 3), P)
    out["rng_ternary"] = g.ternary((33,))
    out["rng_uniform_mod"] = g.uniform_mod((17,), 1073692673)
    out["rng_uniform_ring_after"] = g.uniform_ring((6,), P)
    g2 = R.SeededRng(1, 0)
    out["rng_cbd"] = g2.cbd((64,))
    x = R.encode_tensor(np.linspace(-3, 3, 24).reshape(4, 6), P)
    mo, do = R.share_tensor(x, R.SeededRng(99, 3))
    out["share_x"], out["share_mo"], out["share_do"] = x.values, mo.value.values, do.value.values
    out["share_rec"] = R.reconstruct_tensor(mo, do).values
    y = R.RingTensor(R.encode_fixed(np.linspace(-5, 5, 11), P, 50), 50, P)
    out["shift_in"], out["shift_out"] = y.values, R.arith_shift(y, 25).values
    # R:140-145 __neg__ / scalar_mul and R:185-198 on edge residues (round 2)
    edge = np.array([0, 1, (1 << 58) - 1, 1 << 58, (1 << 58) + 1, (1 << 59) - 1, 12345, 1 << 40], dtype=np.uint64)
    e = R.RingTensor(edge, 25, P)
    out["edge_in"], out["edge_neg"] = edge, (-e).values
    out["edge_smul_ks"] = np.array([3, -7, (1 << 59) - 1, 1 << 40], dtype=np.int64)
    out["edge_smul"] = np.stack([e.scalar_mul(int(k)).values for k in out["edge_smul_ks"]])
    out["edge_signed"] = R.to_signed(edge, P)
    out["edge_dec_f50"] = R.decode_fixed(edge, P, 50)
    # R:80-81 normal: the DP hook's sampler
    out["rng_normal"] = R.SeededRng(2024, 1000003).normal((16,), 0.5)
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kernels_vectors())
    np.savez_compressed(os.path.join(HERE, "ring.npz"), **ring_vectors())
    print("wrote", os.path.join(HERE, "kernels.npz"), os.path.join(HERE, "ring.npz"))


if __name__ == "__main__":
    main()
