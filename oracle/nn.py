"""ORACLE — TEST INFRASTRUCTURE ONLY.

The SPEC-only ``nn`` module restated for the oracle:
models, the private training step composed from oracle/protocols.py, and
``reference_train_step`` -- the fixed-point Z_t pipeline without any
cryptography that SPEC:620-628 defines as THE oracle for training parity.

Step semantics (shared with paper_2403_11166_b200/nn.py):
  forward  Y_l = W_l X_{l-1} + b_l (2f); A_l = trunc_f(relu(Y_l)) (f) for l < last
  loss     DO reconstructs logits (2f), softmax-CE in float64, g = encode_f((p - y)/B)
           with the MO's share of g set to 0
  backward gb_l = rowsum(gY_l) (f); gW_l = arith_shift(gY_l A_{l-1}^T, f) (2f -> f)
           gA_{l-1} = trunc_f(W_l^T gY_l); gY_{l-1} = relu'(Y_{l-1}) * gA_{l-1}
  update   SGD momentum in float64 on master weights:
           v = mu v + g;  w = w - lr v;  W = encode_f(w), b = encode_2f(b)
"""

from __future__ import annotations

import numpy as np

from . import kernels as OK
from . import protocols as PR
from .ring import RingParams, SeededRng, decode_fixed, encode_fixed, to_signed


class Model:
    def __init__(self, sizes, ring: RingParams, seed: int = 0):
        self.sizes = list(sizes)
        self.ring = ring
        self.w, self.b, self.vw, self.vb = [], [], [], []
        for l, (ni, no) in enumerate(zip(sizes[:-1], sizes[1:])):
            g = SeededRng(seed, 500 + l)
            a = np.sqrt(1.0 / ni)
            self.w.append(g.uniform_real((no, ni), -a, a))
            self.b.append(g.uniform_real((no,), -a, a))
            self.vw.append(np.zeros((no, ni)))
            self.vb.append(np.zeros(no))

    @property
    def n_layers(self):
        return len(self.w)

    def W(self, l):
        return encode_fixed(self.w[l], self.ring)

    def Bias(self, l):
        return encode_fixed(self.b[l], self.ring, 2 * self.ring.f)

    def sgd(self, grads_w, grads_b, lr=1e-2, momentum=0.8):
        f = self.ring.f
        for l in range(self.n_layers):
            gw = decode_fixed(grads_w[l], self.ring, f)
            gb = decode_fixed(grads_b[l], self.ring, f)
            self.vw[l] = momentum * self.vw[l] + gw
            self.vb[l] = momentum * self.vb[l] + gb
            self.w[l] = self.w[l] - lr * self.vw[l]
            self.b[l] = self.b[l] - lr * self.vb[l]


def _m(v, ring):
    return np.asarray(v, dtype=np.uint64) & ring.mask


def _shift(v, bits, ring):
    return _m((to_signed(v, ring) >> np.int64(bits)).astype(np.uint64), ring)


def reference_train_step(model: Model, x_enc, labels, lr=1e-2, momentum=0.8):
    """the exact Z_t fixed-point pipeline, no cryptography."""
    ring, f = model.ring, model.ring.f
    acts, pre = [x_enc], []
    for l in range(model.n_layers):
        y = _m(OK.matmul_wrap(model.W(l), acts[-1]) + model.Bias(l)[:, None], ring)
        pre.append(y)
        if l < model.n_layers - 1:
            r = np.where(to_signed(y, ring) >= 0, y, np.uint64(0))
            acts.append(_shift(r, f, ring))
    loss, gy = PR.softmax_ce_grad(pre[-1], labels, ring)
    gws, gbs = [None] * model.n_layers, [None] * model.n_layers
    for l in reversed(range(model.n_layers)):
        gbs[l] = _m(gy.sum(axis=1, dtype=np.uint64), ring)
        gws[l] = _shift(_m(OK.matmul_wrap(gy, np.ascontiguousarray(acts[l].T)), ring), f, ring)
        if l > 0:
            ga = _shift(_m(OK.matmul_wrap(np.ascontiguousarray(model.W(l).T), gy), ring), f, ring)
            gy = np.where(to_signed(pre[l - 1], ring) >= 0, ga, np.uint64(0))
    model.sgd(gws, gbs, lr, momentum)
    return loss, gws, gbs


def private_train_step(ctx: PR.Ctx, model: Model, x_enc, labels, lr=1e-2, momentum=0.8, trace=None):
    """SPEC:629-637 with fullhe linear layers (oracle/protocols.py) and the
    dealer non-linear backend; <X_0>_0 = 0 at MO, <X_0>_1 = X at DO."""
    ring, f = model.ring, model.ring.f
    L = model.n_layers
    x_mo = np.zeros_like(x_enc)
    x_do = x_enc.copy()
    acts = [(x_mo, x_do)]
    ds = []
    ys = []
    for l in range(L):
        W = model.W(l)
        y_mo, y_do = PR.linear_forward(ctx, l, W, model.Bias(l), *acts[-1], mo_x_zero=(l == 0))
        ys.append((y_mo, y_do))
        if l < L - 1:
            z_mo, z_do, d = PR.dealer_op(ctx, l, PR.OP_RELU, y_mo, y_do)
            a_mo, a_do, _ = PR.dealer_op(ctx, l, PR.OP_TRUNC_F, z_mo, z_do, k=f)
            ds.append(d)
            acts.append((a_mo, a_do))
    logits = _m(ys[-1][0] + ys[-1][1], ring)  # MO sends its share; DO reconstructs
    loss, g = PR.softmax_ce_grad(logits, labels, ring)
    gy_mo, gy_do = np.zeros_like(g), g
    gws, gbs = [None] * L, [None] * L
    for l in reversed(range(L)):
        last = l == L - 1
        gbs[l] = PR.reveal_grad_bias(ctx, l, gy_mo, gy_do)
        gw2f = PR.grad_weight(ctx, l, *acts[l], gy_mo, gy_do, mo_x_zero=(l == 0), mo_gy_zero=last)
        gws[l] = _shift(gw2f, f, ring)  # MO: plaintext shift
        if trace is not None:
            trace.append((l, ys[l], gbs[l], gws[l]))
        if l > 0:
            ga_mo, ga_do = PR.linear_backward_input(ctx, l, model.W(l), gy_mo, gy_do, mo_gy_zero=last)
            t_mo, t_do, _ = PR.dealer_op(ctx, l, PR.OP_TRUNC_B, ga_mo, ga_do, k=f)
            gy_mo, gy_do, _ = PR.dealer_op(ctx, l - 1, PR.OP_RELU_B, t_mo, t_do, d=ds[l - 1])
    model.sgd(gws, gbs, lr, momentum)
    return loss, gws, gbs


def synthetic_mnist(seed: int, B: int, ring: RingParams):
    """MNIST-shaped synthetic batch: pixels U[0,1] standardised, labels U{0..9}."""
    g = SeededRng(seed, 900)
    x = g.uniform_real((784, B), 0.0, 1.0)
    x = (x - 0.1307) / 0.3081
    labels = g._gen.integers(0, 10, size=B)
    return encode_fixed(x, ring), labels
