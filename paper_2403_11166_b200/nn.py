"""Models and the private training step (the SPEC-only ``nn`` module,
SPEC.md:583-658) driving the B200 linear-layer engine.

``private_train_step`` follows SPEC:629-637: <X_0>_0 = 0 at MO and
<X_0>_1 = X at DO; every FC layer runs Alg.1 forward, Alg.2 weight
gradient, the bias reveal and (except the first layer) the input-gradient
protocol; ReLU and truncation use the dealer backend (nonlinear.py); the DO
computes the softmax-CE loss in float64 from the reconstructed logits
 and installs g = encode_f((p - y)/B) as its share of grad Y
with the MO's share 0; the MO keeps float64 master weights and momentum in
HBM and applies SGD + re-quantisation in one kernel (pb_sgd_momentum).

With sigma = 0 and faithful truncation the revealed gradients and the
updated weights are bit-identical to ``reference_train_step`` of the oracle
(SPEC:626, 635, 640).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .errors import EncodeRangeError, ShapeError
from .linear_protocols import Session, grad_weight, linear_backward_input, linear_forward, reveal_grad_bias
from .nonlinear import relu_backward, relu_forward, truncate
from .ring import DO, MO, RingParams, RingTensor, SeededRng, ShareTensor, arith_shift, encode_fixed

MODELS = {
    "mnist_mlp": [784, 128, 128, 10],  # SPEC:608, PAPER Fig. 5
}


class Model:
    """FC stack with MO-held float64 master weights on the device."""

    def __init__(self, sizes, ring: RingParams, seed: int = 0):
        self.sizes = list(sizes)
        self.ring = ring
        dev = _dev.device()
        self.w, self.b, self.vw, self.vb = [], [], [], []
        for l, (ni, no) in enumerate(zip(sizes[:-1], sizes[1:])):
            g = SeededRng(seed, 500 + l)  # SPEC:646 init, same draws as the oracle
            a = np.sqrt(1.0 / ni)
            self.w.append(torch.from_numpy(g.uniform_real((no, ni), -a, a)).to(dev))
            self.b.append(torch.from_numpy(g.uniform_real((no,), -a, a)).to(dev))
            self.vw.append(torch.zeros(no, ni, dtype=torch.float64, device=dev))
            self.vb.append(torch.zeros(no, dtype=torch.float64, device=dev))
        self.W = [RingTensor(encode_fixed(w, ring), ring.f, ring, _canonical=True) for w in self.w]
        self.B = [RingTensor(encode_fixed(b, ring, 2 * ring.f), 2 * ring.f, ring, _canonical=True) for b in self.b]
        self._flag = torch.zeros(1, dtype=torch.int32, device=dev)

    @property
    def n_layers(self):
        return len(self.w)

    def sgd(self, gws, gbs, lr=1e-2, momentum=0.8, check=True):
        ring = self.ring
        st = _dev.stream()
        for l in range(self.n_layers):
            for w, v, g, ring_t, scale in ((self.w[l], self.vw[l], gws[l], self.W[l], ring.f),
                                           (self.b[l], self.vb[l], gbs[l], self.B[l], 2 * ring.f)):
                _lib.call("pb_sgd_momentum", _dev.ptr(w), _dev.ptr(v), _dev.ptr(g.values), w.numel(), g.scale,
                          float(lr), float(momentum), ring.ell, scale, _dev.ptr(ring_t.values), _dev.ptr(self._flag),
                          st)
        if check and int(self._flag.item()):
            raise EncodeRangeError("weights left the fixed-point range")


def build_model(name, ring: RingParams, seed: int = 0) -> Model:
    if isinstance(name, str):
        if name not in MODELS:
            raise ShapeError(f"unknown model {name!r}")
        return Model(MODELS[name], ring, seed)
    return Model(name, ring, seed)


def softmax_ce_grad(logits_2f: np.ndarray, labels: np.ndarray, ring: RingParams):
    """DO-side loss in float64 on the reconstructed logits."""
    half = np.uint64(1 << (ring.ell - 1))
    v = np.asarray(logits_2f, dtype=np.uint64) & ring.mask
    sv = v.astype(np.int64) - ((v >= half).astype(np.int64) << np.int64(ring.ell))
    z = sv.astype(np.float64) / float(1 << (2 * ring.f))
    z = z - z.max(axis=0, keepdims=True)
    ez = np.exp(z)
    sm = ez / ez.sum(axis=0, keepdims=True)
    B = z.shape[1]
    onehot = np.zeros_like(sm)
    onehot[labels, np.arange(B)] = 1.0
    loss = float(-np.mean(np.log(sm[labels, np.arange(B)])))
    g = (sm - onehot) / B
    return loss, np.floor(g * float(1 << ring.f)).astype(np.int64).astype(np.uint64) & ring.mask


def forward_phase(sess: Session, model: Model, x: RingTensor):
    """Private forward pass; returns (state for the backward pass, logits = MO share + DO share)."""
    ring, f = model.ring, model.ring.f
    L = model.n_layers
    acts = [(ShareTensor(MO, RingTensor(torch.zeros_like(x.values), f, ring, _canonical=True)), ShareTensor(DO, x))]
    ds, ys = [], []
    for l in range(L):
        y = linear_forward(sess, l, model.W[l], model.B[l], *acts[-1], mo_x_zero=(l == 0))
        ys.append(y)
        if l < L - 1:
            z_mo, z_do, d = relu_forward(sess, l, *y)
            acts.append(truncate(sess, l, z_mo, z_do, f))
            ds.append(d)
    # the MO sends its share of the logits; the DO reconstructs them
    y_mo, y_do = ys[-1]
    logits = y_mo.value + y_do.value
    return (acts, ds, ys), logits


def backward_phase(sess: Session, model: Model, state, g_do: torch.Tensor, lr=1e-2, momentum=0.8, trace=None,
                   check=True):
    """Private backward pass from the DO's loss gradient share (MO share 0) + SGD at the MO."""
    ring, f = model.ring, model.ring.f
    L = model.n_layers
    acts, ds, ys = state
    gy_do = ShareTensor(DO, RingTensor(g_do, f, ring, _canonical=True))
    gy_mo = ShareTensor(MO, RingTensor(torch.zeros_like(g_do), f, ring, _canonical=True))
    gws, gbs = [None] * L, [None] * L
    for l in reversed(range(L)):
        last = l == L - 1
        gbs[l] = reveal_grad_bias(sess, l, gy_mo, gy_do)
        gws[l] = arith_shift(grad_weight(sess, l, *acts[l], gy_mo, gy_do, mo_x_zero=(l == 0), mo_gy_zero=last), f)
        if trace is not None:
            trace.append((l, ys[l], gbs[l], gws[l]))
        if l > 0:
            ga = linear_backward_input(sess, l, model.W[l], gy_mo, gy_do, mo_gy_zero=last)
            t_mo, t_do = truncate(sess, l, *ga, f, backward=True)
            gy_mo, gy_do = relu_backward(sess, l - 1, ds[l - 1], t_mo, t_do)
    model.sgd(gws, gbs, lr, momentum, check=check)
    return gws, gbs


def private_train_step(sess: Session, model: Model, x: RingTensor, labels, lr=1e-2, momentum=0.8,
                       trace=None, check=True):
    """One private step; x (784, B) at scale f, held by the DO."""
    state, logits = forward_phase(sess, model, x)
    loss, g = softmax_ce_grad(logits.numpy(), np.asarray(labels), model.ring)  # DO, float64 (host)
    gws, gbs = backward_phase(sess, model, state, _dev.u64_to_device(g), lr, momentum, trace, check)
    return loss, gws, gbs


class GraphStep:
    """A private training step replayed from two CUDA graphs (forward up to
    the logits, backward + SGD from the DO's loss gradient), with the DO's
    float64 softmax-CE on the host in between.  All randomness is re-keyed
    per step through the device seed word (Session.enable_graph_mode), and
    every kernel of the step is the same sm_100a kernel the eager path runs:
    the graphs only remove per-launch host overhead."""

    def __init__(self, sess: Session, model: Model, x: RingTensor, lr=1e-2, momentum=0.8):
        self.sess, self.model, self.lr, self.momentum = sess, model, lr, momentum
        sess.enable_graph_mode()
        self.x = x  # device input buffer; callers copy new batches into x.values
        n_cls, B = model.sizes[-1], x.shape[1]
        self.g_do = torch.zeros(n_cls, B, dtype=torch.int64, device=x.values.device)
        self.logits_host = torch.empty(n_cls, B, dtype=torch.int64).pin_memory()
        self.g_host = torch.empty(n_cls, B, dtype=torch.int64).pin_memory()
        # warm-up (eager, graph-mode keys): builds plans/maps, sizes scratch buffers
        st, lg = forward_phase(sess, model, x)
        backward_phase(sess, model, st, self.g_do, lr, momentum, check=False)
        torch.cuda.synchronize()
        self.g_fwd = torch.cuda.CUDAGraph()
        self.g_bwd = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g_fwd):
            self.state, self.logits = forward_phase(sess, model, x)
        with torch.cuda.graph(self.g_bwd, pool=self.g_fwd.pool()):
            self.grads = backward_phase(sess, model, self.state, self.g_do, lr, momentum, check=False)
        torch.cuda.synchronize()

    def step(self, seed: int, labels):
        self.sess.reseed(seed)
        self.g_fwd.replay()
        self.logits_host.copy_(self.logits.values, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        loss, g = softmax_ce_grad(self.logits_host.numpy().view(np.uint64), np.asarray(labels), self.model.ring)
        self.g_host.numpy().view(np.uint64)[...] = g
        self.g_do.copy_(self.g_host, non_blocking=True)
        self.g_bwd.replay()
        return loss


def synthetic_mnist(seed: int, B: int, ring: RingParams):
    """Same synthetic batch as the oracle: U[0,1] pixels standardised, labels U{0..9}.
    Returns host float64 features (784, B) and labels."""
    g = SeededRng(seed, 900)
    x = g.uniform_real((784, B), 0.0, 1.0)
    x = (x - 0.1307) / 0.3081
    labels = g._host_draw(lambda gen: gen.integers(0, 10, size=B))
    return x, labels
