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
from .errors import EncodeRangeError, ParamsError, ShapeError
from .linear_protocols import (OP_BWD_X, OP_FWD, OP_GRAD_B, OP_GRAD_W, Session, conv_backward_input, conv_forward,
                               conv_grad_weight, dp_noise, grad_w_flipped, grad_w_geometry, grad_weight, linear_backward_input,
                               linear_forward, reveal_grad_bias, reveal_grad_bias_conv)
from . import preprocessing as PP
from .nonlinear import (avgpool_backward, avgpool_forward, relu_backward, relu_forward, relu_truncate, truncate,
                        truncate_relu_backward)
from .poly_encoding import MatmulGeometry, conv_out_hw, plan_conv_layer, plan_matmul
from .ring import DO, MO, RingParams, RingTensor, SeededRng, ShareTensor, arith_shift, encode_fixed

MODELS = {
    # PAPER Fig. 5 / SPEC:608
    "mnist_mlp": ((784,), [("fc", 784, 128), ("fc", 128, 128), ("fc", 128, 10)]),
    # PAPER Fig. 6 / SPEC:609: Conv 1->5 5x5 s2 p2, FC 980->100, FC 100->10
    "mnist_cnn": ((1, 28, 28), [("conv", 1, 5, 5, 2, 2), ("flatten",), ("fc", 980, 100), ("fc", 100, 10)]),
    # BASELINE configs[2] "2 x conv5x5 + FC": the paper's CNN plus a second conv
    "mnist_cnn2": ((1, 28, 28), [("conv", 1, 5, 5, 2, 2), ("conv", 5, 5, 5, 2, 1), ("flatten",),
                                 ("fc", 980, 100), ("fc", 100, 10)]),
    # PAPER Fig. 7: the private-conv CIFAR-10 CNN (BASELINE configs[3])
    "cifar_cnn": ((3, 32, 32), [("conv", 3, 64, 5, 2, 1), ("pool",), ("conv", 64, 64, 5, 2, 1), ("pool",),
                                ("conv", 64, 64, 3, 1, 1), ("conv", 64, 64, 1, 0, 1), ("conv", 64, 16, 1, 0, 1),
                                ("flatten",), ("fc", 1024, 10)]),
}


def mlp_spec(sizes):
    return (sizes[0],), [("fc", a, b) for a, b in zip(sizes[:-1], sizes[1:])]


def shapes(in_shape, layers):
    """Per-entry (input shape, output shape) of one sample; raises ShapeError
    when adjacent layers do not compose."""
    cur = tuple(in_shape)
    out = []
    for e in layers:
        if e[0] == "fc":
            if cur != (e[1],):
                raise ShapeError(f"fc expects ({e[1]},), got {cur}")
            nxt = (e[2],)
        elif e[0] == "conv":
            _, ci, co, s, p, st = e
            if len(cur) != 3 or cur[0] != ci:
                raise ShapeError(f"conv expects {ci} channels, got {cur}")
            nxt = (co, *conv_out_hw(cur[1], cur[2], s, p, st))
        elif e[0] == "pool":
            if len(cur) != 3 or cur[1] % 2 or cur[2] % 2:
                raise ShapeError("avgpool2 needs even spatial dims")
            nxt = (cur[0], cur[1] // 2, cur[2] // 2)
        elif e[0] == "flatten":
            nxt = (int(np.prod(cur)),)
        else:
            raise ShapeError(f"unknown layer {e!r}")
        out.append((cur, nxt))
        cur = nxt
    return out


class Model:
    """Layer graph with MO-held float64 master weights on the device.

    ``Model(sizes)`` builds the FC stack (MLP); ``Model(name)`` one of MODELS;
    ``Model((in_shape, layers))`` any graph of ("fc", n_i, n_o),
    ("conv", c_i, c_o, s, pad, stride), ("pool",), ("flatten",).  Every linear
    layer except the last is followed by ReLU + truncation by f."""

    def __init__(self, arch, ring: RingParams, seed: int = 0):
        if isinstance(arch, str):
            if arch not in MODELS:
                raise ShapeError(f"unknown model {arch!r}")
            arch = MODELS[arch]
        if isinstance(arch, (list, tuple)) and all(isinstance(v, (int, np.integer)) for v in arch):
            arch = mlp_spec(list(arch))
        self.in_shape, self.layers = tuple(arch[0]), list(arch[1])
        self.io = shapes(self.in_shape, self.layers)
        self.lin = [i for i, e in enumerate(self.layers) if e[0] in ("fc", "conv")]
        self.ring = ring
        dev = _dev.device()
        self.w, self.b, self.vw, self.vb = [], [], [], []
        for l, i in enumerate(self.lin):
            e = self.layers[i]
            if e[0] == "fc":
                wshape, fan_in, nb = (e[2], e[1]), e[1], e[2]
            else:
                wshape, fan_in, nb = (e[2], e[1], e[3], e[3]), e[1] * e[3] * e[3], e[2]
            g = SeededRng(seed, 500 + l)  # SPEC:646 init, same draws as the oracle
            a = np.sqrt(1.0 / fan_in)
            self.w.append(torch.from_numpy(g.uniform_real(wshape, -a, a)).to(dev))
            self.b.append(torch.from_numpy(g.uniform_real((nb,), -a, a)).to(dev))
            self.vw.append(torch.zeros(wshape, dtype=torch.float64, device=dev))
            self.vb.append(torch.zeros(nb, dtype=torch.float64, device=dev))
        self.W = [RingTensor(encode_fixed(w, ring), ring.f, ring, _canonical=True) for w in self.w]
        self.B = [RingTensor(encode_fixed(b, ring, 2 * ring.f), 2 * ring.f, ring, _canonical=True) for b in self.b]
        self._flag = torch.zeros(1, dtype=torch.int32, device=dev)
        # step-abort word (GraphStep's loss handoff): nonzero -> the SGD kernels are no-ops
        self.skip = torch.zeros(1, dtype=torch.int32, device=dev)
        self.dp_group, self.dp_world = None, 1
        self._zeros = {}

    def zero_share(self, like: torch.Tensor) -> torch.Tensor:
        """A cached all-zero ring tensor shaped like ``like``: the MO's
        structurally zero shares (the network input, the loss gradient).  Read
        only -- every protocol writes fresh outputs -- so one buffer serves all
        steps, and a graph captured after it exists carries no fill kernel on
        its critical path."""
        key = (tuple(like.shape), like.dtype, like.device)
        z = self._zeros.get(key)
        if z is None:
            z = self._zeros[key] = torch.zeros_like(like)
        return z

    def set_data_parallel(self, group, world: int):
        """Data-parallel private training over ``world`` ranks of ``group``
        (one process per GPU, each with its own batch and session): the DO's
        loss gradient is divided by the global batch and the MO's revealed
        gradients are summed over ranks (one all-reduce per tensor, exact mod
        2^ell since 2^ell | 2^64) before SGD -- the same update as
        reference_train_step on the concatenated batch."""
        self.dp_group, self.dp_world = group, int(world)

    def grad_denom(self, B: int) -> int:
        return B * self.dp_world if self.dp_group is not None else 0

    def reduce_grads(self, *grads):
        """Sum revealed gradients over the data-parallel ranks (current stream)."""
        if self.dp_group is None:
            return
        import torch.distributed as dist

        m = int(self.ring.mask)
        for g in grads:
            dist.all_reduce(g.values, op=dist.ReduceOp.SUM, group=self.dp_group)
            g.values.bitwise_and_(m)

    @property
    def sizes(self):  # MLP compatibility
        return [self.layers[self.lin[0]][1]] + [self.layers[i][2] for i in self.lin]

    @property
    def n_layers(self):
        return len(self.lin)

    @property
    def n_classes(self):
        return self.io[-1][1][0]

    def segments(self):
        """For each linear l: the (pool / flatten) entries up to linear l+1."""
        seg = []
        for l, i in enumerate(self.lin):
            j = self.lin[l + 1] if l + 1 < self.n_layers else len(self.layers)
            seg.append(list(range(i + 1, j)))
        return seg

    def sgd(self, gws, gbs, lr=1e-2, momentum=0.8, check=True):
        for l in range(self.n_layers):
            self.sgd_layer(l, gws[l], gbs[l], lr, momentum)
        if check:
            self.check_range()

    def sgd_layer(self, l: int, gw: RingTensor | None, gb: RingTensor | None, lr=1e-2, momentum=0.8):
        """SGD with momentum for layer l's W and / or b (None: skipped) on the
        current stream (no host sync)."""
        ring = self.ring
        st = _dev.stream()
        for w, v, g, ring_t, scale in ((self.w[l], self.vw[l], gw, self.W[l], ring.f),
                                       (self.b[l], self.vb[l], gb, self.B[l], 2 * ring.f)):
            if g is None:
                continue
            _lib.call("pb_sgd_momentum", _dev.ptr(w), _dev.ptr(v), _dev.ptr(g.values), w.numel(), g.scale,
                      float(lr), float(momentum), ring.ell, scale, _dev.ptr(ring_t.values), _dev.ptr(self._flag),
                      _dev.ptr(self.skip), st)

    def check_range(self):
        if int(self._flag.item()):
            raise EncodeRangeError("weights left the fixed-point range")


def build_model(name, ring: RingParams, seed: int = 0) -> Model:
    return Model(name, ring, seed)


class SoftmaxCE:
    """The DO's loss step for fixed (classes, batch): softmax
    cross-entropy in float64 on the reconstructed logits, bit-identical to
    oracle/protocols.py softmax_ce_grad.  numpy evaluates exp / log (so the
    values are numpy's), the library's host helpers (pb_host_softmax_*,
    pb_host_mean: numpy's pairwise mean) everything around them, on buffers
    whose addresses are resolved once -- ~15 small numpy ops (~50 us) become
    ~12 us on the step's critical path."""

    def __init__(self, ring: RingParams, C: int, B: int, logits=None, g_out=None, denom: int = 0):
        self.ring, self.C, self.B, self.denom = ring, C, B, int(denom)
        self.z = np.empty((C, B), dtype=np.float64)
        self.p = np.empty(B, dtype=np.float64)
        self.lab = np.empty(B, dtype=np.int64)
        self.g = np.empty((C, B), dtype=np.uint64) if g_out is None else g_out
        self.logits = logits
        lib = _lib.load()
        self._pre, self._post, self._mean = lib.pb_host_softmax_pre, lib.pb_host_softmax_post, lib.pb_host_mean
        addr = lambda a: a.__array_interface__["data"][0]  # noqa: E731
        self.az, self.ap, self.alab, self.ag = addr(self.z), addr(self.p), addr(self.lab), addr(self.g)
        self.alog = addr(logits) if logits is not None else None

    def __call__(self, labels, logits=None):
        """(loss, g) with g = encode_f((softmax - onehot) / D) mod 2^ell in self.g
        (D = denom: the global batch under data parallelism; else B)."""
        self.grad(labels, logits)
        return self.value(), self.g

    def grad(self, labels, logits=None):
        """The gradient half: g written into self.g (the backward can go)."""
        if logits is None:
            alog = self.alog
        else:
            logits = np.ascontiguousarray(logits, dtype=np.uint64)
            alog = logits.__array_interface__["data"][0]
        self.lab[...] = labels
        r = self.ring
        _lib.check(self._pre(alog, self.C, self.B, r.ell, 2 * r.f, self.az), "pb_host_softmax_pre")
        np.exp(self.z, out=self.z)
        _lib.check(self._post(self.az, self.C, self.B, self.alab, r.ell, r.f, self.denom, self.ap, self.ag),
                   "pb_host_softmax_post")
        return self.g

    def value(self):
        """The loss of the last grad() call (mean -log p of the labelled class)."""
        np.log(self.p, out=self.p)
        return -self._mean(self.ap, self.B)


_SMCE = {}


def softmax_ce_grad(logits_2f: np.ndarray, labels: np.ndarray, ring: RingParams, denom: int = 0):
    """DO-side loss in float64 on the reconstructed logits (SoftmaxCE);
    ``denom``: the gradient's batch divisor (0: this batch)."""
    C, B = np.shape(logits_2f)
    key = (C, B, ring.ell, ring.f, denom)
    sm = _SMCE.get(key)
    if sm is None:
        sm = _SMCE[key] = SoftmaxCE(ring, C, B, denom=denom)
    loss, g = sm(labels, logits_2f)
    return loss, g.copy()


def _flatten(sh: ShareTensor) -> ShareTensor:  # (B, C, H, W) -> (C*H*W, B), local data movement
    v = sh.value
    return ShareTensor(sh.owner_role, RingTensor(v.values.reshape(v.shape[0], -1).t().contiguous(), v.scale,
                                                 v.params, _canonical=True))


def _unflatten(sh: ShareTensor, chw) -> ShareTensor:  # (C*H*W, B) -> (B, C, H, W)
    v = sh.value
    return ShareTensor(sh.owner_role, RingTensor(v.values.t().contiguous().reshape(-1, *chw), v.scale, v.params,
                                                 _canonical=True))


def forward_phase(sess: Session, model: Model, x: RingTensor, prep=None):
    """Private forward pass; returns (state for the backward pass, logits = MO share + DO share).
    With ``prep`` (a preprocessing.PrepState) the linear layers run Alg. 4's
    HE-free online protocol (SPEC mode "prep")."""
    ring, f = model.ring, model.ring.f
    seg = model.segments()
    cur = (ShareTensor(MO, RingTensor(model.zero_share(x.values), f, ring, _canonical=True)), ShareTensor(DO, x))
    acts, ds, ys = [], [], []
    if prep is None:  # every layer's MO mask depends only on the seed: draw them all up front
        B = x.shape[1] if len(model.in_shape) == 1 else x.shape[0]
        sess.prefetch_masks(_mask_specs(model, B, (OP_FWD,)))
        sess.begin_phase()
    _forward_layers(sess, model, prep, cur, acts, ds, ys, seg)
    sess.join_side()
    # the MO sends its share of the logits; the DO reconstructs them
    y_mo, y_do = ys[-1]
    logits = y_mo.value + y_do.value
    return (acts, ds, ys), logits


def _forward_layers(sess, model, prep, cur, acts, ds, ys, seg):
    f, L = model.ring.f, model.n_layers
    for l, i in enumerate(model.lin):
        e = model.layers[i]
        acts.append(cur)
        if prep is not None:
            y = PP.prep_linear_forward(sess, l, prep.banks[l], model.W[l], model.B[l], *cur, mo_x_zero=(l == 0))
        elif e[0] == "fc":
            y = linear_forward(sess, l, model.W[l], model.B[l], *cur, mo_x_zero=(l == 0))
        else:
            y = conv_forward(sess, l, model.W[l], model.B[l], *cur, e[4], e[5], mo_x_zero=(l == 0))
        ys.append(y)
        if l < L - 1:
            *cur, d = relu_truncate(sess, l, *y, f)  # ReLU + truncation, one dealer round
            ds.append(d)
            for k in seg[l]:
                if model.layers[k][0] == "pool":
                    cur = avgpool_forward(sess, l, *cur)
                elif model.layers[k][0] == "flatten":
                    cur = (_flatten(cur[0]), _flatten(cur[1]))


def backward_phase(sess: Session, model: Model, state, g_do: torch.Tensor, lr=1e-2, momentum=0.8, trace=None,
                   check=True, prep=None, pre_layers=None, on_start=None, early_layers=None):
    """Private backward pass from the DO's loss gradient share (MO share 0) + SGD at the MO.
    ``pre_layers``: prepare these layers' forward-only operands here, on the
    prep stream beside the backward chain (the rest were prepared before).
    ``early_layers``: prepare these layers' operands here too, at full width
    and ahead of ``pre_layers``, ordered by per-operand events.
    ``on_start``: enqueued on this stream after those forks, before anything
    that reads ``g_do`` (GraphStep's host handoff)."""
    ring, f = model.ring, model.ring.f
    L = model.n_layers
    seg = model.segments()
    acts, ds, ys = state
    # the handoff (a one-CTA wait for the host's loss) is enqueued first so it
    # holds an SM before the preparation work below fills them; that work and
    # the encryption pre-draws fork from the point before it
    if prep is None:
        sess.begin_phase()  # the encryption pre-draws run beside the host handoff
    ev0 = torch.cuda.Event()
    ev0.record()
    if on_start is not None:
        on_start()
    if early_layers or pre_layers:
        side = sess.prep_stream()
        side.wait_event(ev0)
        with torch.cuda.stream(side):
            if early_layers:
                prepare_backward(sess, model, state, prep, layers=early_layers, clear=False)
            if pre_layers:
                prepare_backward(sess, model, state, prep, layers=pre_layers, clear=False, background=True)
    gy_do = ShareTensor(DO, RingTensor(g_do, f, ring, _canonical=True))
    gy_mo = ShareTensor(MO, RingTensor(model.zero_share(g_do), f, ring, _canonical=True))
    gws, gbs = [None] * L, [None] * L
    # The weight-gradient protocols (bias reveal + Alg.2) of layer l and the
    # input-gradient chain to layer l-1 are independent given grad Y_l: Alg.2
    # runs on the session's grad stream, overlapping the chain on this stream.
    main, gstream = torch.cuda.current_stream(), sess.grad_stream()
    keep = []  # grad Y shares read on the grad stream stay referenced until the join
    for l in reversed(range(L)):
        e = model.layers[model.lin[l]]
        last = l == L - 1
        ev_gy = torch.cuda.Event()
        ev_gy.record(main)  # grad Y_l is available: both chains fork here
        # the input-gradient protocol (the critical chain) is enqueued first, so its
        # kernels come first in the graph's launch order when both chains are ready
        if l > 0 and _BX_FIRST:
            ga = _backward_input(sess, model, l, e, acts, gy_mo, gy_do, last, prep)
        gstream.wait_event(ev_gy)
        with torch.cuda.stream(gstream):
            # the DO's DP perturbation (None unless sess.dp is enabled)
            wshape = (e[2], e[1]) if e[0] == "fc" else (e[2], e[1], e[3], e[3])
            eb = dp_noise(sess, l, OP_GRAD_B, (e[2],), f)
            ew = dp_noise(sess, l, OP_GRAD_W, wshape, 2 * f)
            gbs[l] = (reveal_grad_bias if e[0] == "fc" else reveal_grad_bias_conv)(sess, l, gy_mo, gy_do, e=eb)
            model.reduce_grads(gbs[l])  # data parallel: sum over ranks before the update
            # b_l is not read again this step: its update goes now, beside the
            # weight-gradient protocol instead of behind it
            model.sgd_layer(l, None, gbs[l], lr, momentum)
            if prep is not None:
                gw = PP.prep_grad_weight(sess, l, prep.banks[l], *acts[l], gy_mo, gy_do, e=ew, mo_x_zero=(l == 0),
                                         mo_gy_zero=last)
            elif e[0] == "fc":
                gw = grad_weight(sess, l, *acts[l], gy_mo, gy_do, e=ew, mo_x_zero=(l == 0), mo_gy_zero=last)
            else:
                gw = conv_grad_weight(sess, l, *acts[l], gy_mo, gy_do, e[3], e[4], e[5], e=ew, mo_x_zero=(l == 0),
                                      mo_gy_zero=last)
            model.reduce_grads(gw)  # at 2f, before the shift
            gws[l] = arith_shift(gw, f)
        keep.append((gy_mo, gy_do))
        if trace is not None:
            trace.append((l, ys[l], gbs[l], gws[l]))
        if l > 0 and not _BX_FIRST:
            ga = _backward_input(sess, model, l, e, acts, gy_mo, gy_do, last, prep)
        # the MO's SGD for layer l as soon as both grad W_l (grad stream) and
        # the last use of W_l (this layer's input-gradient protocol) are enqueued
        gstream.wait_stream(main)
        with torch.cuda.stream(gstream):
            model.sgd_layer(l, gws[l], None, lr, momentum)
        if l > 0:
            if any(model.layers[k][0] == "pool" for k in seg[l - 1]):
                t_mo, t_do = truncate(sess, l, *ga, f, backward=True)
                for k in reversed(seg[l - 1]):
                    if model.layers[k][0] == "pool":
                        t_mo, t_do = avgpool_backward(sess, l - 1, t_mo, t_do)
                    elif model.layers[k][0] == "flatten":
                        chw = model.io[k][0]
                        t_mo, t_do = _unflatten(t_mo, chw), _unflatten(t_do, chw)
                gy_mo, gy_do = relu_backward(sess, l - 1, ds[l - 1], t_mo, t_do)
            else:  # truncation + ReLU' in one dealer round (a flatten in between is a pure permutation)
                t_mo, t_do = ga
                for k in reversed(seg[l - 1]):
                    chw = model.io[k][0]
                    t_mo, t_do = _unflatten(t_mo, chw), _unflatten(t_do, chw)
                gy_mo, gy_do = truncate_relu_backward(sess, l - 1, ds[l - 1], t_mo, t_do, f)
    main.wait_stream(gstream)
    if early_layers or pre_layers:
        main.wait_stream(sess.prep_stream())  # joins the prep fork (graph capture needs every fork joined)
    sess.join_side()
    del keep
    if check:
        model.check_range()
    sess.clear_prepared()
    return gws, gbs



def _mask_specs(model: Model, B: int, ops, layers=None):
    """(layer, op, shape) of the MO masks the protocols of ``ops`` draw (fullhe mode)."""
    out = []
    for l in range(model.n_layers) if layers is None else layers:
        k = model.lin[l]
        e = model.layers[k]
        (shp_in, shp_out), conv = model.io[k], e[0] == "conv"
        for op in ops:
            if op == OP_FWD:
                out.append((l, op, (B, *shp_out) if conv else (shp_out[0], B)))
            elif op == OP_BWD_X and l > 0:
                out.append((l, op, (B, *shp_in) if conv else (shp_in[0], B)))
            elif op == OP_GRAD_W:
                out.append((l, op, tuple(model.W[l].shape)))
    return out


def _backward_input(sess, model, l, e, acts, gy_mo, gy_do, last, prep):
    if prep is not None:
        return PP.prep_linear_backward_input(sess, l, prep.banks[l], model.W[l], gy_mo, gy_do, mo_gy_zero=last)
    if e[0] == "fc":
        return linear_backward_input(sess, l, model.W[l], gy_mo, gy_do, mo_gy_zero=last)
    H, Wd = acts[l][1].shape[2:]
    return conv_backward_input(sess, l, model.W[l], gy_mo, gy_do, H, Wd, e[4], e[5], mo_gy_zero=last)


def prepare_backward(sess: Session, model: Model, state, prep=None, layers=None, clear=True, events=True,
                     background=False):
    """Produce, ahead of the loss gradient, every backward-pass HE operand that
    depends only on the forward pass: the MO's encodings of W_l (input-gradient
    protocols) and of its activation shares, the DO's encryptions of its
    activation shares (weight-gradient cross terms).  Enqueued on the current
    stream; the backward protocols pick them up (Session.prepare_operand) and
    only the gradient-dependent operands remain on their critical path.  FC
    and conv layers of mode "fullhe"; Pencil+ (prep) prepares nothing.
    ``layers``: only these layers (default all)."""
    if clear:
        sess.clear_prepared()
    if prep is not None:
        return
    acts = state[0]
    L = model.n_layers
    N = sess.p.N
    x0 = acts[0][1].value if acts[0][1].owner_role == DO else acts[0][0].value
    B = x0.shape[1] if len(model.in_shape) == 1 else x0.shape[0]
    sess.prefetch_masks(_mask_specs(model, B, (OP_BWD_X, OP_GRAD_W), layers), events)
    pool, jobs = sess.fork_pool(), []

    def prepare(*args):  # independent preparations run concurrently, round-robin over the pool
        with torch.cuda.stream(pool[len(jobs) % len(pool)]):
            sess.prepare_operand(*args, events, background)
        jobs.append(args)

    for l in range(L) if layers is None else layers:
        e = model.layers[model.lin[l]]
        x_mo, x_do = acts[l]
        if x_mo.owner_role != MO:
            x_mo, x_do = x_do, x_mo
        if e[0] == "conv":
            B, c_i, H, Wd = x_do.shape
            c_o, s = model.W[l].shape[0], model.W[l].shape[2]
            pad, stride = e[4], e[5]
            if l > 0:  # conv_backward_input
                plan = plan_conv_layer("bwdx", B, c_i, c_o, H, Wd, s, pad, stride, N)
                prepare(l, OP_BWD_X, plan, "A_pt", model.W[l].values)
            plan = plan_conv_layer("gradw", B, c_i, c_o, H, Wd, s, pad, stride, N)  # conv_grad_weight
            if l < L - 1:
                prepare(l, OP_GRAD_W, plan, "A_ct", x_do.value.values)
            if l > 0:
                prepare(l, OP_GRAD_W, plan, "B_pt", x_mo.value.values)
            continue
        if e[0] != "fc":
            continue
        n_o, n_i = model.W[l].shape
        B = x_do.shape[1]
        if l > 0:  # linear_backward_input: W^T through strides (1, n_i)
            plan = plan_matmul(MatmulGeometry(n_o, n_i, B), N, None, (1, n_i), None)
            prepare(l, OP_BWD_X, plan, "A_pt", model.W[l].values)
        flip = grad_w_flipped(l == 0, l == L - 1)  # grad_weight's orientation and plan
        g, vs, ys = grad_w_geometry(n_o, n_i, B, flip)
        plan = plan_matmul(g, N, vs, None, ys)
        if l < L - 1:  # Enc(X_1) (x) gY_0: term B flipped, term A otherwise
            prepare(l, OP_GRAD_W, plan, "B_ct" if flip else "A_ct", x_do.value.values)
        if l > 0:  # Enc(gY_1) (x) X_0: X_0 is term A's plaintext flipped, term B's otherwise
            prepare(l, OP_GRAD_W, plan, "A_pt" if flip else "B_pt", x_mo.value.values)
    if not events:  # ordered by a stream join instead of events: join every fork now
        sess.join_side()


def private_train_step(sess: Session, model: Model, x: RingTensor, labels, lr=1e-2, momentum=0.8,
                       trace=None, check=True, prep=None):
    """One private step; x held by the DO at scale f: (784, B)
    feature-major for FC-first models, (B, C, H, W) for CNNs.  ``prep``
    selects SPEC's mode "prep" (Pencil+, Alg. 4) over "fullhe"."""
    state, logits = forward_phase(sess, model, x, prep)
    main, side = torch.cuda.current_stream(), sess.prep_stream()
    side.wait_stream(main)
    with torch.cuda.stream(side):  # overlaps the host's loss computation
        prepare_backward(sess, model, state, prep)
    loss, g = softmax_ce_grad(logits.numpy(), np.asarray(labels), model.ring, model.grad_denom(logits.shape[1]))
    main.wait_stream(side)
    gws, gbs = backward_phase(sess, model, state, _dev.u64_to_device(g), lr, momentum, trace, check, prep)
    return loss, gws, gbs


# Step-scheduling constants (round-1 A/B measurements):
_LATE_PREP = True    # prepare layer 0's backward operands inside the backward graph
_PREFETCH_BG = True  # prefetched input encryption grid-capped (background)
_BX_FIRST = True     # enqueue the input-gradient protocol before the grad-W chain
_PROLOGUE = True     # step seed + prefetched input copied by one prologue kernel
# The one run-time switch: PB_HANDOFF=0 replaces the device-side loss handoff
# (a kernel that waits for the host's release word) by an H2D copy + a second
# graph launch -- the mode to profile under ncu, which serialises kernels and
# would time the waiting kernel.
_HANDOFF = __import__("os").environ.get("PB_HANDOFF", "1") == "1"
_HANDOFF_TIMEOUT_NS = 30_000_000_000  # a backward waiting this long for the host's loss gives up (ack fails)


class GraphStep:
    """A private training step replayed from CUDA graphs (forward up to the
    logits; the backward operands prepared beside the host's loss; backward +
    SGD from the DO's loss gradient), with the DO's float64 softmax-CE on the
    host in between.  All randomness is re-keyed per step through the device
    seed word (Session.enable_graph_mode), and every kernel of the step is the
    same sm_100a kernel the eager path runs: the graphs only remove per-launch
    host overhead.

    ``prefetch_input=True`` also takes the DO's encryption of the first
    layer's input off the step: it is produced on a copy stream beside the
    previous step's backward -- right after ``load_batch`` stages a batch, or
    (input resident, no ``load_batch``) at the end of ``step`` -- from a
    DO-owned key stream (a per-encryption counter in its own device seed
    word), and the forward graph consumes it.  In that mode the input must be
    supplied through ``load_batch`` (direct writes to ``x.values`` are not
    seen by the prefetched encryption)."""

    def __init__(self, sess: Session, model: Model, x: RingTensor, lr=1e-2, momentum=0.8, prep=None,
                 prefetch_input: bool = False):
        self.sess, self.model, self.lr, self.momentum, self.prep = sess, model, lr, momentum, prep
        if sess.dp is not None and sess.dp.enabled:  # a per-step host draw cannot be captured
            raise ParamsError("GraphStep replays fixed launches: run DP (sigma > 0) steps with private_train_step")
        sess.enable_graph_mode()
        self.x = x  # device input buffer; callers copy new batches into x.values (or use load_batch)
        self._stage = None
        self._flag_pending = False
        self._batch_pending = False
        n_cls = model.n_classes
        B = x.shape[1] if len(model.in_shape) == 1 else x.shape[0]
        dev = x.values.device
        self.g_do = torch.zeros(n_cls, B, dtype=torch.int64, device=dev)
        self.logits_host = torch.empty(n_cls, B, dtype=torch.int64).pin_memory()
        # the forward graph publishes the logits into logits_host and then bumps
        # this pinned word (pb_host_publish); the host polls it
        self._pub_flag = torch.zeros(1, dtype=torch.int32).pin_memory()
        self._pub_np = self._pub_flag.numpy().view(np.uint32)
        self._pub_seq = torch.zeros(1, dtype=torch.int32, device=dev)
        self._pub_count = 0
        self.g_host = torch.empty(n_cls, B, dtype=torch.int64).pin_memory()
        self._loss = SoftmaxCE(model.ring, n_cls, B, denom=model.grad_denom(B), logits=self.logits_host.numpy().view(np.uint64),
                               g_out=self.g_host.numpy().view(np.uint64))
        first = model.layers[model.lin[0]]
        self.prefetch = bool(prefetch_input) and prep is None and first[0] in ("fc", "conv")
        # warm-up (eager, graph-mode keys): builds plans/maps, sizes scratch buffers
        st, lg = forward_phase(sess, model, x, prep)
        prepare_backward(sess, model, st, prep)
        backward_phase(sess, model, st, self.g_do, lr, momentum, check=False, prep=prep)
        torch.cuda.synchronize()
        self._copy_stream = torch.cuda.Stream()
        if self.prefetch:
            self._x_next = x.values.clone()  # the next step's input (ring encoded)
            self._enc_seed_host = torch.zeros(4, dtype=torch.int64).pin_memory()
            self._enc_seed_dev = torch.zeros(1, dtype=torch.int64, device=dev)
            self._enc_rng = SeededRng(0, 999_001).bind(self._enc_seed_dev.data_ptr())
            self._enc_count = 0
            self._enc_base = (int(sess.seed) * 0x9E3779B9 + 12345) & ((1 << 62) - 1)
            if first[0] == "fc":
                n_o, n_i = model.W[0].shape
                self._enc_plan = plan_matmul(MatmulGeometry(n_i, n_o, B), sess.p.N)
            else:
                _, c_i, H, Wd = x.shape
                c_o, s = model.W[0].shape[0], model.W[0].shape[2]
                self._enc_plan = plan_conv_layer("fwd", B, c_i, c_o, H, Wd, s, first[4], first[5], sess.p.N)
            self._prefetch_encrypt()  # eager once: allocates the persistent operand buffer
            torch.cuda.synchronize()
            sess.clear_prepared()
            self.g_enc = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.g_enc):
                self._prefetch_encrypt()  # leaves the prepared entry the forward capture consumes
        model.zero_share(x.values)  # the zero shares exist before capture: no fill kernels in the graphs
        model.zero_share(self.g_do)
        torch.cuda.synchronize()
        self.g_fwd = torch.cuda.CUDAGraph()
        self.g_pre = torch.cuda.CUDAGraph()
        self.g_bwd = torch.cuda.CUDAGraph()
        hp = None  # capture stream (a high-priority chain stream measured no gain, r01)
        # prologue: the replayed forward graph fetches the step seed from the pinned
        # host word and copies the prefetched input itself (no H2D copy and copy
        # kernel ahead of the launch)
        self.prologue = _PROLOGUE
        with torch.cuda.graph(self.g_fwd, stream=hp):
            if self.prologue:
                nbytes = x.values.numel() * 8 if self.prefetch else 0
                _lib.call("pb_step_prologue", sess._seed_host.data_ptr(), sess._seed_dev.data_ptr(),
                          self._x_next.data_ptr() if self.prefetch else None, x.values.data_ptr(), nbytes,
                          torch.cuda.current_stream().cuda_stream)
            self.state, self.logits = forward_phase(sess, model, x, prep)
            _lib.call("pb_host_publish", self.logits.values.data_ptr(), self.logits_host.data_ptr(),
                      self.logits_host.numel(), self._pub_seq.data_ptr(), self._pub_flag.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
        # the operands the backward consumes first (layers >= 1) are prepared beside
        # the host's loss step; layer 0's (consumed last) inside the backward graph,
        # beside its latency-bound first layers, so it does not wait for them
        L = model.n_layers
        late = [0] if L > 1 and _LATE_PREP else []
        early = [l for l in range(L) if l not in late]
        self.handoff = _HANDOFF
        if not self.handoff:
            with torch.cuda.graph(self.g_pre, pool=self.g_fwd.pool()):
                prepare_backward(sess, model, self.state, prep, layers=early,
                                 events=False)  # ordered by step(): the backward replay waits for this graph
        self._g_dev_ptr, self._g_host_ptr = self.g_do.data_ptr(), self.g_host.data_ptr()
        self._g_bytes = self.g_do.numel() * 8
        # handoff: the backward graph is launched right behind the forward; its
        # operand preparation (all layers) runs during the host's loss and its
        # chain starts with a kernel that waits for the host's release word,
        # then reads the gradient from pinned memory (no H2D copy and no graph
        # launch between the host loss and the backward)
        on_start = None
        if self.handoff:
            self._hflag = torch.zeros(3, dtype=torch.int32).pin_memory()  # [release, ack, abort]
            self._hflag_np = self._hflag.numpy().view(np.uint32)
            self._hseq_dev = torch.zeros(1, dtype=torch.int32, device=dev)
            self._hseq = 0
            n_g = self.g_do.numel()

            def on_start():
                _lib.call("pb_host_handoff", self._hflag.data_ptr(), self._hseq_dev.data_ptr(), self._g_host_ptr,
                          self._g_dev_ptr, n_g, _HANDOFF_TIMEOUT_NS, self.model.skip.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
        with torch.cuda.graph(self.g_bwd, pool=self.g_fwd.pool(), stream=hp):
            self.grads = backward_phase(sess, model, self.state, self.g_do, lr, momentum, check=False, prep=prep,
                                        pre_layers=late, on_start=on_start,
                                        early_layers=early if self.handoff else None)
        self._pre_stream = torch.cuda.Stream()
        self._ev_fwd = torch.cuda.Event()
        self._ev_ready = torch.cuda.Event()
        self._ev_pre = torch.cuda.Event()
        self._loaded_last = False
        torch.cuda.synchronize()
        sess.clear_prepared()
        if self.prefetch:
            self._schedule_encrypt()

    def _prefetch_encrypt(self):
        self.sess.prepare_operand(0, OP_FWD, self._enc_plan, "A_ct", self._x_next, event=False, rng=self._enc_rng,
                                  background=_PREFETCH_BG)

    def _schedule_encrypt(self):
        """On the copy stream: a fresh DO key word, then the prefetch graph."""
        slot = self._enc_count % 4
        self._enc_seed_host[slot] = self._enc_base + self._enc_count
        self._enc_count += 1
        with torch.cuda.stream(self._copy_stream):
            self._enc_seed_dev.copy_(self._enc_seed_host[slot:slot + 1], non_blocking=True)
            self.g_enc.replay()
            self._ev_ready.record()

    def load_batch(self, x_host: torch.Tensor):
        """Stage a new real-valued batch (host float64, pinned for an async
        copy; the DO's input, same shape as x) for the next step: the H2D copy
        runs on a copy stream, overlapping the previous step's backward still
        on the GPU (with ``prefetch_input`` so do the encode and the DO's
        encryption); otherwise the next step() encodes it into the graphs'
        input buffer.  No host sync -- the encode's range flag is checked at
        that step's logits sync."""
        if self._stage is None:
            dev = self.x.values.device
            self._stage = torch.empty(tuple(self.x.values.shape), dtype=torch.float64, device=dev)
            self._flag = torch.zeros(1, dtype=torch.int32, device=dev)
            self._flag_host = torch.zeros(1, dtype=torch.int32).pin_memory()
            self._flag_np = self._flag_host.numpy()  # read on the host's critical path: no torch indexing
            self._ev_loaded, self._ev_free = torch.cuda.Event(), None
        if self.prefetch:
            from .ring import encode_fixed_into

            # the previous forward has read x_next (copied into x) and the prepared ciphertext
            self._copy_stream.wait_event(self._ev_fwd)
            with torch.cuda.stream(self._copy_stream):
                self._stage.copy_(x_host, non_blocking=True)
                encode_fixed_into(self._stage, self.model.ring, self._x_next, self._flag)
                self._flag_host.copy_(self._flag, non_blocking=True)
            self._schedule_encrypt()
            self._flag_pending = True
            self._loaded_last = True
            return
        if self._ev_free is not None:  # the previous batch's encode has read the stage
            self._copy_stream.wait_event(self._ev_free)
        with torch.cuda.stream(self._copy_stream):
            self._stage.copy_(x_host, non_blocking=True)
            self._ev_loaded.record()
        self._batch_pending = True

    def _encode_batch(self, main):
        from .ring import encode_fixed_into

        main.wait_event(self._ev_loaded)
        encode_fixed_into(self._stage, self.model.ring, self.x.values, self._flag)
        if self._ev_free is None:
            self._ev_free = torch.cuda.Event()
        self._ev_free.record(main)
        self._flag_host.copy_(self._flag, non_blocking=True)
        self._batch_pending = False
        self._flag_pending = True

    def join_prefetch(self):
        """Make the current stream wait for the background work step() queued
        on the copy stream (the next step's input encryption), so a timing
        event recorded after this covers it."""
        if self.prefetch:
            torch.cuda.current_stream().wait_event(self._ev_ready)

    timing = None  # diagnostics: a list receives (label, CUDA event) at the step's phase boundaries

    def _mark(self, label):
        if self.timing is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.timing.append((label, ev))

    def _wait_logits(self):
        """Until the forward graph has published this step's logits (polling
        the pinned sequence word: no D2H copy, event or API call between the
        forward's last kernel and the DO's loss)."""
        want = self._pub_count & 0xFFFFFFFF
        pub = self._pub_np
        spins = 0
        while int(pub[0]) != want:
            spins += 1
            if spins & 0xFFFF == 0:  # now and then: a faulted or finished-but-silent forward
                # query() raises on a device fault; a completed forward must have published
                if self._ev_fwd.query() and int(pub[0]) != want:
                    from .errors import DeviceError

                    raise DeviceError("forward graph completed without publishing the logits")

    def _host_grad(self, labels):
        """The DO's loss gradient into g_host (raises on an out-of-range batch)."""
        if self._flag_pending:
            self._flag_pending = False
            if int(self._flag_np[0]):
                from .errors import EncodeRangeError

                limit = float(1 << (self.model.ring.ell - 1)) / float(1 << self.model.ring.f)
                raise EncodeRangeError(f"|x| must stay below {limit}")
        self._loss.grad(labels)

    def _host_loss(self, labels):
        self._host_grad(labels)
        return self._loss.value()

    def step(self, seed: int, labels, next_batch: torch.Tensor | None = None):
        """One private training step on the staged input; returns the DO's loss.
        ``next_batch`` (pinned float64 host tensor): stage the NEXT step's input
        right after this step's launches -- its H2D copy, encode and (with
        prefetch_input) encryption then overlap this step's backward, the
        pipelined form of ``load_batch`` for a training loop."""
        self.sess.reseed(seed, device_copy=not self.prologue)
        main = torch.cuda.current_stream()
        self._mark("start")
        if self.prefetch:
            main.wait_event(self._ev_ready)  # this step's input and its encryption
            if not self.prologue:
                self.x.values.copy_(self._x_next)
        elif self._batch_pending:
            self._encode_batch(main)
        self.g_fwd.replay()
        self._ev_fwd.record(main)
        self._mark("fwd")
        if not self.handoff:
            self._pre_stream.wait_stream(main)
            with torch.cuda.stream(self._pre_stream):  # backward operands, beside the host's loss
                self.g_pre.replay()
                self._ev_pre.record()
        self._pub_count += 1  # this replay's publication
        if self.handoff:  # the backward goes now; its chain waits on the device for the release below
            self.g_bwd.replay()
            self._mark("bwd")
            self._hseq += 1
            abort = 1
            try:
                self._wait_logits()
                if self._hseq > 1 and int(self._hflag_np[1]) != self._hseq - 1:
                    raise RuntimeError("backward graph: the previous step's loss handoff timed out")
                self._host_grad(labels)  # g written into g_host
                abort = 0
            finally:
                # release the backward even on error, so the GPU never waits for the
                # timeout; with the abort word set it runs on no fresh gradient and its
                # SGD launches (reading the skip word the handoff writes) are no-ops
                self._hflag_np[2] = abort
                self._hflag_np[0] = self._hseq & 0xFFFFFFFF
                if abort:  # after the skipped SGDs: later (eager) updates apply again
                    self.model.skip.zero_()
            loss = self._loss.value()  # the loss value after the release (off the GPU's path)
        else:
            self._wait_logits()
            loss = self._host_loss(labels)
            _lib.load().pb_copy_async(self._g_dev_ptr, self._g_host_ptr, self._g_bytes, main.cuda_stream)
            self._mark("host")
            main.wait_event(self._ev_pre)
            self._mark("pre")
            self.g_bwd.replay()
            self._mark("bwd")
        loaded_for_this = self._loaded_last
        self._loaded_last = False
        if next_batch is not None:
            self.load_batch(next_batch)
        elif self.prefetch and not loaded_for_this:  # resident input: encrypt it afresh for the next step
            self._copy_stream.wait_event(self._ev_fwd)
            self._schedule_encrypt()
        return loss


def synthetic_mnist(seed: int, B: int, ring: RingParams):
    """Same synthetic batch as the oracle: U[0,1] pixels standardised, labels U{0..9}.
    Returns host float64 features (784, B) and labels."""
    g = SeededRng(seed, 900)
    x = g.uniform_real((784, B), 0.0, 1.0)
    x = (x - 0.1307) / 0.3081
    labels = g._host_draw(lambda gen: gen.integers(0, 10, size=B))
    return x, labels


def synthetic_images(seed: int, B: int, in_shape, ring: RingParams):
    """Host float64 image batch (B, C, H, W) + labels, the oracle's draws
    (oracle/nn.synthetic_images): MNIST shapes reuse synthetic_mnist's pixels,
    CIFAR shapes draw U[0,1] standardised with (0.5, 0.25)."""
    if tuple(in_shape) == (1, 28, 28):
        x, labels = synthetic_mnist(seed, B, ring)
        return np.ascontiguousarray(x.T).reshape(B, 1, 28, 28), labels
    g = SeededRng(seed, 901)
    x = (g.uniform_real((B, *in_shape), 0.0, 1.0) - 0.5) / 0.25
    labels = g._host_draw(lambda gen: gen.integers(0, 10, size=B))
    return x, labels
