"""ORACLE — TEST INFRASTRUCTURE ONLY.

The SPEC-only ``nn`` module restated for the oracle:
models, the private training step composed from oracle/protocols.py, and
``reference_train_step`` -- the fixed-point Z_t pipeline without any
cryptography that SPEC:620-628 defines as THE oracle for training parity.

Model graphs (PAPER Appendix D) are lists of layer specs:
  ("fc", n_i, n_o)                       feature-major activations (n, B)
  ("conv", c_i, c_o, s, pad, stride)     activations (B, C, H, W)
  ("pool",)                              AvgPool2
  ("flatten",)                           (B, C, H, W) -> (C*H*W, B)
Every linear layer except the last is followed by ReLU + truncation by f.

Step semantics (shared with paper_2403_11166_b200/nn.py):
  forward  Y_l = lin_l(X_{l-1}) + b_l (2f); A_l = trunc_f(relu(Y_l)) (f) for l < last;
           pool: trunc_2(window sums); flatten: local transpose
  loss     DO reconstructs logits (2f), softmax-CE in float64, g = encode_f((p - y)/B)
           with the MO's share of g set to 0
  backward gb_l = sums of gY_l (f); gW_l = arith_shift(grad_w(X_{l-1}, gY_l), f) (2f -> f)
           gA_{l-1} = trunc_f(lin_l^T gY_l); pool: trunc_2(replicate); flatten^-1;
           gY_{l-1} = relu'(Y_{l-1}) * gA_{l-1}
  update   SGD momentum in float64 on master weights:
           v = mu v + g;  w = w - lr v;  W = encode_f(w), b = encode_2f(b)
"""

from __future__ import annotations

import numpy as np

from . import convops as CO
from . import kernels as OK
from . import protocols as PR
from .packing import conv_out_hw
from .ring import RingParams, SeededRng, decode_fixed, encode_fixed, to_signed

MODELS = {
    # PAPER Fig. 5 / SPEC:608
    "mnist_mlp": ((784,), [("fc", 784, 128), ("fc", 128, 128), ("fc", 128, 10)]),
    # PAPER Fig. 6 / SPEC:609: Conv 1->5 5x5 s2 p2, FC 980->100, FC 100->10
    "mnist_cnn": ((1, 28, 28), [("conv", 1, 5, 5, 2, 2), ("flatten",), ("fc", 980, 100), ("fc", 100, 10)]),
    # BASELINE configs[2] "2 x conv5x5 + FC": the paper's CNN plus a documented second conv
    "mnist_cnn2": ((1, 28, 28), [("conv", 1, 5, 5, 2, 2), ("conv", 5, 5, 5, 2, 1), ("flatten",),
                                 ("fc", 980, 100), ("fc", 100, 10)]),
    # PAPER Fig. 7: the private-conv CIFAR-10 CNN
    "cifar_cnn": ((3, 32, 32), [("conv", 3, 64, 5, 2, 1), ("pool",), ("conv", 64, 64, 5, 2, 1), ("pool",),
                                ("conv", 64, 64, 3, 1, 1), ("conv", 64, 64, 1, 0, 1), ("conv", 64, 16, 1, 0, 1),
                                ("flatten",), ("fc", 1024, 10)]),
}


def mlp_spec(sizes):
    return (sizes[0],), [("fc", a, b) for a, b in zip(sizes[:-1], sizes[1:])]


def shapes(in_shape, layers):
    """Per-entry (input shape, output shape) of one sample, validating composition."""
    cur = tuple(in_shape)
    out = []
    for e in layers:
        if e[0] == "fc":
            if cur != (e[1],):
                raise ValueError(f"fc expects ({e[1]},), got {cur}")
            nxt = (e[2],)
        elif e[0] == "conv":
            _, ci, co, s, p, st = e
            if len(cur) != 3 or cur[0] != ci:
                raise ValueError(f"conv expects {ci} channels, got {cur}")
            nxt = (co, *conv_out_hw(cur[1], cur[2], s, p, st))
        elif e[0] == "pool":
            if len(cur) != 3 or cur[1] % 2 or cur[2] % 2:
                raise ValueError("avgpool2 needs even spatial dims")
            nxt = (cur[0], cur[1] // 2, cur[2] // 2)
        elif e[0] == "flatten":
            nxt = (int(np.prod(cur)),)
        else:
            raise ValueError(f"unknown layer {e!r}")
        out.append((cur, nxt))
        cur = nxt
    return out


class Model:
    """``Model(sizes)`` = FC stack (MLP); ``Model(name)`` / ``Model((in_shape, layers))`` = graph."""

    def __init__(self, arch, ring: RingParams, seed: int = 0):
        if isinstance(arch, str):
            arch = MODELS[arch]
        if isinstance(arch, (list, tuple)) and all(isinstance(v, (int, np.integer)) for v in arch):
            arch = mlp_spec(list(arch))
        self.in_shape, self.layers = tuple(arch[0]), list(arch[1])
        self.io = shapes(self.in_shape, self.layers)
        self.lin = [i for i, e in enumerate(self.layers) if e[0] in ("fc", "conv")]
        self.ring = ring
        self.w, self.b, self.vw, self.vb = [], [], [], []
        for l, i in enumerate(self.lin):
            e = self.layers[i]
            if e[0] == "fc":
                wshape, fan_in, nb = (e[2], e[1]), e[1], e[2]
            else:
                wshape, fan_in, nb = (e[2], e[1], e[3], e[3]), e[1] * e[3] * e[3], e[2]
            g = SeededRng(seed, 500 + l)  # SPEC:646 init
            a = np.sqrt(1.0 / fan_in)
            self.w.append(g.uniform_real(wshape, -a, a))
            self.b.append(g.uniform_real((nb,), -a, a))
            self.vw.append(np.zeros(wshape))
            self.vb.append(np.zeros(nb))

    @property
    def sizes(self):  # MLP compatibility
        return [self.layers[self.lin[0]][1]] + [self.layers[i][2] for i in self.lin]

    @property
    def n_layers(self):
        return len(self.lin)

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


def _flatten(x):  # (B, C, H, W) -> (C*H*W, B)
    return np.ascontiguousarray(x.reshape(x.shape[0], -1).T)


def _unflatten(g, shape):  # (C*H*W, B) -> (B, C, H, W)
    return np.ascontiguousarray(g.T).reshape(-1, *shape)


def _segments(model):
    """For each linear l: the entries between linear l and linear l+1."""
    seg = []
    for l, i in enumerate(model.lin):
        j = model.lin[l + 1] if l + 1 < model.n_layers else len(model.layers)
        seg.append(list(range(i + 1, j)))
    return seg


def _dp_noise(dp, seed, l, kind, shape, ring):
    """(grad-b noise at f, grad-W noise at 2f) of layer l: the DO's DP hook."""
    if dp is None or not dp.enabled:
        return None, None
    return (PR.dp_noise(seed, l, PR.OP_GRAD_B, (shape[0],), ring.f, dp, ring),
            PR.dp_noise(seed, l, PR.OP_GRAD_W, shape, 2 * ring.f, dp, ring))


def reference_train_step(model: Model, x_enc, labels, lr=1e-2, momentum=0.8, dp=None, dp_seed=0):
    """the exact Z_t fixed-point pipeline, no cryptography.
    ``dp`` (a DpConfig) adds the DO's perturbation drawn from
    the streams the private step uses under session seed ``dp_seed``
    ("same DP hook")."""
    ring, f = model.ring, model.ring.f
    L = model.n_layers
    seg = _segments(model)
    cur, acts, pre = x_enc, [], []
    for l, i in enumerate(model.lin):
        e = model.layers[i]
        acts.append(cur)
        if e[0] == "fc":
            y = _m(OK.matmul_wrap(model.W(l), cur) + model.Bias(l)[:, None], ring)
        else:
            y = _m(CO.conv_fwd(cur, model.W(l), e[4], e[5]) + model.Bias(l)[None, :, None, None], ring)
        pre.append(y)
        if l < L - 1:
            cur = _shift(np.where(to_signed(y, ring) >= 0, y, np.uint64(0)), f, ring)
            for k in seg[l]:
                if model.layers[k][0] == "pool":
                    cur = _shift(_m(CO.pool_sum(cur), ring), 2, ring)
                elif model.layers[k][0] == "flatten":
                    cur = _flatten(cur)
    loss, gy = PR.softmax_ce_grad(pre[-1], labels, ring)
    gws, gbs = [None] * L, [None] * L
    for l in reversed(range(L)):
        e = model.layers[model.lin[l]]
        wshape = (e[2], e[1]) if e[0] == "fc" else (e[2], e[1], e[3], e[3])
        eb, ew = _dp_noise(dp, dp_seed, l, e[0], wshape, ring)
        if e[0] == "fc":
            gbs[l] = _m(gy.sum(axis=1, dtype=np.uint64), ring)
            gw = _m(OK.matmul_wrap(gy, np.ascontiguousarray(acts[l].T)), ring)
        else:
            gbs[l] = _m(gy.sum(axis=(0, 2, 3), dtype=np.uint64), ring)
            gw = _m(CO.conv_gradw(acts[l], gy, e[3], e[4], e[5]), ring)
        if eb is not None:
            gbs[l], gw = _m(gbs[l] + eb, ring), _m(gw + ew, ring)
        gws[l] = _shift(gw, f, ring)
        if l > 0:
            if e[0] == "fc":
                ga = _m(OK.matmul_wrap(np.ascontiguousarray(model.W(l).T), gy), ring)
            else:
                H, Wd = acts[l].shape[2:]
                ga = _m(CO.conv_bwdx(gy, model.W(l), H, Wd, e[4], e[5]), ring)
            ga = _shift(ga, f, ring)
            for k in reversed(seg[l - 1]):
                if model.layers[k][0] == "pool":
                    ga = _shift(_m(CO.pool_replicate(ga), ring), 2, ring)
                elif model.layers[k][0] == "flatten":
                    ga = _unflatten(ga, model.io[k][0])
            gy = np.where(to_signed(pre[l - 1], ring) >= 0, ga, np.uint64(0))
    model.sgd(gws, gbs, lr, momentum)
    return loss, gws, gbs


def _allsum(v, group, ring):
    """Sum of a revealed gradient over the data-parallel ranks, exactly mod 2^ell
    (all_gather + numpy uint64 sum: no reliance on a backend's int64 wrap)."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(v).view(np.int64))
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    acc = np.zeros_like(np.asarray(v, dtype=np.uint64))
    for p in parts:
        acc = acc + p.numpy().view(np.uint64)
    return _m(acc, ring)


def private_train_step(ctx: PR.Ctx, model: Model, x_enc, labels, lr=1e-2, momentum=0.8, trace=None, prep=None,
                       dp=None, dp_group=None, nonlinear="dealer"):
    """SPEC:629-637 with fullhe linear layers (oracle/protocols.py) -- or, with
    ``prep`` (a preprocessing.PrepState), the HE-free online linear layers of
    Alg. 4 (mode "prep") -- and the dealer non-linear backend;
    <X_0>_0 = 0 at MO, <X_0>_1 = X at DO.  ``dp``: the DO's DP perturbation of
    the revealed gradients, drawn from the ctx.seed streams.
    ``dp_group``: data-parallel ranks (torch.distributed), each with its own
    batch: the loss gradient divided by the global batch, the revealed
    gradients summed over ranks before the shift and SGD (= the reference
    engine on the concatenated batch).  ``nonlinear="ot"``: ReLU / truncation /
    pooling through the OT-based protocols (oracle/nonlinear.py), composed
    exactly as the engine composes them (nn.py: ReLU + truncation fused, the
    backward truncation fused with ReLU' unless a pooling sits in between)."""
    from . import preprocessing as PP

    ring, f = model.ring, model.ring.f
    L = model.n_layers
    seg = _segments(model)
    cur = (np.zeros_like(x_enc), x_enc.copy())
    acts, ds, ys = [], [], []
    for l, i in enumerate(model.lin):
        e = model.layers[i]
        acts.append(cur)
        if prep is not None:
            y = PP.prep_linear_forward(ctx, l, prep.banks[l], model.W(l), model.Bias(l), *cur)
        elif e[0] == "fc":
            y = PR.linear_forward(ctx, l, model.W(l), model.Bias(l), *cur, mo_x_zero=(l == 0))
        else:
            y = PR.conv_forward(ctx, l, model.W(l), model.Bias(l), *cur, e[4], e[5], mo_x_zero=(l == 0))
        ys.append(y)
        if l < L - 1:
            if nonlinear == "ot":
                a_mo, a_do, d = PR.ot_op(ctx, l, PR.OP_TRUNC_F, "relu_trunc", *y, k=f)
            else:
                z_mo, z_do, d = PR.dealer_op(ctx, l, PR.OP_RELU, *y)
                a_mo, a_do, _ = PR.dealer_op(ctx, l, PR.OP_TRUNC_F, z_mo, z_do, k=f)
            ds.append(d)
            cur = (a_mo, a_do)
            for k in seg[l]:
                if model.layers[k][0] == "pool":
                    if nonlinear == "ot":
                        s_mo, s_do = CO.pool_sum(cur[0]), CO.pool_sum(cur[1])
                        cur = PR.ot_op(ctx, l, PR.OP_POOL_F, "trunc", s_mo, s_do, k=2)[:2]
                    else:
                        cur = PR.avgpool_forward(ctx, l, *cur)
                elif model.layers[k][0] == "flatten":
                    cur = (_flatten(cur[0]), _flatten(cur[1]))
    logits = _m(ys[-1][0] + ys[-1][1], ring)  # MO sends its share; DO reconstructs
    denom = 0
    if dp_group is not None:
        import torch.distributed as dist

        denom = logits.shape[1] * dist.get_world_size(dp_group)
    loss, g = PR.softmax_ce_grad(logits, labels, ring, denom)
    gy_mo, gy_do = np.zeros_like(g), g
    gws, gbs = [None] * L, [None] * L
    for l in reversed(range(L)):
        e = model.layers[model.lin[l]]
        last = l == L - 1
        wshape = (e[2], e[1]) if e[0] == "fc" else (e[2], e[1], e[3], e[3])
        eb, ew = _dp_noise(dp, ctx.seed, l, e[0], wshape, ring)
        if prep is not None:
            gbs[l] = (PR.reveal_grad_bias if e[0] == "fc" else PR.reveal_grad_bias_conv)(ctx, l, gy_mo, gy_do, e=eb)
            gw2f = PP.prep_grad_weight(ctx, l, prep.banks[l], *acts[l], gy_mo, gy_do, e=ew)
        elif e[0] == "fc":
            gbs[l] = PR.reveal_grad_bias(ctx, l, gy_mo, gy_do, e=eb)
            gw2f = PR.grad_weight(ctx, l, *acts[l], gy_mo, gy_do, e=ew, mo_x_zero=(l == 0), mo_gy_zero=last)
        else:
            gbs[l] = PR.reveal_grad_bias_conv(ctx, l, gy_mo, gy_do, e=eb)
            gw2f = PR.conv_grad_weight(ctx, l, *acts[l], gy_mo, gy_do, e[3], e[4], e[5], e=ew, mo_x_zero=(l == 0),
                                       mo_gy_zero=last)
        if dp_group is not None:
            gw2f, gbs[l] = _allsum(gw2f, dp_group, ring), _allsum(gbs[l], dp_group, ring)
        gws[l] = _shift(gw2f, f, ring)  # MO: plaintext shift
        if trace is not None:
            trace.append((l, ys[l], gbs[l], gws[l]))
        if l > 0:
            if prep is not None:
                ga = PP.prep_linear_backward_input(ctx, l, prep.banks[l], model.W(l), gy_mo, gy_do)
            elif e[0] == "fc":
                ga = PR.linear_backward_input(ctx, l, model.W(l), gy_mo, gy_do, mo_gy_zero=last)
            else:
                H, Wd = acts[l][1].shape[2:]
                ga = PR.conv_backward_input(ctx, l, model.W(l), gy_mo, gy_do, H, Wd, e[4], e[5], mo_gy_zero=last)
            pooled = any(model.layers[k][0] == "pool" for k in seg[l - 1])
            if nonlinear == "ot" and not pooled:  # truncation + ReLU' fused (the engine's composition)
                t_mo, t_do = ga
                for k in reversed(seg[l - 1]):
                    if model.layers[k][0] == "flatten":
                        t_mo, t_do = _unflatten(t_mo, model.io[k][0]), _unflatten(t_do, model.io[k][0])
                gy_mo, gy_do, _ = PR.ot_op(ctx, l - 1, PR.OP_RELU_B, "trunc_mux", t_mo, t_do, k=f, d=ds[l - 1])
            else:
                if nonlinear == "ot":
                    t_mo, t_do, _ = PR.ot_op(ctx, l, PR.OP_TRUNC_B, "trunc", *ga, k=f)
                else:
                    t_mo, t_do, _ = PR.dealer_op(ctx, l, PR.OP_TRUNC_B, *ga, k=f)
                for k in reversed(seg[l - 1]):
                    if model.layers[k][0] == "pool":
                        if nonlinear == "ot":
                            r_mo, r_do = CO.pool_replicate(t_mo), CO.pool_replicate(t_do)
                            t_mo, t_do, _ = PR.ot_op(ctx, l - 1, PR.OP_POOL_B, "trunc", r_mo, r_do, k=2)
                        else:
                            t_mo, t_do = PR.avgpool_backward(ctx, l - 1, t_mo, t_do)
                    elif model.layers[k][0] == "flatten":
                        t_mo, t_do = _unflatten(t_mo, model.io[k][0]), _unflatten(t_do, model.io[k][0])
                if nonlinear == "ot":
                    gy_mo, gy_do, _ = PR.ot_op(ctx, l - 1, PR.OP_RELU_B, "mux", t_mo, t_do, d=ds[l - 1])
                else:
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


def synthetic_images(seed: int, B: int, in_shape, ring: RingParams):
    """Image-shaped batch (B, C, H, W) for the CNNs: MNIST shapes reuse
    synthetic_mnist's pixels; CIFAR shapes draw U[0,1] per channel,
    standardised with (0.5, 0.25)."""
    if tuple(in_shape) == (1, 28, 28):
        x, labels = synthetic_mnist(seed, B, ring)
        return np.ascontiguousarray(x.T).reshape(B, 1, 28, 28), labels
    g = SeededRng(seed, 901)
    x = (g.uniform_real((B, *in_shape), 0.0, 1.0) - 0.5) / 0.25
    labels = g._gen.integers(0, 10, size=B)
    return encode_fixed(x, ring), labels
