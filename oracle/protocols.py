"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the SPEC-only ``linear_protocols`` module (
PAPER.md Alg. 1, Alg. 2), the dealer-backed
non-linear steps it is composed with and the
reference fixed-point training engine.  Arithmetic goes
through oracle/bfv.py (K restated) and oracle/kernels.py; masks, shares and
reshares come from SeededRng streams (R:48-61), so the device engine, which
reproduces those streams bit-for-bit, must produce IDENTICAL shares.

Protocol conventions fixed here and mirrored by paper_2403_11166_b200:
  * activations are feature-major (n, B); FC weights (n_o, n_i); bias at 2f;
  * Alg.1: DO encrypts pi_v(<X>_1); MO evaluates W o Enc(<X>_1) - s_eff with
    s_eff = s - W o <X>_0 (equivalent to MO adding <X>_0 homomorphically,
    PAPER:341: the DO still decrypts W o X - s); MO outputs s + b;
  * Alg.2: one matmul geometry G1 = (n_i=B, n_o, B'=n_i); the cross terms
    <gY>_0 (x) Enc(pi_v(<X>_1^T)) and Enc(pi_W(<gY>_1)) (x) pi_v(<X>_0^T) land
    in the same pi_y layout (polynomial products commute) and are summed
    homomorphically before ONE mask s (n_o, n_i);
  * a term whose MO operand is known-zero (first layer <X>_0 = 0, loss
    gradient <gY>_0 = 0) is skipped -- it contributes exactly 0;
  * random streams: stream(layer, op, purpose) below; purpose 0 = MO mask,
    1 = DO encryption, 2 = dealer reshare, 3 = DP noise.
"""

from __future__ import annotations

import numpy as np

from . import bfv as OB
from . import convops as CO
from . import kernels as OK
from . import packing as PK
from .ring import DO, MO, RingParams, SeededRng, encode_fixed, to_signed

OP_FWD, OP_BWD_X, OP_GRAD_W, OP_GRAD_B, OP_RELU, OP_TRUNC_F, OP_TRUNC_B, OP_RELU_B, OP_POOL_F, OP_POOL_B = range(10)
P_MASK, P_ENC, P_DEALER, P_DP, P_OT = range(5)


def stream_id(layer: int, op: int, purpose: int) -> int:
    return 1_000_000 + 1000 * layer + 10 * op + purpose


class Ctx:
    """Both parties' state for the oracle run (keys live with the DO)."""

    def __init__(self, params, ring: RingParams, kp, seed: int, ar=None):
        self.p = params
        self.ring = ring
        self.kp = kp
        self.seed = seed
        self.ar = ar or OB.Arith(params)

    def rng(self, layer, op, purpose):
        return SeededRng(self.seed, stream_id(layer, op, purpose))


def _mask(v, ring):
    return np.asarray(v, dtype=np.uint64) & ring.mask


class DpConfig:
    def __init__(self, sigma=0.0, C=1.0, B=1, enabled=False):
        if sigma < 0 or C <= 0:
            raise ValueError("DpConfig needs sigma >= 0 and C > 0")
        self.sigma, self.C, self.B, self.enabled = float(sigma), float(C), int(B), bool(enabled)


def sample_dp_noise(shape, dp, rng):
    """e ~ N(0, sigma^2 C^2 / B) per element via R:80-81 ``normal`` (zeros when disabled or sigma = 0)."""
    if dp is None or not dp.enabled or dp.sigma == 0.0:
        return np.zeros(shape)
    return rng.normal(shape, dp.sigma * dp.C / np.sqrt(dp.B))


def dp_noise(seed, layer, op, shape, scale, dp, ring):
    """The DO's encoded DP perturbation for one reveal: drawn
    from SeededRng(seed, stream_id(layer, op, P_DP)), encoded at the scale of
    the revealed value (grad b: f, grad W before the shift: 2f); None when DP
    is off.  The reference engine draws the same stream ("same DP hook")."""
    if dp is None or not dp.enabled:
        return None
    e = sample_dp_noise(shape, dp, SeededRng(seed, stream_id(layer, op, P_DP)))
    return encode_fixed(e, ring, scale)


def he_matmul(ctx: Ctx, v_ct_vals, v_pt_vals, W_pt_vals, W_ct_vals, g: PK.MatmulGeometry, s_eff, enc_rng):
    """Shared MO/DO evaluation of  W o v  with the cross-term structure:
    sum over present terms of  Enc(pi_v(v_ct)) (x) pi_W(W_pt)  and
    Enc(pi_W(W_ct)) (x) pi_v(v_pt), minus Delta*pi_y(s_eff); returns the DO's
    decrypted share (n_o, B).  Any *_vals may be None (term absent)."""
    plan = PK.plan_blocks(g, ctx.p.N)
    return he_eval(ctx, plan, v_ct_vals, v_pt_vals, W_pt_vals, W_ct_vals, s_eff, g.n_o * g.B,
                   enc_rng).reshape(g.n_o, g.B)


def he_eval(ctx: Ctx, plan, v_ct_vals, v_pt_vals, W_pt_vals, W_ct_vals, s_eff, out_size, enc_rng):
    """he_matmul over an arbitrary block plan (matmul or conv-layer packing):
    returns the DO's decrypted flat share of size ``out_size``."""
    p, ar = ctx.p, ctx.ar
    outs = np.zeros((plan.n_out, 2, p.L, p.N), dtype=np.uint64)

    def mac(cts, pts, ct_col, pt_col):  # outs[r] += sum_k cts[terms[r,k,ct_col]] (x) pts[terms[r,k,pt_col]]
        CH = 32
        for a in range(0, plan.n_out, CH):
            sl = slice(a, min(a + CH, plan.n_out))
            acc = outs[sl].reshape(-1, p.L, p.N)
            for k in range(plan.terms.shape[1]):
                A = np.ascontiguousarray(cts[plan.terms[sl, k, ct_col]]).reshape(-1, p.L, p.N)
                Bm = np.ascontiguousarray(np.repeat(pts[plan.terms[sl, k, pt_col]][:, None], 2, axis=1))
                ar.mac(acc, A, Bm.reshape(-1, p.L, p.N))

    if v_ct_vals is not None:  # Enc(pi_v(v)) (x) pi_W(W)
        ct_v = OB.encrypt_pk(p, ctx.kp, PK.pack(plan.in_src, v_ct_vals), enc_rng, ar)
        pt_w = OB.encode_plain(p, PK.pack(plan.pt_src, W_pt_vals), ar)
        mac(ct_v, pt_w, 0, 1)
    if W_ct_vals is not None:  # Enc(pi_W(W)) (x) pi_v(v)
        ct_w = OB.encrypt_pk(p, ctx.kp, PK.pack(plan.pt_src, W_ct_vals), enc_rng, ar)
        pt_v = OB.encode_plain(p, PK.pack(plan.in_src, v_pt_vals), ar)
        mac(ct_w, pt_v, 1, 0)
    # MO masks every output ciphertext with pi_y(s_eff)
    mpoly = np.zeros((plan.n_out, p.N), dtype=np.uint64)
    ok = plan.out_pos >= 0
    mpoly[np.nonzero(ok)[0], plan.out_pos[ok]] = np.asarray(s_eff, dtype=np.uint64).ravel()[plan.out_dst[ok]]
    outs = OB.he_add_plain(p, outs, mpoly, ar, subtract=True)
    # DO decrypts and gathers pi_y^-1
    dec = OB.decrypt(p, ctx.kp, outs, ar)
    return PK.unpack(dec, plan, out_size)


def linear_forward(ctx: Ctx, layer: int, W, b, x_mo, x_do, mo_x_zero=False):  # Alg.1
    """W (n_o, n_i) at f, b (n_o,) at 2f, x shares (n_i, B) at f -> (y_mo, y_do) at 2f."""
    ring = ctx.ring
    n_o, n_i = W.shape
    B = x_do.shape[1]
    s = ctx.rng(layer, OP_FWD, P_MASK).uniform_ring((n_o, B), ring)
    s_eff = s if mo_x_zero else _mask(s - OK.matmul_wrap(W, x_mo), ring)
    y_do = he_matmul(ctx, x_do, None, W, None, PK.MatmulGeometry(n_i, n_o, B), s_eff,
                     ctx.rng(layer, OP_FWD, P_ENC))
    y_mo = _mask(s + b[:, None], ring)
    return y_mo, y_do


def linear_backward_input(ctx: Ctx, layer: int, W, gy_mo, gy_do, mo_gy_zero=False):
    """grad X = W^T gY at 2f, Alg.1 message pattern with W^T."""
    ring = ctx.ring
    n_o, n_i = W.shape
    B = gy_do.shape[1]
    Wt = np.ascontiguousarray(W.T)
    s = ctx.rng(layer, OP_BWD_X, P_MASK).uniform_ring((n_i, B), ring)
    s_eff = s if mo_gy_zero else _mask(s - OK.matmul_wrap(Wt, gy_mo), ring)
    g_do = he_matmul(ctx, gy_do, None, Wt, None, PK.MatmulGeometry(n_o, n_i, B), s_eff,
                     ctx.rng(layer, OP_BWD_X, P_ENC))
    return s, g_do


def reveal_grad_bias(ctx: Ctx, layer: int, gy_mo, gy_do, e=None):
    """Local batch sums; DO adds encode(e) (scale f); MO reconstructs (scale f)."""
    ring = ctx.ring
    do_sum = _mask(gy_do.sum(axis=1, dtype=np.uint64), ring)
    if e is not None:
        do_sum = _mask(do_sum + e, ring)
    return _mask(gy_mo.sum(axis=1, dtype=np.uint64) + do_sum, ring)


def grad_weight(ctx: Ctx, layer: int, x_mo, x_do, gy_mo, gy_do, e=None, mo_x_zero=False, mo_gy_zero=False):
    """Alg.2: returns grad W revealed at MO, scale 2f (n_o, n_i)."""
    ring = ctx.ring
    n_i, B = x_do.shape
    n_o = gy_do.shape[0]
    g = PK.MatmulGeometry(B, n_o, n_i)  # v = X^T (B x n_i), W = gY (n_o x B)
    s = ctx.rng(layer, OP_GRAD_W, P_MASK).uniform_ring((n_o, n_i), ring)
    xdT = np.ascontiguousarray(x_do.T)
    xmT = np.ascontiguousarray(x_mo.T)
    cross_do = he_matmul(
        ctx,
        None if mo_gy_zero else xdT, None if mo_x_zero else xmT,
        None if mo_gy_zero else gy_mo, None if mo_x_zero else gy_do,
        g, s, ctx.rng(layer, OP_GRAD_W, P_ENC),
    )
    msg = _mask(cross_do + OK.matmul_wrap(gy_do, xdT), ring)  # DO: + local term
    if e is not None:
        msg = _mask(msg + e, ring)
    return _mask(msg + s + OK.matmul_wrap(gy_mo, xmT), ring)  # MO: + s + local term


# ------------------------------------------------------- conv layers ---
# Conv2d layers (SPEC:249-266 packing, SPEC:284-286 transforms): activations
# (B, C, H, W), weights (c_o, c_i, s, s) at f, bias (c_o,) at 2f.  Every
# operator uses the native conv packing with padding / stride / flips folded
# into the plan's index maps (packing.plan_conv_layer); the MO's local terms
# use the matching plaintext operators (convops).


def conv_forward(ctx: Ctx, layer: int, W, b, x_mo, x_do, pad: int, stride: int, mo_x_zero=False):
    """Alg.1 with conv packing: shares of Y = conv(X; W) + b at 2f, (B, c_o, oh, ow)."""
    ring = ctx.ring
    B, c_i, H, Wd = x_do.shape
    c_o, _, s, _ = W.shape
    oh, ow = PK.conv_out_hw(H, Wd, s, pad, stride)
    msk = ctx.rng(layer, OP_FWD, P_MASK).uniform_ring((B, c_o, oh, ow), ring)
    s_eff = msk if mo_x_zero else _mask(msk - CO.conv_fwd(x_mo, W, pad, stride), ring)
    plan = PK.plan_conv_layer("fwd", B, c_i, c_o, H, Wd, s, pad, stride, ctx.p.N)
    y_do = he_eval(ctx, plan, x_do, None, W, None, s_eff, B * c_o * oh * ow,
                   ctx.rng(layer, OP_FWD, P_ENC)).reshape(B, c_o, oh, ow)
    y_mo = _mask(msk + b[None, :, None, None], ring)
    return y_mo, y_do


def conv_backward_input(ctx: Ctx, layer: int, W, gy_mo, gy_do, H: int, Wd: int, pad: int, stride: int,
                        mo_gy_zero=False):
    """SPEC:321-329 for Conv2d: shares of dX = conv_fwd^T(dY) at 2f, (B, c_i, H, W)."""
    ring = ctx.ring
    B, c_o = gy_do.shape[:2]
    c_i, s = W.shape[1], W.shape[2]
    msk = ctx.rng(layer, OP_BWD_X, P_MASK).uniform_ring((B, c_i, H, Wd), ring)
    plan = PK.plan_conv_layer("bwdx", B, c_i, c_o, H, Wd, s, pad, stride, ctx.p.N)
    # input positions no output reads (stride > 1 tails) have gradient exactly 0:
    # no ciphertext slot carries them, so the MO's share there is 0 as well
    covered = np.zeros(B * c_i * H * Wd, dtype=bool)
    covered[plan.out_dst[plan.out_dst >= 0]] = True
    msk = np.where(covered.reshape(msk.shape), msk, np.uint64(0))
    s_eff = msk if mo_gy_zero else _mask(msk - CO.conv_bwdx(gy_mo, W, H, Wd, pad, stride), ring)
    g_do = he_eval(ctx, plan, gy_do, None, W, None, s_eff, B * c_i * H * Wd,
                   ctx.rng(layer, OP_BWD_X, P_ENC)).reshape(B, c_i, H, Wd)
    return msk, g_do


def conv_grad_weight(ctx: Ctx, layer: int, x_mo, x_do, gy_mo, gy_do, s: int, pad: int, stride: int, e=None,
                     mo_x_zero=False, mo_gy_zero=False):
    """Alg.2 for Conv2d: dW = sum_b,y,x dY Xpad revealed at MO, scale 2f, (c_o, c_i, s, s)."""
    ring = ctx.ring
    B, c_i, H, Wd = x_do.shape
    c_o = gy_do.shape[1]
    msk = ctx.rng(layer, OP_GRAD_W, P_MASK).uniform_ring((c_o, c_i, s, s), ring)
    plan = PK.plan_conv_layer("gradw", B, c_i, c_o, H, Wd, s, pad, stride, ctx.p.N)
    cross_do = he_eval(ctx, plan,
                       None if mo_gy_zero else x_do, None if mo_x_zero else x_mo,
                       None if mo_gy_zero else gy_mo, None if mo_x_zero else gy_do,
                       msk, c_o * c_i * s * s, ctx.rng(layer, OP_GRAD_W, P_ENC)).reshape(c_o, c_i, s, s)
    msg = _mask(cross_do + CO.conv_gradw(x_do, gy_do, s, pad, stride), ring)  # DO: + local term
    if e is not None:
        msg = _mask(msg + e, ring)
    return _mask(msg + msk + CO.conv_gradw(x_mo, gy_mo, s, pad, stride), ring)  # MO: + s + local term


def reveal_grad_bias_conv(ctx: Ctx, layer: int, gy_mo, gy_do, e=None):
    """SPEC:330-338 for Conv2d: local sums over batch and spatial positions per channel."""
    ring = ctx.ring
    do_sum = _mask(gy_do.sum(axis=(0, 2, 3), dtype=np.uint64), ring)
    if e is not None:
        do_sum = _mask(do_sum + e, ring)
    return _mask(gy_mo.sum(axis=(0, 2, 3), dtype=np.uint64) + do_sum, ring)


def avgpool_forward(ctx: Ctx, layer: int, a_mo, a_do):
    """local 2x2 window sums, then a 2-bit truncation (dealer)."""
    s_mo, s_do = CO.pool_sum(a_mo), CO.pool_sum(a_do)
    r, y, _ = dealer_op(ctx, layer, OP_POOL_F, s_mo, s_do, k=2)
    return r, y


def avgpool_backward(ctx: Ctx, layer: int, g_mo, g_do):
    """Replicate each gradient to its 2x2 window, then a 2-bit truncation (dealer)."""
    r, y, _ = dealer_op(ctx, layer, OP_POOL_B, CO.pool_replicate(g_mo), CO.pool_replicate(g_do), k=2)
    return r, y


# ----------------------------------------------------- dealer non-linear ---

def ot_op(ctx: Ctx, layer: int, op: int, kind: str, y_mo, y_do, k: int = 0, d=None):
    """The OT-protocol backend (oracle/nonlinear.py) on stream (layer, op, P_OT):
    kind in drelu / mux / trunc / relu_trunc / trunc_mux; returns (mo, do, d)."""
    from . import nonlinear as NL

    shape = np.shape(y_mo)
    y0, y1, dd = NL.nl_op(kind, y_mo, y_do, ctx.ring.ell, k=k, d=d, seed=ctx.seed,
                          stream=stream_id(layer, op, P_OT))
    if dd is not None:
        dd = dd.reshape(shape)
    if y0 is None:
        return None, None, dd
    return y0.reshape(shape), y1.reshape(shape), dd


def dealer_op(ctx: Ctx, layer: int, op: int, y_mo, y_do, k: int = 0, d=None):
    """Reconstruct, apply, reshare with r = uniform_ring(stream(layer, op, dealer))."""
    ring = ctx.ring
    x = _mask(y_mo + y_do, ring)
    sx = to_signed(x, ring)
    d_out = None
    if op == OP_RELU:
        d_out = (sx >= 0).astype(np.uint8)
        y = np.where(sx >= 0, x, np.uint64(0))
    elif op in (OP_TRUNC_F, OP_TRUNC_B, OP_POOL_F, OP_POOL_B):
        y = _mask((sx >> np.int64(k)).astype(np.uint64), ring)
    elif op == OP_RELU_B:
        y = np.where(d.astype(bool), x, np.uint64(0))
    else:
        raise ValueError(op)
    r = ctx.rng(layer, op, P_DEALER).uniform_ring(x.shape, ring)
    return r, _mask(y - r, ring), d_out


# ------------------------------------------------------------ the model ---

def softmax_ce_grad(logits_2f, labels, ring: RingParams, denom: int = 0):
    """DO-side loss: logits decoded at 2f (n_classes, B);
    ``denom``: the gradient's batch divisor (0: B; data parallel: the global batch)."""
    z = to_signed(logits_2f, ring).astype(np.float64) / float(1 << (2 * ring.f))
    z = z - z.max(axis=0, keepdims=True)
    ez = np.exp(z)
    sm = ez / ez.sum(axis=0, keepdims=True)
    B = z.shape[1]
    onehot = np.zeros_like(sm)
    onehot[labels, np.arange(B)] = 1.0
    loss = float(-np.mean(np.log(sm[labels, np.arange(B)])))
    g = (sm - onehot) / (denom if denom else B)
    v = np.floor(g * float(1 << ring.f)).astype(np.int64)
    return loss, v.astype(np.uint64) & ring.mask
