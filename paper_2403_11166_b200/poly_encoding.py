"""Coefficient packings pi_v, pi_W, pi_y and block plans (the SPEC-only
``poly_encoding`` module; Appendix A, 1208-1247).

matmul
    input  coefficient  k*n_o*n_i + j            <- v[j, k]
    weight coefficient  i*n_i + n_i - 1 - j      <- W[i, j]
    output y[i, k]  at  k*n_o*n_i + i*n_i + n_i - 1
conv, O = (c_i-1)hw + (s-1)w + s-1
    index_v(b,c,i,j)  = b c_o c_i h w + c h w + i w + j
    index_W(c',c,i,j) = O + c' c_i h w - c h w - i w - j,   i, j in [s]
    index_y(b,c',i,j) = b c_o c_i h w + O + c' c_i h w + i w + j

Block plan: shrink the batch block first, then
the output dimension, then the input dimension; input-dimension blocks are
accumulated homomorphically (the ``terms`` of one output ciphertext).  All
blocks use the nominal block dimensions in their exponents.

Plans are pure index maps computed once per (geometry, layout) on the host
and cached on the device; the fused kernels gather through them (pb_bfv.cu),
so packing never materialises a dense polynomial in HBM.  Operands are
addressed through strides, which lets the backward operators (W^T, X^T)
reuse the same codec without transposing data.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from .errors import GeometryError


@dataclass(frozen=True)
class MatmulGeometry:
    n_i: int
    n_o: int
    B: int


@dataclass(frozen=True)
class ConvGeometry:  # SPEC:221-224 (valid cross-correlation, stride 1)
    B: int
    c_i: int
    c_o: int
    h: int
    w: int
    s: int


@dataclass
class BlockPlan:
    kind: str
    geometry: object
    N: int
    blk: tuple
    nblk: tuple
    in_src: np.ndarray   # [n_in, N]  flat source index of the encrypted-side operand, -1 = zero
    pt_src: np.ndarray   # [n_pt, N]  flat source index of the plaintext-side operand
    out_pos: np.ndarray  # [n_out, U] coefficient positions of useful outputs, -1 = none
    out_dst: np.ndarray  # [n_out, U] flat destination index of each useful output
    terms: np.ndarray    # [n_out, K, 2] (input poly, weight poly) accumulated per output
    _dev: dict = field(default_factory=dict, repr=False)

    @property
    def n_in(self):
        return self.in_src.shape[0]

    @property
    def n_pt(self):
        return self.pt_src.shape[0]

    @property
    def n_out(self):
        return self.out_pos.shape[0]

    @property
    def U(self):
        return self.out_pos.shape[1]

    def device(self):
        """Device copies of the maps (uploaded once)."""
        if not self._dev:
            from . import _dev

            self._dev.update(
                in_src=_dev.i64_to_device(self.in_src),
                pt_src=_dev.i64_to_device(self.pt_src),
                out_pos=_dev.i32_to_device(self.out_pos),
                out_dst=_dev.i64_to_device(self.out_dst),
            )
        return self._dev


def _cdiv(a, b):
    return -(-a // b)


def compact(dense_map: np.ndarray):
    """Dense [P, N] source map (-1 = zero) -> packed (pos, src) int32 [P, Z]:
    the form the device kernels consume (pencil_b200.h "packed source")."""
    dense_map = np.asarray(dense_map)
    P = dense_map.shape[0]
    nz = dense_map >= 0
    cnt = nz.sum(axis=1)
    Z = int(cnt.max()) if P else 0
    pos = np.full((P, max(Z, 1)), -1, dtype=np.int32)
    src = np.zeros((P, max(Z, 1)), dtype=np.int32)
    rows, cols = np.nonzero(nz)
    slot = np.arange(len(rows)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    pos[rows, slot] = cols
    src[rows, slot] = dense_map[rows, cols]
    return pos, src


# Relative device cost of each plan component, measured on B200 at N=8192,
# L=7 (profiles/r01_kernel_latency_small_grids.jsonl, FC-784 forward launch):
# encrypting an input poly 0.40 us, encoding a plaintext 0.19 us, producing +
# decrypting an output ciphertext (mask NTT + INTT + decode) 0.67 us, one
# ct x pt product term 0.049 us (TMA-pipelined MAC).
COST_ENC, COST_PT, COST_OUT, COST_PROD = 8.0, 3.7, 14.0, 1.0
MAX_INPUT_BLOCKS = 32  # bounds the homomorphic accumulation depth (noise)


def matmul_blocks(g: MatmulGeometry, N: int, mode: str = "cost"):
    """(B_blk, n_o_blk, n_i_blk) with n_o_blk * n_i_blk * B_blk <= N.

    mode "spec": SPEC:285 order -- shrink the batch block first, then the
    output dimension, then the input dimension.
    mode "cost": the tiling minimising the engine's cost model above (the
    partition strategy is not fixed by the paper); ties broken
    deterministically.  Decrypted outputs do not depend on the tiling."""
    if min(g.n_i, g.n_o, g.B) < 1:
        raise GeometryError("empty matmul geometry")
    if mode == "spec":
        nib = min(g.n_i, N)
        if g.n_o * nib <= N:
            return min(g.B, N // (g.n_o * nib)), g.n_o, nib
        return 1, max(1, N // nib), nib
    best = None
    for k in range(1, MAX_INPUT_BLOCKS + 1):
        nib = _cdiv(g.n_i, k)
        if nib > N or _cdiv(g.n_i, nib) != k:
            continue
        cap = N // nib
        for nob in range(1, min(g.n_o, cap) + 1):
            Bb = min(g.B, cap // nob)
            nO, nB = _cdiv(g.n_o, nob), _cdiv(g.B, Bb)
            n_out = nB * nO
            cost = COST_ENC * nB * k + COST_PT * nO * k + COST_OUT * n_out + COST_PROD * n_out * k
            key = (round(cost, 6), n_out, k, -nob)
            if best is None or key < best[0]:
                best = (key, (Bb, nob, nib))
        if k >= g.n_i:
            break
    return best[1]


def conv_blocks(g: ConvGeometry, N: int, mode: str = "cost"):
    """(B_blk, c_o_blk, c_i_blk) with B_blk * c_o_blk * c_i_blk * h * w <= N.
    mode "spec": SPEC:285 order; mode "cost": minimise the cost model above."""
    hw = g.h * g.w
    if g.s < 1 or g.s > min(g.h, g.w):
        raise GeometryError("kernel must fit the image")
    if hw > N:
        raise GeometryError(f"h*w = {hw} exceeds N = {N}")
    if mode == "spec":
        cib = min(g.c_i, N // hw)
        if g.c_o * cib * hw <= N:
            return min(g.B, N // (g.c_o * cib * hw)), g.c_o, cib
        return 1, max(1, N // (cib * hw)), cib
    cap = N // hw
    best = None
    for cib in range(1, min(g.c_i, cap) + 1):
        nI = _cdiv(g.c_i, cib)
        if _cdiv(g.c_i, _cdiv(g.c_i, nI)) != nI or _cdiv(g.c_i, nI) != cib:
            continue  # only balanced splits
        for cob in range(1, min(g.c_o, cap // cib) + 1):
            Bb = min(g.B, cap // (cib * cob))
            nB, nO = _cdiv(g.B, Bb), _cdiv(g.c_o, cob)
            n_out = nB * nO
            cost = COST_ENC * nB * nI + COST_PT * nO * nI + COST_OUT * n_out + COST_PROD * n_out * nI
            key = (round(cost, 6), n_out, nI, -cob)
            if best is None or key < best[0]:
                best = (key, (Bb, cob, cib))
    return best[1]


def _scatter(n_poly, N, poly_idx, pos, src, ok):
    out = np.full((n_poly, N), -1, dtype=np.int64)
    out[poly_idx[ok], pos[ok]] = src[ok]
    return out


def _terms(nB, nO, nI):
    bb, oo, ii = np.meshgrid(np.arange(nB), np.arange(nO), np.arange(nI), indexing="ij")
    t = np.stack([bb * nI + ii, oo * nI + ii], axis=-1)  # [nB, nO, nI, 2]
    return t.reshape(nB * nO, nI, 2).astype(np.int64)


@lru_cache(maxsize=256)
def plan_matmul(g: MatmulGeometry, N: int, v_strides=None, w_strides=None, y_strides=None,
                mode: str = "cost") -> BlockPlan:
    """v is (n_i, B), W is (n_o, n_i), Y is (n_o, B); strides default to row-major."""
    vs = v_strides or (g.B, 1)
    ws = w_strides or (g.n_i, 1)
    ys = y_strides or (g.B, 1)
    Bb, nob, nib = matmul_blocks(g, N, mode)
    nB, nO, nI = _cdiv(g.B, Bb), _cdiv(g.n_o, nob), _cdiv(g.n_i, nib)
    # inputs: axes (bb, ii, k, j)
    bb = np.arange(nB)[:, None, None, None]
    ii = np.arange(nI)[None, :, None, None]
    k = np.arange(Bb)[None, None, :, None]
    j = np.arange(nib)[None, None, None, :]
    gj, gk = ii * nib + j, bb * Bb + k
    shape = (nB, nI, Bb, nib)
    ok = np.broadcast_to((gj < g.n_i) & (gk < g.B), shape).ravel()
    in_src = _scatter(nB * nI, N, np.broadcast_to(bb * nI + ii, shape).ravel(),
                      np.broadcast_to(k * nob * nib + j, shape).ravel(),
                      np.broadcast_to(gj * vs[0] + gk * vs[1], shape).ravel(), ok)
    # weights: axes (oo, ii, i, j)
    oo = np.arange(nO)[:, None, None, None]
    i = np.arange(nob)[None, None, :, None]
    gi = oo * nob + i
    shape = (nO, nI, nob, nib)
    ok = np.broadcast_to((gi < g.n_o) & (gj.reshape(1, nI, 1, nib) < g.n_i), shape).ravel()
    gjw = (ii * nib + j).reshape(1, nI, 1, nib)
    pt_src = _scatter(nO * nI, N, np.broadcast_to(oo * nI + ii, shape).ravel(),
                      np.broadcast_to(i * nib + nib - 1 - j, shape).ravel(),
                      np.broadcast_to(gi * ws[0] + gjw * ws[1], shape).ravel(), ok)
    # outputs: axes (bb, oo, i, k) -> slot u = i*Bb + k
    bb = np.arange(nB)[:, None, None, None]
    oo = np.arange(nO)[None, :, None, None]
    i = np.arange(nob)[None, None, :, None]
    k = np.arange(Bb)[None, None, None, :]
    gi, gk = oo * nob + i, bb * Bb + k
    shape = (nB, nO, nob, Bb)
    ok = np.broadcast_to((gi < g.n_o) & (gk < g.B), shape)
    pos = np.broadcast_to(k * nob * nib + i * nib + nib - 1, shape)
    dst = np.broadcast_to(gi * ys[0] + gk * ys[1], shape)
    out_pos = np.where(ok, pos, -1).reshape(nB * nO, nob * Bb).astype(np.int64)
    out_dst = np.where(ok, dst, -1).reshape(nB * nO, nob * Bb).astype(np.int64)
    return BlockPlan("matmul", g, N, (Bb, nob, nib), (nB, nO, nI), in_src, pt_src, out_pos, out_dst,
                     _terms(nB, nO, nI))


@lru_cache(maxsize=256)
def plan_conv(g: ConvGeometry, N: int, mode: str = "spec") -> BlockPlan:
    """v is (B, c_i, h, w), W is (c_o, c_i, s, s), y is (B, c_o, h-s+1, w-s+1)."""
    Bb, cob, cib = conv_blocks(g, N, mode)
    nB, nO, nI = _cdiv(g.B, Bb), _cdiv(g.c_o, cob), _cdiv(g.c_i, cib)
    h, w, s = g.h, g.w, g.s
    hw = h * w
    oh, ow = h - s + 1, w - s + 1
    O = (cib - 1) * hw + (s - 1) * w + s - 1
    bb = np.arange(nB).reshape(-1, 1, 1, 1, 1, 1)
    ii = np.arange(nI).reshape(1, -1, 1, 1, 1, 1)
    b = np.arange(Bb).reshape(1, 1, -1, 1, 1, 1)
    c = np.arange(cib).reshape(1, 1, 1, -1, 1, 1)
    y = np.arange(h).reshape(1, 1, 1, 1, -1, 1)
    x = np.arange(w).reshape(1, 1, 1, 1, 1, -1)
    shape = (nB, nI, Bb, cib, h, w)
    gb, gc = bb * Bb + b, ii * cib + c
    ok = np.broadcast_to((gb < g.B) & (gc < g.c_i), shape).ravel()
    in_src = _scatter(nB * nI, N, np.broadcast_to(bb * nI + ii, shape).ravel(),
                      np.broadcast_to(b * cob * cib * hw + c * hw + y * w + x, shape).ravel(),
                      np.broadcast_to(((gb * g.c_i + gc) * h + y) * w + x, shape).ravel(), ok)
    oo = np.arange(nO).reshape(-1, 1, 1, 1, 1, 1)
    co = np.arange(cob).reshape(1, 1, -1, 1, 1, 1)
    di = np.arange(s).reshape(1, 1, 1, 1, -1, 1)
    dj = np.arange(s).reshape(1, 1, 1, 1, 1, -1)
    shape = (nO, nI, cob, cib, s, s)
    gco = oo * cob + co
    ok = np.broadcast_to((gco < g.c_o) & (gc.reshape(1, nI, 1, cib, 1, 1) < g.c_i), shape).ravel()
    gcw = (ii * cib + c).reshape(1, nI, 1, cib, 1, 1)
    pt_src = _scatter(nO * nI, N, np.broadcast_to(oo * nI + ii, shape).ravel(),
                      np.broadcast_to(O + co * cib * hw - c.reshape(1, 1, 1, cib, 1, 1) * hw - di * w - dj, shape).ravel(),
                      np.broadcast_to(((gco * g.c_i + gcw) * s + di) * s + dj, shape).ravel(), ok)
    bb = np.arange(nB).reshape(-1, 1, 1, 1, 1, 1)
    oo = np.arange(nO).reshape(1, -1, 1, 1, 1, 1)
    b = np.arange(Bb).reshape(1, 1, -1, 1, 1, 1)
    co = np.arange(cob).reshape(1, 1, 1, -1, 1, 1)
    y = np.arange(oh).reshape(1, 1, 1, 1, -1, 1)
    x = np.arange(ow).reshape(1, 1, 1, 1, 1, -1)
    shape = (nB, nO, Bb, cob, oh, ow)
    gb, gco = bb * Bb + b, oo * cob + co
    ok = np.broadcast_to((gb < g.B) & (gco < g.c_o), shape)
    pos = np.broadcast_to(b * cob * cib * hw + O + co * cib * hw + y * w + x, shape)
    dst = np.broadcast_to(((gb * g.c_o + gco) * oh + y) * ow + x, shape)
    U = Bb * cob * oh * ow
    out_pos = np.where(ok, pos, -1).reshape(nB * nO, U).astype(np.int64)
    out_dst = np.where(ok, dst, -1).reshape(nB * nO, U).astype(np.int64)
    return BlockPlan("conv", g, N, (Bb, cob, cib), (nB, nO, nI), in_src, pt_src, out_pos, out_dst,
                     _terms(nB, nO, nI))


def plan_blocks(g, N: int, mode: str = "cost") -> BlockPlan:
    if isinstance(g, MatmulGeometry):
        return plan_matmul(g, N, mode=mode)
    if isinstance(g, ConvGeometry):
        return plan_conv(g, N)
    raise GeometryError(f"unknown geometry {g!r}")


# ------------------------------------------- conv layers (pad / stride) ---
# SPEC:284 keeps the codec at valid-mode stride-1 cross-correlation with
# padding / stride "outside the codec", and SPEC:286 lowers the backward
# operators by local share reshaping.  Each such reshaping (zero padding,
# stride subsampling, zero-stuffing dilation, kernel flip, channel / batch
# transposition) is a data-movement-only linear map, so it is folded into the
# plan's index maps: a plan of the logical geometry (the verified codec) has
# its source / destination indices re-pointed into the physical tensors
# (-1 = structural zero / dropped output).  Forward, input-gradient and
# weight-gradient operators all use the paper's native conv packing
# (PAPER:1226-1247); nothing is materialised.


def conv_out_hw(H, W, s, pad, stride):
    return (H + 2 * pad - s) // stride + 1, (W + 2 * pad - s) // stride + 1


def _compact_out(pos, dst):
    """Move each row's useful (pos, dst) pairs to the front; U = max count."""
    ok = dst >= 0
    cnt = ok.sum(axis=1)
    U = max(1, int(cnt.max()) if len(cnt) else 1)
    P = pos.shape[0]
    npos = np.full((P, U), -1, dtype=np.int64)
    ndst = np.full((P, U), -1, dtype=np.int64)
    rows, cols = np.nonzero(ok)
    slot = np.arange(len(rows)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    npos[rows, slot] = pos[rows, cols]
    ndst[rows, slot] = dst[rows, cols]
    return npos, ndst


def remap(plan: BlockPlan, in_map, pt_map, out_map) -> BlockPlan:
    def re(src, m):
        out = np.full(src.shape, -1, dtype=np.int64)
        ok = src >= 0
        out[ok] = m[src[ok]]
        return out

    dst = re(plan.out_dst, out_map)
    pos, dst = _compact_out(np.where(dst >= 0, plan.out_pos, -1), dst)
    return BlockPlan(plan.kind, plan.geometry, plan.N, plan.blk, plan.nblk, re(plan.in_src, in_map),
                     re(plan.pt_src, pt_map), pos, dst, plan.terms)


def conv_index_maps(kind: str, B, c_i, c_o, H, W, s, pad, stride):
    """(logical ConvGeometry, in_map, pt_map, out_map) of one conv-layer operator:

    fwd   Y[b,o,y,x]  = sum W[o,c,i,j] Xpad[b,c,y*st+i,x*st+j]          v=X,  W=W,  y=Y
    bwdx  dX[b,c,y,x] = sum W[o,c,i,j] dY[b,o,(y+p-i)/st,(x+p-j)/st]    v=dY, W=W,  y=dX
          (correlation of the dilated, (s-1)-padded dY with the flipped, transposed W)
    gradw dW[o,c,i,j] = sum dY[b,o,y,x] Xpad[b,c,y*st+i,x*st+j]         v=X,  W=dY, y=dW
          (correlation of Xpad^T (channels as batch) with the dilated dY^T as kernel)
    """
    oh, ow = conv_out_hw(H, W, s, pad, stride)
    hp, wp = H + 2 * pad, W + 2 * pad

    def pad_map(C, Bn, transpose=False):  # logical (Bn, C, hp, wp) -> X (B, c_i, H, W) index
        b, c, y, x = np.meshgrid(np.arange(Bn), np.arange(C), np.arange(hp), np.arange(wp), indexing="ij")
        yy, xx = y - pad, x - pad
        ok = (yy >= 0) & (yy < H) & (xx >= 0) & (xx < W)
        bb, cc = (c, b) if transpose else (b, c)
        return np.where(ok, ((bb * c_i + cc) * H + yy) * W + xx, -1).ravel()

    if kind == "fwd":
        g = ConvGeometry(B, c_i, c_o, hp, wp, s)
        b, o, y, x = np.meshgrid(np.arange(B), np.arange(c_o), np.arange(hp - s + 1), np.arange(wp - s + 1),
                                 indexing="ij")
        ok = (y % stride == 0) & (x % stride == 0) & (y // stride < oh) & (x // stride < ow)
        out_map = np.where(ok, ((b * c_o + o) * oh + y // stride) * ow + x // stride, -1).ravel()
        return g, pad_map(c_i, B), np.arange(c_o * c_i * s * s), out_map
    if kind == "bwdx":
        hd, wd = (oh - 1) * stride + 1 + 2 * (s - 1), (ow - 1) * stride + 1 + 2 * (s - 1)
        g = ConvGeometry(B, c_o, c_i, hd, wd, s)
        b, o, y, x = np.meshgrid(np.arange(B), np.arange(c_o), np.arange(hd), np.arange(wd), indexing="ij")
        u, v = y - (s - 1), x - (s - 1)
        ok = (u >= 0) & (v >= 0) & (u % stride == 0) & (v % stride == 0) & (u // stride < oh) & (v // stride < ow)
        in_map = np.where(ok, ((b * c_o + o) * oh + u // stride) * ow + v // stride, -1).ravel()
        c, o2, i, j = np.meshgrid(np.arange(c_i), np.arange(c_o), np.arange(s), np.arange(s), indexing="ij")
        pt_map = (((o2 * c_i + c) * s + (s - 1 - i)) * s + (s - 1 - j)).ravel()
        b, c, y, x = np.meshgrid(np.arange(B), np.arange(c_i), np.arange(hd - s + 1), np.arange(wd - s + 1),
                                 indexing="ij")
        yy, xx = y - pad, x - pad
        ok = (yy >= 0) & (yy < H) & (xx >= 0) & (xx < W)
        return g, in_map, pt_map, np.where(ok, ((b * c_i + c) * H + yy) * W + xx, -1).ravel()
    if kind == "gradw":
        sd_h, sd_w = (oh - 1) * stride + 1, (ow - 1) * stride + 1
        if sd_h != sd_w:
            raise GeometryError("gradw lowering needs a square output")
        g = ConvGeometry(c_i, B, c_o, hp, wp, sd_h)
        o, b, i, j = np.meshgrid(np.arange(c_o), np.arange(B), np.arange(sd_h), np.arange(sd_w), indexing="ij")
        ok = (i % stride == 0) & (j % stride == 0)
        pt_map = np.where(ok, ((b * c_o + o) * oh + i // stride) * ow + j // stride, -1).ravel()
        c, o, y, x = np.meshgrid(np.arange(c_i), np.arange(c_o), np.arange(hp - sd_h + 1), np.arange(wp - sd_w + 1),
                                 indexing="ij")
        ok = (y < s) & (x < s)
        return g, pad_map(B, c_i, transpose=True), pt_map, np.where(ok, ((o * c_i + c) * s + y) * s + x, -1).ravel()
    raise GeometryError(f"unknown conv operator {kind!r}")


@lru_cache(maxsize=128)
def plan_conv_layer(kind: str, B, c_i, c_o, H, W, s, pad, stride, N, mode: str = "cost") -> BlockPlan:
    """Block plan of one conv-layer operator (kind fwd / bwdx / gradw) over the
    physical tensors; its maps feed the same fused kernels as matmul plans."""
    g, in_map, pt_map, out_map = conv_index_maps(kind, B, c_i, c_o, H, W, s, pad, stride)
    return remap(plan_conv(g, N, mode), in_map, pt_map, out_map)


# --------------------------------------------- plaintext codecs (host) ---

def matmul_poly_encode(which: str, tensor, g: MatmulGeometry, N: int):
    """Single-block encode (the SPEC operation); raises GeometryError on overflow."""
    if g.n_o * g.n_i * g.B > N:
        raise GeometryError("n_o * n_i * B must not exceed N")
    plan = plan_matmul(g, N, mode="spec")
    src = plan.in_src if which == "input" else plan.pt_src
    vals = np.asarray(tensor, dtype=np.uint64).ravel()
    out = np.zeros(N, dtype=np.uint64)
    ok = src[0] >= 0
    out[ok] = vals[src[0][ok]]
    return out


def matmul_poly_decode(y, g: MatmulGeometry, N: int):
    plan = plan_matmul(g, N, mode="spec")
    y = np.asarray(y, dtype=np.uint64)
    out = np.zeros(g.n_o * g.B, dtype=np.uint64)
    ok = plan.out_pos[0] >= 0
    out[plan.out_dst[0][ok]] = y[plan.out_pos[0][ok]]
    return out.reshape(g.n_o, g.B)


def conv_poly_encode(which: str, tensor, g: ConvGeometry, N: int):
    if g.B * g.c_o * g.c_i * g.h * g.w > N:
        raise GeometryError("B * c_o * c_i * h * w must not exceed N")
    plan = plan_conv(g, N)
    src = plan.in_src if which == "input" else plan.pt_src
    vals = np.asarray(tensor, dtype=np.uint64).ravel()
    out = np.zeros(N, dtype=np.uint64)
    ok = src[0] >= 0
    out[ok] = vals[src[0][ok]]
    return out


def conv_poly_decode(y, g: ConvGeometry, N: int):
    plan = plan_conv(g, N)
    y = np.asarray(y, dtype=np.uint64)
    oh, ow = g.h - g.s + 1, g.w - g.s + 1
    out = np.zeros(g.B * g.c_o * oh * ow, dtype=np.uint64)
    ok = plan.out_pos[0] >= 0
    out[plan.out_dst[0][ok]] = y[plan.out_pos[0][ok]]
    return out.reshape(g.B, g.c_o, oh, ow)
