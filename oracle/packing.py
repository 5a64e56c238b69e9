"""ORACLE — TEST INFRASTRUCTURE ONLY.

Restatement of the SPEC-only ``poly_encoding`` module (SPEC.md:212-295,
PAPER.md Appendix A): the coefficient packings pi_v, pi_W,
pi_y for batched matmul and batched 2D convolution, and the block plan.

Packing formulas:
  matmul  input  x^(k*n_o*n_i + j)          <- v[j, k]
          weight x^(i*n_i + n_i - 1 - j)    <- W[i, j]
          output y[i, k] at k*n_o*n_i + i*n_i + n_i - 1
  conv    index_v(b,c,i,j)  = b*c_o*c_i*h*w + c*h*w + i*w + j
          index_W(c',c,i,j) = O + c'*c_i*h*w - c*h*w - i*w - j,  i,j in [s]
          index_y(b,c',i,j) = b*c_o*c_i*h*w + O + c'*c_i*h*w + i*w + j
          O = (c_i - 1)*h*w + (s - 1)*w + s - 1
Block plan: split batch first, then the output
dimension, then the input dimension; input-dimension partials accumulate
homomorphically.  Every block uses the nominal block dimensions in its
exponents (partial edge blocks leave positions empty), so all blocks share
one index template.

A plan is described by dense/compact int64 index maps that both the oracle
and the device engine consume:
  in_src [n_in, N]   flat source element of the encrypted operand or -1
  pt_src [n_pt, N]   flat source element of the plaintext operand or -1
  out_pos/out_dst [n_out, U]  useful coefficient positions and the flat
                     output element they decode to (-1 padded)
  terms [n_out, K, 2] (input-ct index, plaintext index) pairs summed per output
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class GeometryError(Exception):
    pass


@dataclass(frozen=True)
class MatmulGeometry:
    n_i: int
    n_o: int
    B: int


@dataclass(frozen=True)
class ConvGeometry:  # SPEC:221-224 (valid mode, stride 1)
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
    blk: tuple  # matmul: (B_blk, n_o_blk, n_i_blk); conv: (B_blk, c_o_blk, c_i_blk)
    nblk: tuple  # number of blocks per dimension, same order
    in_src: np.ndarray
    pt_src: np.ndarray
    out_pos: np.ndarray
    out_dst: np.ndarray
    terms: np.ndarray

    @property
    def n_in(self):
        return self.in_src.shape[0]

    @property
    def n_pt(self):
        return self.pt_src.shape[0]

    @property
    def n_out(self):
        return self.out_pos.shape[0]


def _cdiv(a, b):
    return -(-a // b)


def plan_matmul_blocks(g: MatmulGeometry, N: int, mode: str = "cost"):
    """mode "spec": SPEC:285 order, shrink the batch block first, then n_o,
    then n_i.  mode "cost": minimise the weighted count of encryptions (1.3),
    plaintext encodings (1.0), output ciphertexts (2.0: mask NTT + INTT) and
    ct x pt terms (0.5) over input splits k <= 32 (the paper leaves the
    partition strategy open; the block tiling does not change any
    decrypted value)."""
    if min(g.n_i, g.n_o, g.B) < 1:
        raise GeometryError("empty matmul geometry")
    if mode == "spec":
        n_i_blk = min(g.n_i, N)
        if g.n_o * n_i_blk <= N:
            return min(g.B, N // (g.n_o * n_i_blk)), g.n_o, n_i_blk
        return 1, max(1, N // n_i_blk), n_i_blk
    best = None
    k = 0
    while k < min(32, g.n_i):
        k += 1
        nib = -(-g.n_i // k)
        if nib > N or -(-g.n_i // nib) != k:
            continue
        cap = N // nib
        for nob in range(1, min(g.n_o, cap) + 1):
            Bb = min(g.B, cap // nob)
            n_out = (-(-g.B // Bb)) * (-(-g.n_o // nob))
            cost = 8.0 * (-(-g.B // Bb)) * k + 3.7 * (-(-g.n_o // nob)) * k + 14.0 * n_out + 1.0 * n_out * k
            cand = ((round(cost, 6), n_out, k, -nob), (Bb, nob, nib))
            best = cand if best is None or cand[0] < best[0] else best
    return best[1]


def plan_blocks(g, N: int, mode: str = "cost") -> BlockPlan:
    if isinstance(g, MatmulGeometry):
        return _plan_matmul(g, N, mode)
    if isinstance(g, ConvGeometry):
        return _plan_conv(g, N)
    raise GeometryError(f"unknown geometry {g!r}")


def _plan_matmul(g: MatmulGeometry, N: int, mode: str = "cost") -> BlockPlan:
    Bb, nob, nib = plan_matmul_blocks(g, N, mode)
    nB, nO, nI = _cdiv(g.B, Bb), _cdiv(g.n_o, nob), _cdiv(g.n_i, nib)
    # input template: (k, j) -> k*nob*nib + j
    k = np.arange(Bb)[:, None]
    j = np.arange(nib)[None, :]
    in_pos_t = (k * nob * nib + j).ravel()
    in_src = np.full((nB * nI, N), -1, dtype=np.int64)
    for bb in range(nB):
        for ii in range(nI):
            gj = ii * nib + j
            gk = bb * Bb + k
            ok = ((gj < g.n_i) & (gk < g.B)).ravel()
            src = (gj * g.B + gk).ravel()  # v is (n_i, B) row-major
            in_src[bb * nI + ii, in_pos_t[ok]] = src[ok]
    # weight template: (i, j) -> i*nib + nib - 1 - j
    i = np.arange(nob)[:, None]
    w_pos_t = (i * nib + nib - 1 - j).ravel()
    pt_src = np.full((nO * nI, N), -1, dtype=np.int64)
    for oo in range(nO):
        for ii in range(nI):
            gi = oo * nob + i
            gj = ii * nib + j
            ok = ((gi < g.n_o) & (gj < g.n_i)).ravel()
            src = (gi * g.n_i + gj).ravel()  # W is (n_o, n_i)
            pt_src[oo * nI + ii, w_pos_t[ok]] = src[ok]
    # output template: (i, k) -> k*nob*nib + i*nib + nib - 1
    U = nob * Bb
    kk = np.arange(Bb)[None, :]
    out_pos_t = (kk * nob * nib + i * nib + nib - 1).ravel()  # order (i, k)
    out_pos = np.full((nB * nO, U), -1, dtype=np.int64)
    out_dst = np.full((nB * nO, U), -1, dtype=np.int64)
    terms = np.zeros((nB * nO, nI, 2), dtype=np.int64)
    for bb in range(nB):
        for oo in range(nO):
            r = bb * nO + oo
            gi = oo * nob + i
            gk = bb * Bb + kk
            ok = ((gi < g.n_o) & (gk < g.B)).ravel()
            dst = (gi * g.B + gk).ravel()  # Y is (n_o, B)
            out_pos[r, ok] = out_pos_t[ok]
            out_dst[r, ok] = dst[ok]
            for ii in range(nI):
                terms[r, ii] = (bb * nI + ii, oo * nI + ii)
    return BlockPlan("matmul", g, N, (Bb, nob, nib), (nB, nO, nI), in_src, pt_src, out_pos, out_dst, terms)


def plan_conv_blocks(g: ConvGeometry, N: int):
    hw = g.h * g.w
    if g.s > min(g.h, g.w):
        raise GeometryError("kernel larger than image")
    if hw > N:
        raise GeometryError(f"h*w={hw} exceeds N={N}; spatial tiling is not supported")
    c_i_blk = min(g.c_i, N // hw)
    if g.c_o * c_i_blk * hw <= N:
        c_o_blk = g.c_o
        B_blk = min(g.B, N // (g.c_o * c_i_blk * hw))
    else:
        B_blk = 1
        c_o_blk = max(1, N // (c_i_blk * hw))
    return B_blk, c_o_blk, c_i_blk


def _plan_conv(g: ConvGeometry, N: int) -> BlockPlan:
    Bb, cob, cib = plan_conv_blocks(g, N)
    nB, nO, nI = _cdiv(g.B, Bb), _cdiv(g.c_o, cob), _cdiv(g.c_i, cib)
    h, w, s = g.h, g.w, g.s
    hw = h * w
    oh, ow = h - s + 1, w - s + 1
    O = (cib - 1) * hw + (s - 1) * w + s - 1
    b = np.arange(Bb)[:, None, None, None]
    c = np.arange(cib)[None, :, None, None]
    yi = np.arange(h)[None, None, :, None]
    xj = np.arange(w)[None, None, None, :]
    in_pos_t = (b * cob * cib * hw + c * hw + yi * w + xj).ravel()
    in_src = np.full((nB * nI, N), -1, dtype=np.int64)
    for bb in range(nB):
        for ii in range(nI):
            gb = bb * Bb + b
            gc = ii * cib + c
            ok = np.broadcast_to((gb < g.B) & (gc < g.c_i), (Bb, cib, h, w)).ravel()
            src = (((gb * g.c_i + gc) * h + yi) * w + xj).ravel()  # v is (B, c_i, h, w)
            in_src[bb * nI + ii, in_pos_t[ok]] = src[ok]
    co = np.arange(cob)[:, None, None, None]
    di = np.arange(s)[None, None, :, None]
    dj = np.arange(s)[None, None, None, :]
    w_pos_t = (O + co * cib * hw - c * hw - di * w - dj).ravel()
    pt_src = np.full((nO * nI, N), -1, dtype=np.int64)
    for oo in range(nO):
        for ii in range(nI):
            gco = oo * cob + co
            gc = ii * cib + c
            ok = np.broadcast_to((gco < g.c_o) & (gc < g.c_i), (cob, cib, s, s)).ravel()
            src = (((gco * g.c_i + gc) * s + di) * s + dj).ravel()  # W is (c_o, c_i, s, s)
            pt_src[oo * nI + ii, w_pos_t[ok]] = src[ok]
    oi = np.arange(oh)[None, None, :, None]
    oj = np.arange(ow)[None, None, None, :]
    bo = np.arange(Bb)[:, None, None, None]
    coo = np.arange(cob)[None, :, None, None]
    out_pos_t = (bo * cob * cib * hw + O + coo * cib * hw + oi * w + oj).ravel()  # order (b, c', i, j)
    U = Bb * cob * oh * ow
    out_pos = np.full((nB * nO, U), -1, dtype=np.int64)
    out_dst = np.full((nB * nO, U), -1, dtype=np.int64)
    terms = np.zeros((nB * nO, nI, 2), dtype=np.int64)
    for bb in range(nB):
        for oo in range(nO):
            r = bb * nO + oo
            gb = bb * Bb + bo
            gco = oo * cob + coo
            ok = np.broadcast_to((gb < g.B) & (gco < g.c_o), (Bb, cob, oh, ow)).ravel()
            dst = (((gb * g.c_o + gco) * oh + oi) * ow + oj).ravel()  # y is (B, c_o, oh, ow)
            out_pos[r, ok] = out_pos_t[ok]
            out_dst[r, ok] = dst[ok]
            for ii in range(nI):
                terms[r, ii] = (bb * nI + ii, oo * nI + ii)
    return BlockPlan("conv", g, N, (Bb, cob, cib), (nB, nO, nI), in_src, pt_src, out_pos, out_dst, terms)


# ------------------------------------------------------ plaintext codecs ---

def pack(src_map, values, N=None):
    """Scatter flat ``values`` into polynomials per a [P, N] source map."""
    values = np.asarray(values, dtype=np.uint64).ravel()
    out = np.zeros(src_map.shape, dtype=np.uint64)
    ok = src_map >= 0
    out[ok] = values[src_map[ok]]
    return out


def unpack(polys, plan: BlockPlan, out_size: int):
    """Gather useful coefficients of output polys into a flat tensor."""
    out = np.zeros(out_size, dtype=np.uint64)
    ok = plan.out_pos >= 0
    rows = np.nonzero(ok)[0]
    out[plan.out_dst[ok]] = polys[rows, plan.out_pos[ok]]
    return out


# ------------------------------------------- conv layers (pad / stride) ---
#
# SPEC:284 keeps the codec at valid-mode stride-1 cross-correlation and puts
# padding / stride "outside the codec"; SPEC:286 lowers the backward
# operators by local share reshaping.  Here every such reshaping (zero
# padding, stride subsampling, zero-stuffing dilation, kernel flip,
# channel/batch transposition) is a data-movement-only linear map, folded
# into the plan's index maps: a logical-geometry plan is built with the
# verified codec and its source / destination indices are re-pointed into
# the physical tensors (-1 = structural zero / dropped output).  The three
# layer operators (forward, input gradient, weight gradient) all use the
# paper's native conv packing.

def remap(plan: BlockPlan, in_map, pt_map, out_map) -> BlockPlan:
    def re(src, m):
        out = np.full(src.shape, -1, dtype=np.int64)
        ok = src >= 0
        out[ok] = m[src[ok]]
        return out

    dst = re(plan.out_dst, out_map)
    pos = np.where(dst >= 0, plan.out_pos, -1)
    return BlockPlan(plan.kind, plan.geometry, plan.N, plan.blk, plan.nblk, re(plan.in_src, in_map),
                     re(plan.pt_src, pt_map), pos, dst, plan.terms)


def conv_out_hw(H, W, s, pad, stride):
    return (H + 2 * pad - s) // stride + 1, (W + 2 * pad - s) // stride + 1


def conv_index_maps(kind: str, B, c_i, c_o, H, W, s, pad, stride):
    """(logical ConvGeometry, in_map, pt_map, out_map) of one conv-layer operator.

    fwd   Y[b,o,y,x]   = sum W[o,c,i,j] Xpad[b,c,y*st+i,x*st+j]      v=X,  W=W,  y=Y
    bwdx  dX[b,c,y,x]  = sum W[o,c,i,j] dY[b,o,(y+p-i)/st,(x+p-j)/st]  v=dY, W=W,  y=dX
    gradw dW[o,c,i,j]  = sum dY[b,o,y,x] Xpad[b,c,y*st+i,x*st+j]       v=X,  W=dY, y=dW
    """
    oh, ow = conv_out_hw(H, W, s, pad, stride)
    hp, wp = H + 2 * pad, W + 2 * pad

    def pad_map(C, Bn, transpose=False):  # logical (Bn, C, hp, wp) of Xpad -> X (B, c_i, H, W) index
        b, c, y, x = np.meshgrid(np.arange(Bn), np.arange(C), np.arange(hp), np.arange(wp), indexing="ij")
        yy, xx = y - pad, x - pad
        ok = (yy >= 0) & (yy < H) & (xx >= 0) & (xx < W)
        bb, cc = (c, b) if transpose else (b, c)  # transpose: logical batch = channel
        src = ((bb * c_i + cc) * H + yy) * W + xx
        return np.where(ok, src, -1).ravel()

    if kind == "fwd":
        g = ConvGeometry(B, c_i, c_o, hp, wp, s)
        in_map = pad_map(c_i, B)
        pt_map = np.arange(c_o * c_i * s * s)
        b, o, y, x = np.meshgrid(np.arange(B), np.arange(c_o), np.arange(hp - s + 1), np.arange(wp - s + 1),
                                 indexing="ij")
        ok = (y % stride == 0) & (x % stride == 0) & (y // stride < oh) & (x // stride < ow)
        out_map = np.where(ok, ((b * c_o + o) * oh + y // stride) * ow + x // stride, -1).ravel()
        return g, in_map, pt_map, out_map
    if kind == "bwdx":
        hd, wd = (oh - 1) * stride + 1 + 2 * (s - 1), (ow - 1) * stride + 1 + 2 * (s - 1)
        g = ConvGeometry(B, c_o, c_i, hd, wd, s)
        b, o, y, x = np.meshgrid(np.arange(B), np.arange(c_o), np.arange(hd), np.arange(wd), indexing="ij")
        u, v = y - (s - 1), x - (s - 1)
        ok = (u >= 0) & (v >= 0) & (u % stride == 0) & (v % stride == 0) & (u // stride < oh) & (v // stride < ow)
        in_map = np.where(ok, ((b * c_o + o) * oh + u // stride) * ow + v // stride, -1).ravel()
        c, o2, i, j = np.meshgrid(np.arange(c_i), np.arange(c_o), np.arange(s), np.arange(s), indexing="ij")
        pt_map = (((o2 * c_i + c) * s + (s - 1 - i)) * s + (s - 1 - j)).ravel()  # logical K[c,o,i,j]
        b, c, y, x = np.meshgrid(np.arange(B), np.arange(c_i), np.arange(hd - s + 1), np.arange(wd - s + 1),
                                 indexing="ij")
        yy, xx = y - pad, x - pad
        ok = (yy >= 0) & (yy < H) & (xx >= 0) & (xx < W)
        out_map = np.where(ok, ((b * c_i + c) * H + yy) * W + xx, -1).ravel()
        return g, in_map, pt_map, out_map
    if kind == "gradw":
        sd_h, sd_w = (oh - 1) * stride + 1, (ow - 1) * stride + 1
        if sd_h != sd_w:
            raise GeometryError("gradw lowering needs a square output")
        g = ConvGeometry(c_i, B, c_o, hp, wp, sd_h)
        in_map = pad_map(B, c_i, transpose=True)
        o, b, i, j = np.meshgrid(np.arange(c_o), np.arange(B), np.arange(sd_h), np.arange(sd_w), indexing="ij")
        ok = (i % stride == 0) & (j % stride == 0)
        pt_map = np.where(ok, ((b * c_o + o) * oh + i // stride) * ow + j // stride, -1).ravel()
        c, o, y, x = np.meshgrid(np.arange(c_i), np.arange(c_o), np.arange(hp - sd_h + 1), np.arange(wp - sd_w + 1),
                                 indexing="ij")
        ok = (y < s) & (x < s)
        out_map = np.where(ok, ((o * c_i + c) * s + y) * s + x, -1).ravel()
        return g, in_map, pt_map, out_map
    raise GeometryError(f"unknown conv operator {kind!r}")


def plan_conv_layer(kind: str, B, c_i, c_o, H, W, s, pad, stride, N) -> BlockPlan:
    g, in_map, pt_map, out_map = conv_index_maps(kind, B, c_i, c_o, H, W, s, pad, stride)
    return remap(_plan_conv(g, N), in_map, pt_map, out_map)
