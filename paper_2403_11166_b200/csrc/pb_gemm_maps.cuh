// pb_gemm_maps.cuh — index maps of the ring GEMM operators: the conv
// forward / input-gradient / weight-gradient local terms (K:260-278
// conv2d_wrap with the protocols' pad / stride / dilation lowerings,
// SPEC:284-286) and K:206-218 matmul_wrap as one generic
// out(n x m) = sum_k A(n, k) B(k, m), with A / B gathered on the fly.
#pragma once

#include "pb_common.cuh"

struct GemmMap {  // generic GEMM out(n x m) = sum_k A(n,k) B(k,m) with conv / matmul gathers
  int kind;        // 0..2 PB_CONV_*, 3 matmul
  int B, ci, co, H, W, s, p, st, oh, ow;  // conv
  int n, k, m, ta, tb;                    // matmul
};

__device__ __forceinline__ uint64_t gemm_a(const GemmMap& d, const uint64_t* A, int row, int kk) {
  const int SS = d.s * d.s;
  switch (d.kind) {
    case PB_CONV_FWD: return __ldg(A + (size_t)row * (d.ci * SS) + kk);  // W[o][(c,i,j)]
    case PB_CONV_BWDX: {                                                 // W[o][c][i][j], row = c, kk = (o,i,j)
      const int o = kk / SS, r = kk - o * SS;
      return __ldg(A + (size_t)(o * d.ci + row) * SS + r);
    }
    case PB_CONV_GRADW: {  // dY[b][o][y][x], row = o, kk = (b,y,x)
      const unsigned hw = (unsigned)(d.oh * d.ow), b = (unsigned)kk / hw, r = (unsigned)kk - b * hw;
      return __ldg(A + (size_t)(b * d.co + row) * hw + r);
    }
    default: return __ldg(A + (d.ta ? (size_t)kk * d.n + row : (size_t)row * d.k + kk));
  }
}

__device__ __forceinline__ uint64_t gemm_b(const GemmMap& d, const uint64_t* Bm, int kk, int col) {
  const int SS = d.s * d.s;
  switch (d.kind) {
    case PB_CONV_FWD:
    case PB_CONV_GRADW: {
      const int kc = d.kind == PB_CONV_FWD ? kk : col;             // (c,i,j)
      const unsigned kp = (unsigned)(d.kind == PB_CONV_FWD ? col : kk);  // (b,y,x)
      const int c = kc / SS, r = kc - c * SS, i = r / d.s, j = r - i * d.s;
      const unsigned hw = (unsigned)(d.oh * d.ow), ow = (unsigned)d.ow;
      const unsigned b = kp / hw, q = kp - b * hw, y = q / ow, x = q - y * ow;
      const int yy = (int)y * d.st + i - d.p, xx = (int)x * d.st + j - d.p;
      if (yy < 0 || yy >= d.H || xx < 0 || xx >= d.W) return 0ull;
      return __ldg(Bm + ((size_t)(b * d.ci + c) * d.H + yy) * d.W + xx);
    }
    case PB_CONV_BWDX: {  // kk = (o,i,j), col = (b,y,x) of dX
      const int o = kk / SS, r = kk - o * SS, i = r / d.s, j = r - i * d.s;
      const unsigned hw = (unsigned)(d.H * d.W), Wd = (unsigned)d.W;
      const unsigned b = (unsigned)col / hw, q = (unsigned)col - b * hw, y = q / Wd, x = q - y * Wd;
      const int u = (int)y + d.p - i, v = (int)x + d.p - j;
      if (u < 0 || v < 0) return 0ull;
      const unsigned yy = (unsigned)u / (unsigned)d.st, xx = (unsigned)v / (unsigned)d.st;
      if (yy * d.st != (unsigned)u || xx * d.st != (unsigned)v || yy >= (unsigned)d.oh || xx >= (unsigned)d.ow)
        return 0ull;
      return __ldg(Bm + ((size_t)(b * d.co + o) * d.oh + yy) * d.ow + xx);
    }
    default: return __ldg(Bm + (d.tb ? (size_t)col * d.k + kk : (size_t)kk * d.m + col));
  }
}

__device__ __forceinline__ size_t gemm_out(const GemmMap& d, int row, int col) {
  switch (d.kind) {
    case PB_CONV_FWD: {
      const unsigned hw = (unsigned)(d.oh * d.ow), b = (unsigned)col / hw, q = (unsigned)col - b * hw;
      return (size_t)(b * d.co + row) * hw + q;
    }
    case PB_CONV_BWDX: {
      const unsigned hw = (unsigned)(d.H * d.W), b = (unsigned)col / hw, q = (unsigned)col - b * hw;
      return (size_t)(b * d.ci + row) * hw + q;
    }
    case PB_CONV_GRADW: return (size_t)row * (d.ci * d.s * d.s) + col;
    default: return (size_t)row * d.m + col;
  }
}

// balanced base-256 digits of v (< 2^59 after masking): v = sum d_i 256^i
__device__ __forceinline__ void digits8(uint64_t v, int8_t (&d)[8]) {
  int carry = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int x = (int)((v >> (8 * i)) & 0xFFu) + carry;
    carry = x >= 128;
    d[i] = (int8_t)(x - (carry << 8));
  }
}

// Incremental conv gathers of one GEMM operand row (pb_tc.cu digit planes and
// fused producers, pb_conv.cu skinny kernel): side 0 = the output-row operand
// (gemm_a), side 1 = the output-column one (gemm_b); specialised on the
// kernel size S, the contraction index walked without per-element divisions.
template <int KIND, int S, int SIDE>
struct Gather {
  // per-thread state for row `row` starting at contraction index k: the kernel
  // / output indices and a pointer to the current (image, channel) plane, so
  // each element costs an add, two unsigned bound checks and a 32-bit offset
  int c, i, j, y, x, o;
  int y0, x0;             // FWD: y st - p, x st - p;  GRADW side 1: i - p + y st, j - p + x st (walking)
  const uint64_t* base;   // the current plane (side 1) / row (side 0)
  __device__ __forceinline__ void init(const GemmMap& d, const uint64_t* src, int row, int k) {
    constexpr int SS = S * S;
    base = src;
    if (KIND == PB_CONV_FWD) {
      if (SIDE == 0) { base = src + (size_t)row * (d.ci * SS) + k; return; }   // W[o][(c,i,j)]
      const int hw = d.oh * d.ow;                                              // X im2col: row = (b,y,x)
      const int b = row / hw, q = row - b * hw;
      y = q / d.ow; x = q - y * d.ow;
      c = k / SS; const int r = k - c * SS; i = r / S; j = r - i * S;
      y0 = y * d.st - d.p; x0 = x * d.st - d.p;
      base = src + (size_t)(b * d.ci + c) * d.H * d.W;
    } else if (KIND == PB_CONV_BWDX) {
      if (SIDE == 0) { o = k / SS; const int r = k - o * SS; i = r / S; j = r - i * S; c = row; return; }
      const int hw = d.H * d.W;                                                // dY dilated: row = (b,y,x) of dX
      const int b = row / hw, q = row - b * hw;
      y = q / d.W; x = q - y * d.W;
      o = k / SS; const int r = k - o * SS; i = r / S; j = r - i * S;
      base = src + (size_t)(b * d.co + o) * d.oh * d.ow;
    } else {  // GRADW, k = (b, y, x) of dY
      const int hw = d.oh * d.ow;
      const int b = k / hw, q = k - b * hw;
      y = q / d.ow; x = q - y * d.ow;
      if (SIDE == 0) { o = row; base = src + ((size_t)(b * d.co + o) * d.oh + y) * d.ow + x; return; }
      c = row / SS; const int r = row - c * SS; i = r / S; j = r - i * S;     // row = (c,i,j)
      y0 = y * d.st + i - d.p; x0 = x * d.st + j - d.p;
      base = src + (size_t)(b * d.ci + c) * d.H * d.W;
    }
  }
  __device__ __forceinline__ uint64_t next(const GemmMap& d) {
    constexpr int SS = S * S;
    uint64_t v = 0;
    if (KIND == PB_CONV_FWD) {
      if (SIDE == 0) return __ldg(base++);
      const int yy = y0 + i, xx = x0 + j;
      if ((unsigned)yy < (unsigned)d.H && (unsigned)xx < (unsigned)d.W) v = __ldg(base + yy * d.W + xx);
      if (++j == S) { j = 0; if (++i == S) { i = 0; base += (size_t)d.H * d.W; } }
    } else if (KIND == PB_CONV_BWDX) {
      if (SIDE == 0) {
        v = __ldg(base + (size_t)(o * d.ci + c) * SS + i * S + j);
      } else {
        const int u = y + d.p - i, w = x + d.p - j;
        if (d.st == 1) {  // stride 1: no division
          if ((unsigned)u < (unsigned)d.oh && (unsigned)w < (unsigned)d.ow) v = __ldg(base + u * d.ow + w);
        } else if (u >= 0 && w >= 0) {
          const int yy = u / d.st, xx = w / d.st;
          if (yy * d.st == u && xx * d.st == w && yy < d.oh && xx < d.ow) v = __ldg(base + yy * d.ow + xx);
        }
      }
      if (++j == S) { j = 0; if (++i == S) { i = 0; ++o; if (SIDE == 1) base += (size_t)d.oh * d.ow; } }
    } else {
      if (SIDE == 0) {
        v = __ldg(base++);  // dY[b][o][y][x], walking (x, y) then jumping to the next image's plane o
        if (++x == d.ow) { x = 0; if (++y == d.oh) { y = 0; base += (size_t)(d.co - 1) * d.oh * d.ow; } }
        return v;
      }
      if ((unsigned)y0 < (unsigned)d.H && (unsigned)x0 < (unsigned)d.W) v = __ldg(base + y0 * d.W + x0);
      x0 += d.st;
      if (++x == d.ow) {
        x = 0; x0 = j - d.p; y0 += d.st;
        if (++y == d.oh) { y = 0; y0 = i - d.p; base += (size_t)d.ci * d.H * d.W; }
      }
    }
    return v;
  }
};

