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
