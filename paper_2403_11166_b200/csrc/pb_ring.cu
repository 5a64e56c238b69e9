// pb_ring.cu — share arithmetic over Z_{2^ell} (R:93-233), the ring GEMM /
// convolution kernels (K:206-278), the numpy-identical Philox share RNG
// (R:48-61) and the dealer-assisted non-linear steps.
//
// Elementwise kernels move 128-bit vectors (two u64 per lane access) and
// use grid-stride loops sized to a multiple of the SM count.
#include <math.h>

#include "pb_common.cuh"

#include <algorithm>

namespace {

__device__ __forceinline__ uint64_t ring_mask(int ell) { return ell >= 64 ? ~0ull : ((1ull << ell) - 1); }

__device__ __forceinline__ int64_t to_signed(uint64_t v, int ell) {  // R:194-198
  const uint64_t m = ring_mask(ell);
  v &= m;
  const uint64_t half = 1ull << (ell - 1);
  return (v >= half) ? (int64_t)(v - m - 1) : (int64_t)v;
}

__global__ void k_ring_binary(int op, uint64_t* out, const uint64_t* a, const uint64_t* b, int64_t n, int64_t bn,
                              int ell) {
  const uint64_t m = ring_mask(ell);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = a[i], y = b[bn == n ? i : i % bn];
    uint64_t r;
    switch (op) {
      case PB_RING_ADD: r = x + y; break;
      case PB_RING_SUB: r = x - y; break;
      default: r = x * y; break;
    }
    out[i] = r & m;
  }
}

// out[i] = a[i] + b[(i / inner) % bn] mod 2^ell: bias add along a channel axis.
__global__ void k_ring_add_bcast(uint64_t* out, const uint64_t* a, const uint64_t* b, int64_t n, int64_t inner,
                                 int64_t bn, int ell) {
  const uint64_t m = ring_mask(ell);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (a[i] + b[(i / inner) % bn]) & m;
}

__global__ void k_ring_unary(int op, uint64_t* out, const uint64_t* a, uint64_t k, int64_t n, int ell) {
  const uint64_t m = ring_mask(ell);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = a[i];
    uint64_t r;
    switch (op) {
      case PB_RING_NEG: r = 0ull - x; break;
      case PB_RING_SCALAR_MUL: r = x * (k & m); break;
      case PB_RING_MASK: r = x; break;
      default: r = (uint64_t)(to_signed(x, ell) >> (int)k); break;  // arith shift
    }
    out[i] = r & m;
  }
}

// R:174-182: floor(x * 2^scale) as two's complement mod 2^ell.
__global__ void k_encode_fixed(const double* x, int64_t n, int ell, int scale, uint64_t* out, int32_t* flag) {
  const double limit = ldexp(1.0, ell - 1) / ldexp(1.0, scale);
  const double s = ldexp(1.0, scale);
  const uint64_t m = ring_mask(ell);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    if (!(fabs(v) < limit)) {
      if (flag) atomicExch(flag, 1);
      out[i] = 0;
      continue;
    }
    const int64_t f = (int64_t)floor(__dmul_rn(v, s));
    out[i] = (uint64_t)f & m;
  }
}

// R:185-191
__global__ void k_decode_fixed(const uint64_t* v, int64_t n, int ell, int scale, double* out) {
  const double s = ldexp(1.0, scale);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ddiv_rn((double)to_signed(v[i], ell), s);
}

// R:60-61 uniform_ring == raw >> (64 - ell) (Lemire with a power-of-two
// range never rejects).  Each thread produces one Philox block (4 raw words).
__global__ void k_uniform_ring(uint64_t* out, const uint64_t* x, uint64_t* do_out, int64_t n, uint64_t seed_arg,
                               const uint64_t* seed_dev, uint64_t stream_id, uint64_t off, int ell) {
  const uint64_t seed = np_seed(seed_arg, seed_dev);
  const int shift = 64 - ell;
  const uint64_t m = ring_mask(ell);
  const uint64_t first_blk = off >> 2;
  const int64_t nblk = (int64_t)(((off + n + 3) >> 2) - first_blk);
  for (int64_t bi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; bi < nblk; bi += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t blk = first_blk + bi;
    const u64x4 r = philox4x64_10(blk + 1, 0, 0, 0, seed, stream_id);
#pragma unroll
    for (int lane = 0; lane < 4; ++lane) {
      const uint64_t raw_idx = blk * 4 + lane;
      if (raw_idx < off || raw_idx >= off + (uint64_t)n) continue;
      const int64_t i = (int64_t)(raw_idx - off);
      const uint64_t v = r.v[lane] >> shift;
      out[i] = v;
      if (do_out) do_out[i] = (x[i] - v) & m;
    }
  }
}

// Scalar-weighted sums of mask tensors (Pencil+ online phase, Alg. 3 steps
// 7-10): out = base (+|-) sum_{i<ma, j<mb} a_i * b_j * T[i][j][:]  mod 2^ell
// (b == NULL: weights a_i alone).  One thread per element; the <= 64
// coefficients live in shared memory.
__global__ void k_ring_lincomb(int sub, uint64_t* out, const uint64_t* base, const uint64_t* a, int ma,
                               const uint64_t* b, int mb, const uint64_t* T, int64_t n, uint64_t mask) {
  __shared__ uint64_t coef[256];
  for (int t = threadIdx.x; t < ma * mb; t += blockDim.x) {
    const int i = t / mb, j = t - i * mb;
    coef[t] = a[i] * (b ? b[j] : 1ull);
  }
  __syncthreads();
  const int mm = ma * mb;
  // two consecutive elements per thread with 16-byte loads when every mask
  // row is 16-byte aligned (n even, aligned bases), eight rows in flight per batch
  const bool al = (((uintptr_t)T | (uintptr_t)out | (uintptr_t)base) & 15) == 0;
  const int64_t np = ((n & 1) || !al) ? 0 : n >> 1;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < np; x += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2* T2 = reinterpret_cast<const ulonglong2*>(T) + x;
    uint64_t acc0 = 0, acc1 = 0;
    int t = 0;
    for (; t + 8 <= mm; t += 8) {
      ulonglong2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(T2 + (int64_t)(t + u) * np);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc0 += coef[t + u] * v[u].x, acc1 += coef[t + u] * v[u].y;
    }
    for (; t < mm; ++t) {
      const ulonglong2 v = __ldg(T2 + (int64_t)t * np);
      acc0 += coef[t] * v.x, acc1 += coef[t] * v.y;
    }
    ulonglong2 b0 = make_ulonglong2(0ull, 0ull);
    if (base) b0 = reinterpret_cast<const ulonglong2*>(base)[x];
    reinterpret_cast<ulonglong2*>(out)[x] =
        make_ulonglong2((sub ? b0.x - acc0 : b0.x + acc0) & mask, (sub ? b0.y - acc1 : b0.y + acc1) & mask);
  }
  if (np) return;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    uint64_t acc = 0;
    for (int t = 0; t < mm; ++t) acc += coef[t] * __ldg(T + (int64_t)t * n + x);
    const uint64_t b0 = base ? base[x] : 0ull;
    out[x] = (sub ? b0 - acc : b0 + acc) & mask;
  }
}

// K:206-218 ring GEMM for the FC layers' local terms (n k m < 2^24): a CTA
// owns a 16x16 output tile and stages a whole 128-deep slab of its A rows and
// B columns in shared memory with every load issued at once (coalesced in
// the operand's contiguous direction), then each thread runs the slab's MACs
// from shared memory with two accumulators -- one global round trip per 128
// of k instead of one per 16 (the 16x16 k-tile loop was latency-bound: 9.9 us
// for 128x128x64).  Fused epilogue: out = C + sign * (A B)  (C may be NULL).
// TS = 8: 4 lanes per output split each slab (kk = lane mod 4) and combine
// with two shuffles -- 4x the CTAs and a quarter of the serial MACs for the
// mid-size local terms (128x128x64: 32 -> 128 CTAs).
constexpr int MM_KC = 128;
template <int TS>
__global__ void __launch_bounds__(256) k_ring_mm_tile(const uint64_t* __restrict__ A, const uint64_t* __restrict__ B,
                                                      int n, int k, int m, int ta, int tb,
                                                      const uint64_t* __restrict__ C, int sign, uint64_t mask,
                                                      uint64_t* __restrict__ out) {
  constexpr int LK = 256 / (TS * TS);  // lanes per output
  __shared__ uint64_t sa[TS][MM_KC + 1];
  __shared__ uint64_t sb[MM_KC][TS + 1];
  const int tid = threadIdx.x, lane = tid % LK, oi = tid / LK, tx = oi % TS, ty = oi / TS;
  const int row0 = blockIdx.y * TS, col0 = blockIdx.x * TS;
  uint64_t acc0 = 0, acc1 = 0;
  for (int k0 = 0; k0 < k; k0 += MM_KC) {
    const int kc = min(MM_KC, k - k0);
#pragma unroll 4
    for (int idx = tid; idx < TS * MM_KC; idx += 256) {
      int r, kk;
      if (ta) kk = idx / TS, r = idx % TS;  // A stored (k, n): rows contiguous
      else r = idx / MM_KC, kk = idx % MM_KC;  // A stored (n, k): k contiguous
      const int gr = row0 + r, gk = k0 + kk;
      sa[r][kk] = (gr < n && kk < kc) ? (ta ? __ldg(A + (int64_t)gk * n + gr) : __ldg(A + (int64_t)gr * k + gk)) : 0ull;
      int c, kb;
      if (tb) c = idx / MM_KC, kb = idx % MM_KC;  // B stored (m, k): k contiguous
      else kb = idx / TS, c = idx % TS;           // B stored (k, m): columns contiguous
      const int gc = col0 + c, gkb = k0 + kb;
      sb[kb][c] = (gc < m && kb < kc) ? (tb ? __ldg(B + (int64_t)gc * k + gkb) : __ldg(B + (int64_t)gkb * m + gc)) : 0ull;
    }
    __syncthreads();
    int kk = lane;
    for (; kk + LK < kc; kk += 2 * LK) {
      acc0 += sa[ty][kk] * sb[kk][tx];
      acc1 += sa[ty][kk + LK] * sb[kk + LK][tx];
    }
    if (kk < kc) acc0 += sa[ty][kk] * sb[kk][tx];
    __syncthreads();
  }
  uint64_t v = acc0 + acc1;
#pragma unroll
  for (int off = LK / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off, LK);
  const int row = row0 + ty, col = col0 + tx;
  if (lane == 0 && row < n && col < m) {
    const int64_t o = (int64_t)row * m + col;
    out[o] = (C ? (sign >= 0 ? C[o] + v : C[o] - v) : v) & mask;
  }
}

// Latency variant for few outputs (n m < 2^14): G lanes per output split the
// contraction, each lane issues all loads of its next 8 k-values at once, MACs
// them, and a shuffle tree combines the lanes -- one global round trip per 8 G
// of k (the CTA-tile kernel needs 7.4 us for 128x128x64 with 32 CTAs on B200).
template <int G>
__global__ void __launch_bounds__(256) k_ring_mm_lanes(const uint64_t* __restrict__ A, const uint64_t* __restrict__ B,
                                                       int n, int k, int m, int ta, int tb,
                                                       const uint64_t* __restrict__ C, int sign, uint64_t mask,
                                                       uint64_t* __restrict__ out) {
  const int lane = threadIdx.x % G;
  const int64_t o = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const bool valid = o < (int64_t)n * m;
  const int row = valid ? (int)(o / m) : 0, col = valid ? (int)(o % m) : 0;
  uint64_t acc = 0;
  for (int k0 = 0; k0 < k; k0 += 8 * G) {
    uint64_t av[8], bv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int kk = k0 + j * G + lane;
      const bool in = kk < k;
      av[j] = in ? (ta ? __ldg(A + (int64_t)kk * n + row) : __ldg(A + (int64_t)row * k + kk)) : 0ull;
      bv[j] = in ? (tb ? __ldg(B + (int64_t)col * k + kk) : __ldg(B + (int64_t)kk * m + col)) : 0ull;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += av[j] * bv[j];
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off, G);
  if (lane == 0 && valid) out[o] = (C ? (sign >= 0 ? C[o] + acc : C[o] - acc) : acc) & mask;
}

__global__ void k_rowsum(const uint64_t* a, int64_t rows, int64_t cols, uint64_t mask, uint64_t* out) {
  const int64_t r = blockIdx.x;
  uint64_t acc = 0;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) acc += a[r * cols + j];
  __shared__ uint64_t red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[r] = red[0] & mask;
}

// Per-channel sums of a (B, C, HW) tensor, out[c] = sum_{b,i} a[b][c][i] mod
// 2^ell (the conv bias gradient), straight from the NCHW layout:
// CTA (s, c) adds a contiguous chunk of channel c's flattened (b, i) range
// into part[c][s] (u64 sums wrap mod 2^64: any split is exact), then one warp
// per channel adds its S partials and masks.  Replaces a permute copy and a
// one-CTA-per-channel reduction (C = 64 CTAs: 35 us per call on CIFAR conv1).
__device__ __forceinline__ uint64_t block_sum_u64(uint64_t acc) {
  __shared__ uint64_t red[32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ull;
  if (threadIdx.x < 32) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  }
  return acc;
}

__global__ void __launch_bounds__(256) k_chansum_part(const uint64_t* __restrict__ a, int C, uint32_t HW,
                                                      uint32_t total, uint32_t chunk, uint64_t* __restrict__ part) {
  const int c = blockIdx.y;
  const uint32_t j0 = blockIdx.x * chunk, j1 = min(total, j0 + chunk);
  uint64_t acc = 0;
  if (HW >= blockDim.x) {  // (b, i) of the first element once, then walked (at most one wrap per step)
    uint32_t b = (j0 + threadIdx.x) / HW, i = j0 + threadIdx.x - b * HW;
    for (uint32_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
      acc += __ldg(a + ((uint64_t)b * C + c) * HW + i);
      i += blockDim.x;
      if (i >= HW) { i -= HW; ++b; }
    }
  } else {
    for (uint32_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
      const uint32_t b = j / HW;
      acc += __ldg(a + ((uint64_t)b * C + c) * HW + (j - b * HW));
    }
  }
  acc = block_sum_u64(acc);
  if (threadIdx.x == 0) part[(uint64_t)c * gridDim.x + blockIdx.x] = acc;
}

__global__ void k_chansum_fin(const uint64_t* __restrict__ part, int C, int S, uint64_t mask, uint64_t* out) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= C) return;
  uint64_t acc = 0;
  for (int s = lane; s < S; s += 32) acc += part[(int64_t)c * S + s];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) out[c] = acc & mask;
}

// K:221-238 im2col (gather form: one thread per output element).
__global__ void k_im2col(const uint64_t* x, int B, int C, int H, int W, int s, int stride, uint64_t* out) {
  const int oh = (H - s) / stride + 1, ow = (W - s) / stride + 1;
  const int64_t ncol = (int64_t)B * oh * ow;
  const int64_t total = ncol * C * s * s;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / ncol, col = e - row * ncol;
    const int dj = (int)(row % s), di = (int)((row / s) % s), c = (int)(row / (s * s));
    const int j = (int)(col % ow), i = (int)((col / ow) % oh), b = (int)(col / ((int64_t)oh * ow));
    out[e] = x[(((int64_t)b * C + c) * H + i * stride + di) * W + j * stride + dj];
  }
}

// K:241-257 col2im (gather form of the scatter-add: each output pixel sums
// the patch entries that map onto it, so no atomics are needed).
__global__ void k_col2im(const uint64_t* cols, int B, int C, int H, int W, int s, int stride, uint64_t* out) {
  const int oh = (H - s) / stride + 1, ow = (W - s) / stride + 1;
  const int64_t ncol = (int64_t)B * oh * ow;
  const int64_t total = (int64_t)B * C * H * W;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int xw = (int)(e % W), xh = (int)((e / W) % H), c = (int)((e / ((int64_t)W * H)) % C);
    const int b = (int)(e / ((int64_t)W * H * C));
    uint64_t acc = 0;
    for (int di = 0; di < s; ++di) {
      const int ii = xh - di;
      if (ii < 0 || ii % stride) continue;
      const int i = ii / stride;
      if (i >= oh) continue;
      for (int dj = 0; dj < s; ++dj) {
        const int jj = xw - dj;
        if (jj < 0 || jj % stride) continue;
        const int j = jj / stride;
        if (j >= ow) continue;
        const int64_t row = ((int64_t)c * s + di) * s + dj;
        const int64_t col = ((int64_t)b * oh + i) * ow + j;
        acc += cols[row * ncol + col];
      }
    }
    out[e] = acc;
  }
}

// K:260-278 conv2d_wrap (valid, stride 1).
__global__ void k_conv2d(const uint64_t* x, const uint64_t* w, int B, int Ci, int H, int W, int Co, int s, uint64_t mask,
                         uint64_t* out) {
  const int oh = H - s + 1, ow = W - s + 1;
  const int64_t total = (int64_t)B * Co * oh * ow;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % ow), i = (int)((e / ow) % oh), co = (int)((e / ((int64_t)ow * oh)) % Co);
    const int b = (int)(e / ((int64_t)ow * oh * Co));
    uint64_t acc = 0;
    for (int ci = 0; ci < Ci; ++ci)
      for (int di = 0; di < s; ++di)
        for (int dj = 0; dj < s; ++dj)
          acc += x[(((int64_t)b * Ci + ci) * H + i + di) * W + j + dj] * w[(((int64_t)co * Ci + ci) * s + di) * s + dj];
    out[e] = acc & mask;
  }
}

// Dealer-assisted non-linear step: reconstruct, apply, reshare with the
// numpy-identical uniform_ring stream (so oracle and device shares agree).
// One thread per numpy Philox block (4 raw draws): the reshare words of four
// consecutive elements from one Philox4x64-10 evaluation (one per element
// recomputed the block 4x -- the kernel was RNG-bound, 60 us on 4M elements).
__global__ void k_dealer(int op, const uint64_t* in_mo, const uint64_t* in_do, uint64_t* mo, uint64_t* dov, int64_t n,
                         int k, const uint8_t* d_in, uint8_t* d_out, uint64_t seed_arg, const uint64_t* seed_dev,
                         uint64_t stream_id, uint64_t off, int ell) {
  const uint64_t seed = np_seed(seed_arg, seed_dev);
  const uint64_t m = ring_mask(ell);
  const int shift = 64 - ell;
  const uint64_t first_blk = off >> 2;
  const int64_t nblk = (int64_t)(((off + n + 3) >> 2) - first_blk);
  const bool al = (((uintptr_t)in_mo | (uintptr_t)in_do | (uintptr_t)mo | (uintptr_t)dov) & 15) == 0;
  for (int64_t bi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; bi < nblk; bi += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t blk = first_blk + bi;
    const u64x4 rv = philox4x64_10(blk + 1, 0, 0, 0, seed, stream_id);  // numpy pre-increments the counter
    // the block's four elements as two 16-byte vectors when they are all in
    // range and 16-byte aligned (off even), else element by element
    const int64_t i0 = (int64_t)(blk * 4) - (int64_t)off;
    const bool vec = al && !(off & 1) && i0 >= 0 && i0 + 4 <= n;
    uint64_t xs[4];
    if (vec) {
      const ulonglong2 a0 = *reinterpret_cast<const ulonglong2*>(in_mo + i0),
                       a1 = *reinterpret_cast<const ulonglong2*>(in_mo + i0 + 2),
                       b0 = *reinterpret_cast<const ulonglong2*>(in_do + i0),
                       b1 = *reinterpret_cast<const ulonglong2*>(in_do + i0 + 2);
      xs[0] = (a0.x + b0.x) & m, xs[1] = (a0.y + b0.y) & m, xs[2] = (a1.x + b1.x) & m, xs[3] = (a1.y + b1.y) & m;
    }
    uint64_t ro[4], rd[4];
#pragma unroll
    for (int lane = 0; lane < 4; ++lane) {
      const uint64_t raw = blk * 4 + lane;
      if (!vec && (raw < off || raw >= off + (uint64_t)n)) continue;
      const int64_t i = (int64_t)(raw - off);
      const uint64_t x = vec ? xs[lane] : (in_mo[i] + in_do[i]) & m;
      uint64_t y;
      switch (op) {
        case PB_DEALER_RELU: {
          const bool pos = to_signed(x, ell) >= 0;
          if (d_out) d_out[i] = pos ? 1 : 0;
          y = pos ? x : 0ull;
          break;
        }
        case PB_DEALER_TRUNC: y = (uint64_t)(to_signed(x, ell) >> k) & m; break;
        case PB_DEALER_SELECT: y = d_in[i] ? x : 0ull; break;
        case PB_DEALER_RELU_TRUNC: {  // trunc_k(relu(x)): the relu reshare is never observed
          const bool pos = to_signed(x, ell) >= 0;
          if (d_out) d_out[i] = pos ? 1 : 0;
          y = pos ? ((uint64_t)(to_signed(x, ell) >> k) & m) : 0ull;
          break;
        }
        case PB_DEALER_TRUNC_SELECT: y = d_in[i] ? ((uint64_t)(to_signed(x, ell) >> k) & m) : 0ull; break;
        default: y = x; break;
      }
      const uint64_t r = rv.v[lane] >> shift;
      ro[lane] = r, rd[lane] = (y - r) & m;
      if (!vec) mo[i] = r, dov[i] = rd[lane];
    }
    if (vec) {
      *reinterpret_cast<ulonglong2*>(mo + i0) = make_ulonglong2(ro[0], ro[1]);
      *reinterpret_cast<ulonglong2*>(mo + i0 + 2) = make_ulonglong2(ro[2], ro[3]);
      *reinterpret_cast<ulonglong2*>(dov + i0) = make_ulonglong2(rd[0], rd[1]);
      *reinterpret_cast<ulonglong2*>(dov + i0 + 2) = make_ulonglong2(rd[2], rd[3]);
    }
  }
}

__global__ void k_sgd(double* w, double* v, const uint64_t* g, int64_t n, int gscale, double lr, double mom, int ell,
                      int wscale, uint64_t* w_ring, int32_t* flag, const uint32_t* skip) {
  if (skip && *skip) return;  // the step was aborted before its gradient was released: keep w, v, W
  const double gs = ldexp(1.0, gscale), ws = ldexp(1.0, wscale);
  const double limit = ldexp(1.0, ell - 1) / ws;
  const uint64_t m = ring_mask(ell);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = __ddiv_rn((double)to_signed(g[i], ell), gs);
    const double vi = __dadd_rn(__dmul_rn(mom, v[i]), gi);
    const double wi = __dsub_rn(w[i], __dmul_rn(lr, vi));
    v[i] = vi;
    w[i] = wi;
    if (!(fabs(wi) < limit)) {
      if (flag) atomicExch(flag, 1);
      w_ring[i] = 0;
    } else {
      w_ring[i] = (uint64_t)(int64_t)floor(__dmul_rn(wi, ws)) & m;
    }
  }
}

__global__ void k_scatter_u64(uint64_t* __restrict__ out, const uint64_t* __restrict__ src,
                              const int64_t* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = __ldg(dst + i);
    if (d >= 0) out[d] = __ldg(src + i);
  }
}

bool bad_ell(int ell) { return ell < 2 || ell > 64; }

}  // namespace

// ================================================================ C ABI ===
#define RING_GRID(n) pb_grid_1d((n), 256), 256, 0, pb_stream_of(stream)

extern "C" int pb_ring_binary(int op, uint64_t* out, const uint64_t* a, const uint64_t* b, int64_t n, int64_t b_n,
                              int32_t ell, void* stream) {
  if (n > 0 && (!out || !a || !b)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (op < PB_RING_ADD || op > PB_RING_MUL || bad_ell(ell)) return pb_set_error(PB_ERR_ARG, "bad ring op / ell");
  if (n <= 0) return PB_OK;
  if (b_n <= 0 || n % b_n) return pb_set_error(PB_ERR_SHAPE, "broadcast size must divide n");
  k_ring_binary<<<RING_GRID(n)>>>(op, out, a, b, n, b_n, ell);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_ring_unary(int op, uint64_t* out, const uint64_t* a, uint64_t k, int64_t n, int32_t ell, void* stream) {
  if (n > 0 && (!out || !a)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (op < PB_RING_NEG || op > PB_RING_ARITH_SHIFT || bad_ell(ell)) return pb_set_error(PB_ERR_ARG, "bad ring op / ell");
  if (op == PB_RING_ARITH_SHIFT && k >= 64) return pb_set_error(PB_ERR_ARG, "shift too large");
  if (n <= 0) return PB_OK;
  k_ring_unary<<<RING_GRID(n)>>>(op, out, a, k, n, ell);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_encode_fixed(const double* x, int64_t n, int32_t ell, int32_t scale, uint64_t* out, int32_t* flag,
                               void* stream) {
  if (n > 0 && (!x || !out)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (bad_ell(ell) || scale < 0 || scale >= ell) return pb_set_error(PB_ERR_SCALE, "bad scale");
  if (n <= 0) return PB_OK;
  k_encode_fixed<<<RING_GRID(n)>>>(x, n, ell, scale, out, flag);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_decode_fixed(const uint64_t* v, int64_t n, int32_t ell, int32_t scale, double* out, void* stream) {
  if (n > 0 && (!v || !out)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (bad_ell(ell) || scale < 0 || scale >= ell) return pb_set_error(PB_ERR_SCALE, "bad scale");
  if (n <= 0) return PB_OK;
  k_decode_fixed<<<RING_GRID(n)>>>(v, n, ell, scale, out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_uniform_ring(uint64_t* out, int64_t n, uint64_t seed, const uint64_t* seed_dev, uint64_t stream_id,
                               uint64_t raw_offset,
                               int32_t ell, void* stream) {
  if (n > 0 && !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (ell < 1 || ell > 63) return pb_set_error(PB_ERR_ARG, "bad ell");
  if (n <= 0) return PB_OK;
  k_uniform_ring<<<RING_GRID((n + 3) / 4 + 1)>>>(out, nullptr, nullptr, n, seed, seed_dev, stream_id, raw_offset, ell);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_share(const uint64_t* x, int64_t n, uint64_t seed, const uint64_t* seed_dev, uint64_t stream_id,
                        uint64_t raw_offset,
                        int32_t ell, uint64_t* mo_out, uint64_t* do_out, void* stream) {
  if (n > 0 && (!x || !mo_out || !do_out)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (ell < 1 || ell > 63) return pb_set_error(PB_ERR_ARG, "bad ell");
  if (n <= 0) return PB_OK;
  k_uniform_ring<<<RING_GRID((n + 3) / 4 + 1)>>>(mo_out, x, do_out, n, seed, seed_dev, stream_id, raw_offset, ell);
  PB_CHECK_LAUNCH();
  return PB_OK;
}


extern "C" int pb_ring_rowsum(const uint64_t* a, int64_t rows, int64_t cols, int32_t ell, uint64_t* out, void* stream) {
  if (rows > 0 && (!a || !out)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (rows <= 0) return PB_OK;
  const uint64_t mask = (ell >= 64 || ell <= 0) ? ~0ull : ((1ull << ell) - 1);
  k_rowsum<<<(unsigned)rows, 256, 0, pb_stream_of(stream)>>>(a, rows, cols, mask, out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_ring_chansum(const uint64_t* a, int32_t B, int32_t C, int64_t HW, int32_t ell, uint64_t* out,
                               void* stream) {
  if (B < 0 || C < 0 || HW < 0) return pb_set_error(PB_ERR_SHAPE, "negative extent");
  if (C == 0) return PB_OK;
  if (!out || (!a && (int64_t)B * HW > 0)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (C > 65535 || (int64_t)B * HW > 0x7fffffffLL) return pb_set_error(PB_ERR_SHAPE, "tensor too large");
  const uint64_t mask = (ell >= 64 || ell <= 0) ? ~0ull : ((1ull << ell) - 1);
  cudaStream_t st = pb_stream_of(stream);
  const uint32_t total = (uint32_t)((int64_t)B * HW);
  // splits: about four CTAs per SM over all channels, at least 2048 elements each
  int S = (int)std::max<int64_t>(1, std::min<int64_t>((4 * 148 + C - 1) / C, (total + 2047) / 2048));
  const uint32_t chunk = (total + S - 1) / S;
  if (total) S = (int)((total + chunk - 1) / chunk);
  uint64_t* part = nullptr;
  if (cudaMallocAsync((void**)&part, (size_t)C * S * sizeof(uint64_t), st) != cudaSuccess)
    return pb_set_error(PB_ERR_CUDA, "channel-sum scratch allocation failed");
  if (total)
    k_chansum_part<<<dim3((unsigned)S, (unsigned)C), 256, 0, st>>>(a, C, (uint32_t)HW, total, chunk, part);
  else
    cudaMemsetAsync(part, 0, (size_t)C * S * sizeof(uint64_t), st);
  k_chansum_fin<<<(unsigned)((C + 7) / 8), 256, 0, st>>>(part, C, S, mask, out);
  cudaFreeAsync(part, st);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_im2col(const uint64_t* x, int32_t B, int32_t C, int32_t H, int32_t W, int32_t s, int32_t stride,
                         uint64_t* out, void* stream) {
  if (!x || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (s < 1 || stride < 1 || s > H || s > W) return pb_set_error(PB_ERR_GEOMETRY, "bad im2col geometry");
  const int64_t total = (int64_t)B * ((H - s) / stride + 1) * ((W - s) / stride + 1) * C * s * s;
  if (total <= 0) return PB_OK;
  k_im2col<<<RING_GRID(total)>>>(x, B, C, H, W, s, stride, out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_col2im(const uint64_t* cols, int32_t B, int32_t C, int32_t H, int32_t W, int32_t s, int32_t stride,
                         uint64_t* out, void* stream) {
  if (!cols || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (s < 1 || stride < 1 || s > H || s > W) return pb_set_error(PB_ERR_GEOMETRY, "bad col2im geometry");
  const int64_t total = (int64_t)B * C * H * W;
  if (total <= 0) return PB_OK;
  k_col2im<<<RING_GRID(total)>>>(cols, B, C, H, W, s, stride, out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_conv2d(const uint64_t* x, const uint64_t* w, int32_t B, int32_t Ci, int32_t H, int32_t W, int32_t Co,
                         int32_t s, int32_t ell, uint64_t* out, void* stream) {
  if (!x || !w || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (s < 1 || s > H || s > W) return pb_set_error(PB_ERR_GEOMETRY, "bad conv geometry");
  const int64_t total = (int64_t)B * Co * (H - s + 1) * (W - s + 1);
  if (total <= 0) return PB_OK;
  const uint64_t mask = (ell >= 64 || ell <= 0) ? ~0ull : ((1ull << ell) - 1);
  k_conv2d<<<RING_GRID(total)>>>(x, w, B, Ci, H, W, Co, s, mask, out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_dealer_op(int op, uint64_t* mo, uint64_t* do_, int64_t n, int32_t k, const uint8_t* d_in,
                            uint8_t* d_out, uint64_t seed, const uint64_t* seed_dev, uint64_t stream_id,
                            uint64_t raw_offset, int32_t ell,
                            void* stream) {
  return pb_dealer_op_out(op, mo, do_, mo, do_, n, k, d_in, d_out, seed, seed_dev, stream_id, raw_offset, ell, stream);
}

extern "C" int pb_dealer_op_out(int op, const uint64_t* in_mo, const uint64_t* in_do, uint64_t* mo, uint64_t* do_,
                                int64_t n, int32_t k, const uint8_t* d_in, uint8_t* d_out, uint64_t seed,
                                const uint64_t* seed_dev, uint64_t stream_id, uint64_t raw_offset, int32_t ell,
                                void* stream) {
  if (n > 0 && (!mo || !do_ || !in_mo || !in_do)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (op < PB_DEALER_RELU || op > PB_DEALER_TRUNC_SELECT) return pb_set_error(PB_ERR_ARG, "bad dealer op");
  if ((op == PB_DEALER_SELECT || op == PB_DEALER_TRUNC_SELECT) && !d_in)
    return pb_set_error(PB_ERR_ARG, "select needs d_in");
  if (ell < 2 || ell > 63 || k < 0 || k >= ell) return pb_set_error(PB_ERR_ARG, "bad ell / shift");
  if (n <= 0) return PB_OK;
  k_dealer<<<RING_GRID((n + 3) / 4 + 1)>>>(op, in_mo, in_do, mo, do_, n, k, d_in, d_out, seed, seed_dev, stream_id, raw_offset,
                             ell);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_sgd_momentum(double* w, double* v, const uint64_t* grad_ring, int64_t n, int32_t grad_scale, double lr,
                               double momentum, int32_t ell, int32_t w_scale, uint64_t* w_ring, int32_t* range_flag,
                               const uint32_t* skip, void* stream) {
  if (n > 0 && (!w || !v || !grad_ring || !w_ring)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (bad_ell(ell)) return pb_set_error(PB_ERR_ARG, "bad ell");
  if (n <= 0) return PB_OK;
  k_sgd<<<RING_GRID(n)>>>(w, v, grad_ring, n, grad_scale, lr, momentum, ell, w_scale, w_ring, range_flag, skip);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_ring_lincomb(int subtract, uint64_t* out, const uint64_t* base, const uint64_t* a, int32_t ma,
                               const uint64_t* b, int32_t mb, const uint64_t* T, int64_t n, int32_t ell, void* stream) {
  if (n > 0 && (!out || !a || !T)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (ma < 1 || mb < 1 || ma * mb > 256) return pb_set_error(PB_ERR_ARG, "ma * mb must be in [1, 256]");
  if (bad_ell(ell)) return pb_set_error(PB_ERR_ARG, "bad ell");
  if (n <= 0) return PB_OK;
  const uint64_t mask = ell >= 64 ? ~0ull : ((1ull << ell) - 1);
  k_ring_lincomb<<<RING_GRID(n)>>>(subtract ? 1 : 0, out, base, a, ma, b, mb, T, n, mask);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

// Small-shape matmul launcher used by pb_ring_matmul (pb_conv.cu).
void pb_launch_ring_matmul_small(const uint64_t* a, const uint64_t* b, int64_t n, int64_t k, int64_t m, int trans_a,
                                 int trans_b, const uint64_t* c, int sign, uint64_t mask, uint64_t* out,
                                 cudaStream_t st) {
  const int64_t outs = n * m;
  if (outs >= (1 << 16)) {  // enough outputs to fill the GPU with 16x16 tiles
    dim3 grd((unsigned)((m + 15) / 16), (unsigned)((n + 15) / 16));
    k_ring_mm_tile<16><<<grd, 256, 0, st>>>(a, b, (int)n, (int)k, (int)m, trans_a, trans_b, c, sign, mask, out);
    return;
  }
  if (outs >= (1 << 12)) {  // mid-size: 8x8 tiles, 4 lanes per output
    dim3 grd((unsigned)((m + 7) / 8), (unsigned)((n + 7) / 8));
    k_ring_mm_tile<8><<<grd, 256, 0, st>>>(a, b, (int)n, (int)k, (int)m, trans_a, trans_b, c, sign, mask, out);
    return;
  }
  auto go = [&](auto kern, int g) {
    kern<<<(unsigned)((outs * g + 255) / 256), 256, 0, st>>>(a, b, (int)n, (int)k, (int)m, trans_a, trans_b, c, sign,
                                                             mask, out);
  };
  if (k <= 8)
    go(k_ring_mm_lanes<1>, 1);
  else if (k <= 16)
    go(k_ring_mm_lanes<2>, 2);
  else if (k <= 32)
    go(k_ring_mm_lanes<4>, 4);
  else if (k <= 64)
    go(k_ring_mm_lanes<8>, 8);
  else if (k <= 128)
    go(k_ring_mm_lanes<16>, 16);
  else
    go(k_ring_mm_lanes<32>, 32);
}

extern "C" int pb_ring_add_bcast(uint64_t* out, const uint64_t* a, const uint64_t* b, int64_t n, int64_t inner,
                                 int64_t bn, int32_t ell, void* stream) {
  if (n > 0 && (!out || !a || !b)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (inner < 1 || bn < 1 || bad_ell(ell)) return pb_set_error(PB_ERR_ARG, "bad broadcast / ell");
  if (n <= 0) return PB_OK;
  k_ring_add_bcast<<<RING_GRID(n)>>>(out, a, b, n, inner, bn, ell);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

// The multi-rank combine's last step (linear_protocols.gather_maps): the
// all-gathered compact share tiles scattered into the output tensor.
extern "C" int pb_scatter_u64(uint64_t* out, const uint64_t* src, const int64_t* dst, int64_t n, void* stream) {
  if (n > 0 && (!out || !src || !dst)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (n <= 0) return PB_OK;
  k_scatter_u64<<<RING_GRID(n)>>>(out, src, dst, n);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

// Pencil+ online scalars of one operator in one launch: k_i (the MO's, stream
// stream_k) and l_j (the DO's, stream_l), i, j < m, each the first m
// uniform_ring draws of its numpy-identical stream (R:60-61, raw >> (64 - ell))
// with 0 replaced by 1 (the weights must be nonzero; P[0] = 2^-ell).
namespace {
__global__ void k_prep_scalars(uint64_t* k_out, uint64_t* l_out, int m, uint64_t seed_arg, const uint64_t* seed_dev,
                               uint64_t stream_k, uint64_t stream_l, int ell) {
  const uint64_t seed = np_seed(seed_arg, seed_dev);
  const int t = threadIdx.x;
  if (t >= 2 * m) return;
  const int who = t >= m, i = t - who * m;
  const uint64_t v = philox_np_raw(seed, who ? stream_l : stream_k, (uint64_t)i) >> (64 - ell);
  (who ? l_out : k_out)[i] = v ? v : 1ull;
}
}  // namespace

extern "C" int pb_prep_scalars(uint64_t* k_out, uint64_t* l_out, int32_t m, uint64_t seed, const uint64_t* seed_dev,
                               uint64_t stream_k, uint64_t stream_l, int32_t ell, void* stream) {
  if (!k_out || !l_out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (m < 1 || m > 256 || bad_ell(ell) || ell > 63) return pb_set_error(PB_ERR_ARG, "bad m / ell");
  k_prep_scalars<<<1, 2 * m, 0, pb_stream_of(stream)>>>(k_out, l_out, m, seed, seed_dev, stream_k, stream_l, ell);
  PB_CHECK_LAUNCH();
  return PB_OK;
}
