// pb_conv.cu — plaintext Z_{2^ell} conv-layer operators with padding and
// stride (the parties' local terms of the conv protocols and of Alg. 2), and
// AvgPool2 window sums / gradient replication.
//
// The reference ships only valid-mode stride-1 conv2d_wrap (K:260-278) and
// im2col/col2im (K:221-257); padding and stride are "pre/post tensor
// transforms outside the codec".  These kernels apply the
// transforms on the fly (index arithmetic, no padded / dilated copies):
//
//   FWD    Y[b,o,y,x]  = sum_{c,i,j} W[o,c,i,j] X[b,c,y*st+i-p,x*st+j-p]
//   BWDX   dX[b,c,y,x] = sum_{o,i,j: st | y+p-i, x+p-j} W[o,c,i,j] dY[b,o,(y+p-i)/st,(x+p-j)/st]
//   GRADW  dW[o,c,i,j] = sum_{b,y,x} dY[b,o,y,x] X[b,c,y*st+i-p,x*st+j-p]
//
// all with uint64 wraparound, masked to ell bits (bit-identical to the
// oracle's conv2d_wrap composition, oracle/convops.py).  GRADW reduces over
// B*oh*ow terms per output: one CTA per (o, c) pair keeps the S*S
// accumulators in registers and reduces them through shared memory.
#include "pb_common.cuh"
#include "pb_gemm_maps.cuh"

#include <stdlib.h>

namespace {

__host__ __device__ __forceinline__ uint64_t cmask(int ell) { return ell >= 64 ? ~0ull : ((1ull << ell) - 1); }

__global__ void k_conv_fwd(const uint64_t* __restrict__ X, const uint64_t* __restrict__ Wt, int B, int ci, int co,
                           int H, int W, int s, int p, int st, int oh, int ow, uint64_t m, uint64_t* __restrict__ Y) {
  const int64_t total = (int64_t)B * co * oh * ow;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(e % ow), y = (int)((e / ow) % oh), o = (int)((e / ((int64_t)ow * oh)) % co);
    const int b = (int)(e / ((int64_t)ow * oh * co));
    uint64_t acc = 0;
    for (int c = 0; c < ci; ++c) {
      const uint64_t* xp = X + ((int64_t)b * ci + c) * H * W;
      const uint64_t* wp = Wt + ((int64_t)o * ci + c) * s * s;
      for (int i = 0; i < s; ++i) {
        const int yy = y * st + i - p;
        if (yy < 0 || yy >= H) continue;
        for (int j = 0; j < s; ++j) {
          const int xx = x * st + j - p;
          if (xx < 0 || xx >= W) continue;
          acc += __ldg(xp + (int64_t)yy * W + xx) * __ldg(wp + i * s + j);
        }
      }
    }
    Y[e] = acc & m;
  }
}

__global__ void k_conv_bwdx(const uint64_t* __restrict__ dY, const uint64_t* __restrict__ Wt, int B, int ci, int co,
                            int H, int W, int s, int p, int st, int oh, int ow, uint64_t m, uint64_t* __restrict__ dX) {
  const int64_t total = (int64_t)B * ci * H * W;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(e % W), y = (int)((e / W) % H), c = (int)((e / ((int64_t)W * H)) % ci);
    const int b = (int)(e / ((int64_t)W * H * ci));
    uint64_t acc = 0;
    for (int o = 0; o < co; ++o) {
      const uint64_t* gp = dY + ((int64_t)b * co + o) * oh * ow;
      const uint64_t* wp = Wt + ((int64_t)o * ci + c) * s * s;
      for (int i = 0; i < s; ++i) {
        const int u = y + p - i;
        if (u < 0 || u % st) continue;
        const int yy = u / st;
        if (yy >= oh) continue;
        for (int j = 0; j < s; ++j) {
          const int v = x + p - j;
          if (v < 0 || v % st) continue;
          const int xx = v / st;
          if (xx >= ow) continue;
          acc += __ldg(gp + (int64_t)yy * ow + xx) * __ldg(wp + i * s + j);
        }
      }
    }
    dX[e] = acc & m;
  }
}

// One CTA per (o, c); threads stride over the (b, y, x) reduction.
template <int S>
__global__ void __launch_bounds__(256) k_conv_gradw(const uint64_t* __restrict__ X, const uint64_t* __restrict__ dY,
                                                    int B, int ci, int co, int H, int W, int p, int st, int oh, int ow,
                                                    uint64_t m, uint64_t* __restrict__ dW) {
  const int o = blockIdx.x / ci, c = blockIdx.x % ci;
  uint64_t acc[S * S];
#pragma unroll
  for (int k = 0; k < S * S; ++k) acc[k] = 0;
  const int64_t n = (int64_t)B * oh * ow;
  for (int64_t r = threadIdx.x; r < n; r += blockDim.x) {
    const int x = (int)(r % ow), y = (int)((r / ow) % oh), b = (int)(r / ((int64_t)ow * oh));
    const uint64_t g = __ldg(dY + (((int64_t)b * co + o) * oh + y) * ow + x);
    const uint64_t* xp = X + ((int64_t)b * ci + c) * H * W;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const int yy = y * st + i - p;
      const bool oky = yy >= 0 && yy < H;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const int xx = x * st + j - p;
        if (oky && xx >= 0 && xx < W) acc[i * S + j] += g * __ldg(xp + (int64_t)yy * W + xx);
      }
    }
  }
  __shared__ uint64_t red[256 / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < S * S; ++k) {
    uint64_t v = acc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      dW[((int64_t)o * ci + c) * S * S + k] = t & m;
    }
    __syncthreads();
  }
}

// Generic kernel size: one thread per dW element (small outputs only).
__global__ void k_conv_gradw_any(const uint64_t* __restrict__ X, const uint64_t* __restrict__ dY, int B, int ci,
                                 int co, int H, int W, int s, int p, int st, int oh, int ow, uint64_t m,
                                 uint64_t* __restrict__ dW) {
  const int64_t total = (int64_t)co * ci * s * s;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % s), i = (int)((e / s) % s), c = (int)((e / ((int64_t)s * s)) % ci);
    const int o = (int)(e / ((int64_t)s * s * ci));
    uint64_t acc = 0;
    for (int b = 0; b < B; ++b)
      for (int y = 0; y < oh; ++y) {
        const int yy = y * st + i - p;
        if (yy < 0 || yy >= H) continue;
        for (int x = 0; x < ow; ++x) {
          const int xx = x * st + j - p;
          if (xx < 0 || xx >= W) continue;
          acc += dY[(((int64_t)b * co + o) * oh + y) * ow + x] * X[(((int64_t)b * ci + c) * H + yy) * W + xx];
        }
      }
    dW[e] = acc & m;
  }
}

__global__ void k_pool2(int op, const uint64_t* __restrict__ in, int64_t bc, int H, int W, uint64_t m,
                        uint64_t* __restrict__ out) {
  // op 0: in (bc, H, W) -> out (bc, H/2, W/2) window sums; op 1: in (bc, H/2, W/2) -> out (bc, H, W)
  const int h2 = H / 2, w2 = W / 2;
  const int64_t total = op == 0 ? bc * h2 * w2 : bc * H * W;
  if (total < (1ll << 31)) {  // 32-bit index arithmetic (64-bit division dominated the kernel)
    const uint32_t t32 = (uint32_t)total, hw2 = (uint32_t)(h2 * w2), hw = (uint32_t)(H * W);
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < t32; e += gridDim.x * blockDim.x) {
      if (op == 0) {
        const uint32_t q = e / hw2, r = e - q * hw2, y = r / (uint32_t)w2, x = r - y * (uint32_t)w2;
        const uint64_t* ip = in + (uint64_t)q * hw + (2 * y) * (uint32_t)W + 2 * x;
        out[e] = (ip[0] + ip[1] + ip[W] + ip[W + 1]) & m;
      } else {
        const uint32_t q = e / hw, r = e - q * hw, y = r / (uint32_t)W, x = r - y * (uint32_t)W;
        out[e] = in[(uint64_t)q * hw2 + (y / 2) * (uint32_t)w2 + x / 2] & m;
      }
    }
    return;
  }
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    if (op == 0) {
      const int x = (int)(e % w2), y = (int)((e / w2) % h2);
      const int64_t q = e / ((int64_t)w2 * h2);
      const uint64_t* ip = in + q * H * W + (int64_t)(2 * y) * W + 2 * x;
      out[e] = (ip[0] + ip[1] + ip[W] + ip[W + 1]) & m;
    } else {
      const int x = (int)(e % W), y = (int)((e / W) % H);
      const int64_t q = e / ((int64_t)W * H);
      out[e] = in[q * h2 * w2 + (int64_t)(y / 2) * w2 + x / 2] & m;
    }
  }
}

// ---------------------------------------------------------- implicit GEMM ---
// The three operators as one tiled u64 GEMM  out[m][n] = sum_k A[m][k] B[k][n]
// with A / B gathered on the fly (no im2col buffer):
//   FWD    m = o,  n = (b,y,x) of Y,  k = (c,i,j):  A = W[o,c,i,j],  B = X[b,c,y*st+i-p,x*st+j-p]
//   BWDX   m = c,  n = (b,y,x) of dX, k = (o,i,j):  A = W[o,c,i,j],  B = dY[b,o,(y+p-i)/st,(x+p-j)/st]
//   GRADW  m = o,  n = (c,i,j),       k = (b,y,x):  A = dY[b,o,y,x], B = X[b,c,y*st+i-p,x*st+j-p]
// CTA tile 64 x 64 x 16 through shared memory, 256 threads x (4 x 4) register
// accumulators; a u64 multiply-add is 3 IMAD-class instructions.  GRADW
// (K = B*oh*ow, small M*N) splits K over gridDim.z and accumulates with u64
// atomics (exact mod 2^64), then masks in a second pass.
struct ConvDims {
  int B, ci, co, H, W, p, st, oh, ow;
};

template <int S, int KIND>
struct ConvGemm {  // 32-bit index arithmetic (the launcher checks every tensor has < 2^31 elements)
  using Dims = ConvDims;
  static constexpr int SS = S * S;
  __device__ __forceinline__ static void mnk(const ConvDims& d, int& M, int& N, int& K) {
    if (KIND == PB_CONV_FWD) { M = d.co; N = d.B * d.oh * d.ow; K = d.ci * SS; }
    else if (KIND == PB_CONV_BWDX) { M = d.ci; N = d.B * d.H * d.W; K = d.co * SS; }
    else { M = d.co; N = d.ci * SS; K = d.B * d.oh * d.ow; }
  }
  __device__ __forceinline__ static uint64_t a_at(const ConvDims& d, const uint64_t* A, int m, int k) {
    if (KIND == PB_CONV_FWD) return __ldg(A + (size_t)m * (d.ci * SS) + k);
    if (KIND == PB_CONV_BWDX) {  // k = (o, i, j)
      const int o = k / SS, r = k - o * SS;
      return __ldg(A + (size_t)(o * d.ci + m) * SS + r);
    }
    const unsigned hw = (unsigned)(d.oh * d.ow);  // GRADW: k = (b, y, x) of dY, m = o
    const unsigned b = (unsigned)k / hw, r = (unsigned)k - b * hw;
    return __ldg(A + (size_t)(b * d.co + m) * hw + r);
  }
  __device__ __forceinline__ static uint64_t b_at(const ConvDims& d, const uint64_t* Bm, int k, int n) {
    if (KIND == PB_CONV_FWD || KIND == PB_CONV_GRADW) {
      const int kc = KIND == PB_CONV_FWD ? k : n;  // (c,i,j)
      const unsigned kp = (unsigned)(KIND == PB_CONV_FWD ? n : k);  // (b,y,x)
      const int c = kc / SS, r = kc - c * SS, i = r / S, j = r - i * S;
      const unsigned hw = (unsigned)(d.oh * d.ow), ow = (unsigned)d.ow;
      const unsigned b = kp / hw, q = kp - b * hw, y = q / ow, x = q - y * ow;
      const int yy = (int)y * d.st + i - d.p, xx = (int)x * d.st + j - d.p;
      if (yy < 0 || yy >= d.H || xx < 0 || xx >= d.W) return 0ull;
      return __ldg(Bm + ((size_t)(b * d.ci + c) * d.H + yy) * d.W + xx);
    }
    const int o = k / SS, r = k - o * SS, i = r / S, j = r - i * S;  // BWDX: k = (o,i,j), n = (b,y,x) of dX
    const unsigned hw = (unsigned)(d.H * d.W), Wd = (unsigned)d.W;
    const unsigned b = (unsigned)n / hw, q = (unsigned)n - b * hw, y = q / Wd, x = q - y * Wd;
    const int u = (int)y + d.p - i, v = (int)x + d.p - j;
    if (u < 0 || v < 0) return 0ull;
    const unsigned yy = (unsigned)u / (unsigned)d.st, xx = (unsigned)v / (unsigned)d.st;
    if (yy * d.st != (unsigned)u || xx * d.st != (unsigned)v || yy >= (unsigned)d.oh || xx >= (unsigned)d.ow)
      return 0ull;
    return __ldg(Bm + ((size_t)(b * d.co + o) * d.oh + yy) * d.ow + xx);
  }
  __device__ __forceinline__ static size_t out_at(const ConvDims& d, int m, int n) {
    if (KIND == PB_CONV_FWD) {
      const unsigned hw = (unsigned)(d.oh * d.ow), b = (unsigned)n / hw, q = (unsigned)n - b * hw;
      return (size_t)(b * d.co + m) * hw + q;
    }
    if (KIND == PB_CONV_BWDX) {
      const unsigned hw = (unsigned)(d.H * d.W), b = (unsigned)n / hw, q = (unsigned)n - b * hw;
      return (size_t)(b * d.ci + m) * hw + q;
    }
    return (size_t)m * (d.ci * SS) + n;
  }
};

// K:206-218 matmul_wrap as the same tiled GEMM: out (n x m) = A (n x k) B (k x m),
// A / B optionally stored transposed (trans_a: A read as (k x n), trans_b: B as (m x k)).
struct MatDims {
  int n, k, m, ta, tb;
};
struct MatGemm {
  using Dims = MatDims;
  __device__ __forceinline__ static void mnk(const MatDims& d, int& M, int& N, int& K) { M = d.n; N = d.m; K = d.k; }
  __device__ __forceinline__ static uint64_t a_at(const MatDims& d, const uint64_t* A, int i, int kk) {
    return __ldg(A + (d.ta ? (size_t)kk * d.n + i : (size_t)i * d.k + kk));
  }
  __device__ __forceinline__ static uint64_t b_at(const MatDims& d, const uint64_t* B, int kk, int j) {
    return __ldg(B + (d.tb ? (size_t)j * d.k + kk : (size_t)kk * d.m + j));
  }
  __device__ __forceinline__ static size_t out_at(const MatDims& d, int i, int j) { return (size_t)i * d.m + j; }
};

template <class G>
__global__ void __launch_bounds__(256) k_gemm(typename G::Dims d, const uint64_t* __restrict__ A,
                                              const uint64_t* __restrict__ Bm, int64_t k_per_split, uint64_t m,
                                              uint64_t* __restrict__ out) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ uint64_t As[BK][BM];
  __shared__ uint64_t Bs[BK][BN + 1];
  int M, N, K;
  G::mnk(d, M, N, K);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kb = (int)(blockIdx.z * k_per_split), ke = min(K, kb + (int)k_per_split);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  uint64_t acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  // load assignment: A tile element (k = tid & 15, m = (tid >> 4) + 16 r); B tile (k = tid >> 6 + 4 r, n = tid & 63)
  const int la_k = tid & 15, la_m = tid >> 4;
  const int lb_n = tid & 63, lb_k = tid >> 6;
  for (int k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int mm = m0 + la_m + 16 * r, kk = k0 + la_k;
      As[la_k][la_m + 16 * r] = (mm < M && kk < ke) ? G::a_at(d, A, mm, kk) : 0ull;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int kk = k0 + lb_k + 4 * r, nn = n0 + lb_n;
      Bs[lb_k + 4 * r][lb_n] = (nn < N && kk < ke) ? G::b_at(d, Bm, kk, nn) : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      uint64_t a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int mm = m0 + ty + 16 * i;
    if (mm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int nn = n0 + tx + 16 * j;
      if (nn >= N) continue;
      const size_t o = G::out_at(d, mm, nn);
      if (gridDim.z == 1) out[o] = acc[i][j] & m;
      else atomicAdd(reinterpret_cast<unsigned long long*>(out + o), (unsigned long long)acc[i][j]);
    }
  }
}

// Skinny GEMMs (M <= 16 rows: the few-channel convolutions of the MNIST CNNs,
// 1x1 convolutions into 16 channels): one thread per output column holding
// all MM row accumulators, the A chunk (MM x 32, zero-padded rows) staged in
// shared memory and broadcast, one B gather per (k, column) feeding MM MACs
// -- instead of a 64 x 64 tile whose rows sit >= 75 % idle.  Split-K over
// gridDim.z with u64 atomics as k_gemm.
__global__ void k_mask_inplace(uint64_t* v, int64_t n, uint64_t m);
constexpr int SK_T = 128, SK_KT = 32;
template <int KIND, int S, int MM>
__global__ void __launch_bounds__(SK_T) k_gemm_skinny(GemmMap gm, ConvDims d, const uint64_t* __restrict__ A,
                                                      const uint64_t* __restrict__ Bm, int64_t k_per_split,
                                                      uint64_t m, uint64_t* __restrict__ out) {
  using G = ConvGemm<S, KIND>;
  __shared__ uint64_t As[MM][SK_KT];
  int M, N, K;
  G::mnk(d, M, N, K);
  const int n = blockIdx.x * SK_T + threadIdx.x;
  const int kb = (int)(blockIdx.z * k_per_split), ke = min(K, kb + (int)k_per_split);
  uint64_t acc[MM];
#pragma unroll
  for (int i = 0; i < MM; ++i) acc[i] = 0;
  Gather<KIND, S, 1> g;  // this column's operand, walked along k without divisions
  if (n < N) g.init(gm, Bm, n, kb);
  for (int k0 = kb; k0 < ke; k0 += SK_KT) {
    for (int e = threadIdx.x; e < MM * SK_KT; e += SK_T) {
      const int i = e / SK_KT, kk = e - i * SK_KT;
      As[i][kk] = (i < M && k0 + kk < ke) ? G::a_at(d, A, i, k0 + kk) : 0ull;
    }
    __syncthreads();
    if (n < N) {
      const int kc = min(SK_KT, ke - k0);
#pragma unroll 4
      for (int kk = 0; kk < kc; ++kk) {
        const uint64_t b = g.next(gm);
#pragma unroll
        for (int i = 0; i < MM; ++i) acc[i] += As[i][kk] * b;
      }
    }
    __syncthreads();
  }
  if (n >= N) return;
#pragma unroll
  for (int i = 0; i < MM; ++i) {
    if (i >= M) break;
    const size_t o = G::out_at(d, i, n);
    if (gridDim.z == 1) out[o] = acc[i] & m;
    else atomicAdd(reinterpret_cast<unsigned long long*>(out + o), (unsigned long long)acc[i]);
  }
}

template <int KIND, int S>
void launch_skinny(const ConvDims& d, const uint64_t* A, const uint64_t* Bm, int64_t M, int64_t N, int64_t K,
                   uint64_t m, uint64_t* out, cudaStream_t st) {
  const GemmMap gm{KIND, d.B, d.ci, d.co, d.H, d.W, S, d.p, d.st, d.oh, d.ow, 0, 0, 0, 0, 0};
  const int64_t tiles = (N + SK_T - 1) / SK_T;
  int splits = 1;
  while (tiles * splits < 2 * 148 * 4 && K / (splits * 2) >= 16) splits *= 2;
  const int64_t kps = ((K + splits - 1) / splits + SK_KT - 1) / SK_KT * SK_KT;
  const dim3 grid((unsigned)tiles, 1, (unsigned)splits);
  if (splits > 1) cudaMemsetAsync(out, 0, (size_t)(M * N) * sizeof(uint64_t), st);
  if (M <= 8) k_gemm_skinny<KIND, S, 8><<<grid, SK_T, 0, st>>>(gm, d, A, Bm, kps, m, out);
  else k_gemm_skinny<KIND, S, 16><<<grid, SK_T, 0, st>>>(gm, d, A, Bm, kps, m, out);
  if (splits > 1) k_mask_inplace<<<pb_grid_1d(M * N, 256), 256, 0, st>>>(out, M * N, m);
}

__global__ void k_mask_inplace(uint64_t* v, int64_t n, uint64_t m) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] &= m;
}

template <int S>
int conv_gemm_launch(int kind, const ConvDims& d, const uint64_t* a, const uint64_t* b, uint64_t m, uint64_t* out,
                     cudaStream_t st) {
  int64_t M, N, K;
  if (kind == PB_CONV_FWD) { M = d.co; N = (int64_t)d.B * d.oh * d.ow; K = (int64_t)d.ci * S * S; }
  else if (kind == PB_CONV_BWDX) { M = d.ci; N = (int64_t)d.B * d.H * d.W; K = (int64_t)d.co * S * S; }
  else { M = d.co; N = (int64_t)d.ci * S * S; K = (int64_t)d.B * d.oh * d.ow; }
  if (M <= 16) {  // few output channels (or input channels for the input gradient)
    if (kind == PB_CONV_FWD) launch_skinny<PB_CONV_FWD, S>(d, b, a, M, N, K, m, out, st);
    else if (kind == PB_CONV_BWDX) launch_skinny<PB_CONV_BWDX, S>(d, b, a, M, N, K, m, out, st);
    else launch_skinny<PB_CONV_GRADW, S>(d, b, a, M, N, K, m, out, st);
    return 0;
  }
  const int64_t tiles = ((M + 63) / 64) * ((N + 63) / 64);
  // split K until ~2 waves of 3 resident CTAs per SM are filled (GRADW has a tiny
  // M x N and K = B*oh*ow; the forward / input-gradient GEMMs of a 64-channel
  // layer have only 256 tiles) while keeping >= 128 K per split
  int splits = 1;
  while (tiles * splits < 2 * 148 * 3 && K / (splits * 2) >= 128) splits *= 2;
  const int64_t kps = ((K + splits - 1) / splits + 15) / 16 * 16;
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64), (unsigned)splits);
  if (splits > 1) cudaMemsetAsync(out, 0, (size_t)(M * N) * sizeof(uint64_t), st);
  if (kind == PB_CONV_FWD) k_gemm<ConvGemm<S, PB_CONV_FWD>><<<grid, 256, 0, st>>>(d, b, a, kps, m, out);  // A = W, B = X
  else if (kind == PB_CONV_BWDX) k_gemm<ConvGemm<S, PB_CONV_BWDX>><<<grid, 256, 0, st>>>(d, b, a, kps, m, out);  // A = W, B = dY
  else k_gemm<ConvGemm<S, PB_CONV_GRADW>><<<grid, 256, 0, st>>>(d, b, a, kps, m, out);  // A = dY, B = X
  if (splits > 1) k_mask_inplace<<<pb_grid_1d(M * N, 256), 256, 0, st>>>(out, M * N, m);
  return 0;
}

}  // namespace

int pb_tc_conv(int kind, const uint64_t* a, const uint64_t* b, int B, int ci, int co, int H, int W, int s, int p,
               int st_, int oh, int ow, int ell, uint64_t* out, cudaStream_t st);
int pb_tc_matmul(const uint64_t* a, const uint64_t* b, int n, int k, int m, int ta, int tb, int ell, uint64_t* out,
                 cudaStream_t st);

// Backend choice is a function of the shape alone (no environment switch, no
// fallback): ring GEMMs of >= 2^26 u64 MACs and convolutions of >= 2^24
// run on the tcgen05 int8 tensor cores (pb_tc.cu; the fused implicit-GEMM
// conv has no plane pass, so it wins down to CIFAR conv4's 2^24: 27 vs
// 29-33 us), conv weight gradients (skinny outputs, long K: the CUDA-core
// tiles need split-K atomics) from 2^22 (conv5 32 vs 57 us); smaller ones on
// the u64 CUDA-core kernels (profiles/r02_ring_gemm_backends.jsonl).
// pb_ring_conv_ex / pb_ring_matmul_ex take the backend explicitly (the
// parity tests run every backend on every shape).
// Convolutions with <= 16 output rows (M: output channels, input channels for
// the input gradient -- the MNIST CNNs' 1- and 5-channel layers, 1x1 convs
// into 16 channels) run on the CUDA-core skinny kernel (k_gemm_skinny) at any
// size; other skinny ones (an output side < 32) on the tensor cores, where
// the 64 x 64 CUDA-core tiles would leave most rows idle.
static int auto_backend(int kind, int64_t macs, int64_t side_m = 1 << 30, int64_t side_n = 1 << 30) {
  if (kind >= 0 && side_m <= 16) return PB_BACKEND_CUDA_CORE;
  if (kind >= 0 && (side_m < 32 || side_n < 32)) return PB_BACKEND_TENSOR;
  const int64_t min_macs = kind == PB_CONV_GRADW ? (1ll << 22) : kind >= 0 ? (1ll << 24) : (1ll << 26);
  return macs >= min_macs ? PB_BACKEND_TENSOR : PB_BACKEND_CUDA_CORE;
}

extern "C" int pb_ring_conv(int kind, const uint64_t* a, const uint64_t* b, int32_t B, int32_t c_i, int32_t c_o,
                            int32_t H, int32_t W, int32_t s, int32_t pad, int32_t stride, int32_t ell, uint64_t* out,
                            void* stream) {
  return pb_ring_conv_ex(kind, a, b, B, c_i, c_o, H, W, s, pad, stride, ell, out, PB_BACKEND_AUTO, stream);
}

extern "C" int pb_ring_conv_ex(int kind, const uint64_t* a, const uint64_t* b, int32_t B, int32_t c_i, int32_t c_o,
                               int32_t H, int32_t W, int32_t s, int32_t pad, int32_t stride, int32_t ell, uint64_t* out,
                               int32_t backend, void* stream) {
  if (!a || !b || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (B < 1 || c_i < 1 || c_o < 1 || s < 1 || pad < 0 || stride < 1 || H + 2 * pad < s || W + 2 * pad < s)
    return pb_set_error(PB_ERR_GEOMETRY, "bad conv geometry");
  if (ell < 2 || ell > 64) return pb_set_error(PB_ERR_ARG, "bad ell");
  const int oh = (H + 2 * pad - s) / stride + 1, ow = (W + 2 * pad - s) / stride + 1;
  const uint64_t m = cmask(ell);
  cudaStream_t st = pb_stream_of(stream);
  if (kind < PB_CONV_FWD || kind > PB_CONV_GRADW) return pb_set_error(PB_ERR_ARG, "bad conv kind");
  const ConvDims d{B, c_i, c_o, H, W, pad, stride, oh, ow};
  const int64_t big = (int64_t)B * (c_i > c_o ? c_i : c_o) * (H > oh ? H : oh) * (W > ow ? W : ow);
  if (big >= (1ll << 31) || (int64_t)c_o * c_i * s * s >= (1ll << 31))
    return pb_set_error(PB_ERR_GEOMETRY, "conv tensor too large for 32-bit indexing");
  if (backend < PB_BACKEND_AUTO || backend > PB_BACKEND_TENSOR) return pb_set_error(PB_ERR_ARG, "bad backend");
  if (backend == PB_BACKEND_AUTO) {
    const int64_t side_m = kind == PB_CONV_BWDX ? c_i : c_o;
    const int64_t side_n = kind == PB_CONV_FWD ? (int64_t)B * oh * ow
                         : kind == PB_CONV_BWDX ? (int64_t)B * H * W : (int64_t)c_i * s * s;
    backend = auto_backend(kind, (int64_t)B * c_o * c_i * s * s * oh * ow, side_m, side_n);
  }
  if (backend == PB_BACKEND_TENSOR) return pb_tc_conv(kind, a, b, B, c_i, c_o, H, W, s, pad, stride, oh, ow, ell, out, st);
  switch (s) {  // tiled implicit GEMM for the kernel sizes the models use
    case 1: conv_gemm_launch<1>(kind, d, a, b, m, out, st); PB_CHECK_LAUNCH(); return PB_OK;
    case 3: conv_gemm_launch<3>(kind, d, a, b, m, out, st); PB_CHECK_LAUNCH(); return PB_OK;
    case 5: conv_gemm_launch<5>(kind, d, a, b, m, out, st); PB_CHECK_LAUNCH(); return PB_OK;
    default: break;
  }
  switch (kind) {
    case PB_CONV_FWD: {
      const int64_t n = (int64_t)B * c_o * oh * ow;
      k_conv_fwd<<<pb_grid_1d(n, 256), 256, 0, st>>>(a, b, B, c_i, c_o, H, W, s, pad, stride, oh, ow, m, out);
      break;
    }
    case PB_CONV_BWDX: {
      const int64_t n = (int64_t)B * c_i * H * W;
      k_conv_bwdx<<<pb_grid_1d(n, 256), 256, 0, st>>>(a, b, B, c_i, c_o, H, W, s, pad, stride, oh, ow, m, out);
      break;
    }
    case PB_CONV_GRADW: {
      const unsigned g = (unsigned)((int64_t)c_o * c_i);
#define PB_GW(S) k_conv_gradw<S><<<g, 256, 0, st>>>(a, b, B, c_i, c_o, H, W, pad, stride, oh, ow, m, out)
      switch (s) {
        case 1: PB_GW(1); break;
        case 2: PB_GW(2); break;
        case 3: PB_GW(3); break;
        case 5: PB_GW(5); break;
        default: {
          const int64_t n = (int64_t)c_o * c_i * s * s;
          k_conv_gradw_any<<<pb_grid_1d(n, 128), 128, 0, st>>>(a, b, B, c_i, c_o, H, W, s, pad, stride, oh, ow, m,
                                                                out);
        }
      }
#undef PB_GW
      break;
    }
    default:
      return pb_set_error(PB_ERR_ARG, "bad conv kind");
  }
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_pool2(int op, const uint64_t* in, int64_t bc, int32_t H, int32_t W, int32_t ell, uint64_t* out,
                        void* stream) {
  if (!in || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (op != PB_POOL_SUM && op != PB_POOL_REPLICATE) return pb_set_error(PB_ERR_ARG, "bad pool op");
  if (H < 2 || W < 2 || (H & 1) || (W & 1)) return pb_set_error(PB_ERR_GEOMETRY, "avgpool2 needs even spatial dims");
  if (ell < 2 || ell > 64) return pb_set_error(PB_ERR_ARG, "bad ell");
  if (bc <= 0) return PB_OK;
  const int64_t n = op == PB_POOL_SUM ? bc * (H / 2) * (W / 2) : bc * H * W;
  k_pool2<<<pb_grid_1d(n, 256), 256, 0, pb_stream_of(stream)>>>(op, in, bc, H, W, cmask(ell), out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

void pb_launch_ring_matmul_small(const uint64_t* a, const uint64_t* b, int64_t n, int64_t k, int64_t m, int trans_a,
                                 int trans_b, const uint64_t* c, int sign, uint64_t mask, uint64_t* out,
                                 cudaStream_t st);

// out = c + sign * (a b) mod 2^ell: the small shapes fuse the add into the
// GEMM epilogue; larger ones run pb_ring_matmul then one elementwise kernel.
extern "C" int pb_ring_matmul_add(const uint64_t* a, const uint64_t* b, int64_t n, int64_t k, int64_t m, int trans_a,
                                  int trans_b, const uint64_t* c, int32_t sign, int32_t ell, uint64_t* out,
                                  void* stream) {
  if (!c || sign == 0) return pb_ring_matmul(a, b, n, k, m, trans_a, trans_b, ell, out, stream);
  if (n > 0 && m > 0 && k > 0 && (!a || !b || !out)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (n <= 0 || m <= 0) return PB_OK;
  if (k < 0 || n * k >= (1ll << 31) || k * m >= (1ll << 31) || n * m >= (1ll << 31))
    return pb_set_error(PB_ERR_SHAPE, "bad matmul shape");
  const uint64_t mask = (ell >= 64 || ell <= 0) ? ~0ull : ((1ull << ell) - 1);
  cudaStream_t st = pb_stream_of(stream);
  if (n * k * m < (1ll << 24)) {
    pb_launch_ring_matmul_small(a, b, n, k, m, trans_a, trans_b, c, sign, mask, out, st);
    PB_CHECK_LAUNCH();
    return PB_OK;
  }
  if (c == out) return pb_set_error(PB_ERR_ARG, "large shapes need out != c");
  if (int s = pb_ring_matmul(a, b, n, k, m, trans_a, trans_b, ell, out, stream)) return s;
  return pb_ring_binary(sign > 0 ? PB_RING_ADD : PB_RING_SUB, out, c, out, n * m, n * m, ell, stream);
}

extern "C" int pb_ring_matmul(const uint64_t* a, const uint64_t* b, int64_t n, int64_t k, int64_t m, int trans_a,
                              int trans_b, int32_t ell, uint64_t* out, void* stream) {
  return pb_ring_matmul_ex(a, b, n, k, m, trans_a, trans_b, ell, out, PB_BACKEND_AUTO, stream);
}

extern "C" int pb_ring_matmul_ex(const uint64_t* a, const uint64_t* b, int64_t n, int64_t k, int64_t m, int trans_a,
                                 int trans_b, int32_t ell, uint64_t* out, int32_t backend, void* stream) {
  if (n > 0 && m > 0 && k > 0 && (!a || !b || !out)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (n <= 0 || m <= 0) return PB_OK;
  if (k < 0 || n * k >= (1ll << 31) || k * m >= (1ll << 31) || n * m >= (1ll << 31))
    return pb_set_error(PB_ERR_SHAPE, "bad matmul shape");
  const uint64_t mask = (ell >= 64 || ell <= 0) ? ~0ull : ((1ull << ell) - 1);
  cudaStream_t st = pb_stream_of(stream);
  if (k == 0) {
    cudaMemsetAsync(out, 0, (size_t)(n * m) * sizeof(uint64_t), st);
    return PB_OK;
  }
  if (backend < PB_BACKEND_AUTO || backend > PB_BACKEND_TENSOR) return pb_set_error(PB_ERR_ARG, "bad backend");
  if (backend == PB_BACKEND_AUTO) backend = auto_backend(-1, n * k * m);
  if (backend == PB_BACKEND_TENSOR)
    return pb_tc_matmul(a, b, (int)n, (int)k, (int)m, trans_a, trans_b, ell, out, st);
  if (n * k * m < (1ll << 24)) {  // the FC layers' local terms: one small launch beats tiles + split-K passes
    pb_launch_ring_matmul_small(a, b, n, k, m, trans_a, trans_b, nullptr, 0, mask, out, st);
    PB_CHECK_LAUNCH();
    return PB_OK;
  }
  const MatDims d{(int)n, (int)k, (int)m, trans_a ? 1 : 0, trans_b ? 1 : 0};
  const int64_t tiles = ((n + 63) / 64) * ((m + 63) / 64);
  int splits = 1;  // split the contraction to fill the GPU (the FC weight gradients have small n x m, large k)
  while (tiles * splits < 2 * 148 * 3 && k / (splits * 2) >= 128) splits *= 2;
  const int64_t kps = ((k + splits - 1) / splits + 15) / 16 * 16;
  dim3 grid((unsigned)((m + 63) / 64), (unsigned)((n + 63) / 64), (unsigned)splits);
  if (splits > 1) cudaMemsetAsync(out, 0, (size_t)(n * m) * sizeof(uint64_t), st);
  k_gemm<MatGemm><<<grid, 256, 0, st>>>(d, a, b, kps, mask, out);
  if (splits > 1) k_mask_inplace<<<pb_grid_1d(n * m, 256), 256, 0, st>>>(out, n * m, mask);
  PB_CHECK_LAUNCH();
  return PB_OK;
}
