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

}  // namespace

extern "C" int pb_ring_conv(int kind, const uint64_t* a, const uint64_t* b, int32_t B, int32_t c_i, int32_t c_o,
                            int32_t H, int32_t W, int32_t s, int32_t pad, int32_t stride, int32_t ell, uint64_t* out,
                            void* stream) {
  if (!a || !b || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (B < 1 || c_i < 1 || c_o < 1 || s < 1 || pad < 0 || stride < 1 || H + 2 * pad < s || W + 2 * pad < s)
    return pb_set_error(PB_ERR_GEOMETRY, "bad conv geometry");
  if (ell < 2 || ell > 64) return pb_set_error(PB_ERR_ARG, "bad ell");
  const int oh = (H + 2 * pad - s) / stride + 1, ow = (W + 2 * pad - s) / stride + 1;
  const uint64_t m = cmask(ell);
  cudaStream_t st = pb_stream_of(stream);
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
