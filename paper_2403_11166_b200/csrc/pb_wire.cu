// pb_wire.cu — the PBFV ciphertext/plaintext wire format on the
// device: serialization straight into the frame buffer (device memory or
// pinned host memory, which with UVA fuses the D2H copy into the kernel) and
// validating deserialization back into device-order residue rows.
//
// Frame (little-endian, packed): magic "PBFV", version u16, N u32,
// L u8, form u8 (12 bytes), then n_polys x L x N u64 residues, c0 rows then
// c1 rows for a ciphertext, one row block for a plaintext.  form 0 =
// coefficient rows, 1 = NTT rows in the reference's bit-reversed order (what
// K:ntt_forward produces; the device order is converted inside the kernel).
//
// Bound: HBM (or the host link for a pinned destination) — 4 bytes read and
// 8 bytes written per residue; one CTA per L x N row, the row staged in
// shared memory so both the device-order gather and the 16-byte stores stay
// coalesced whatever the frame's 4-byte alignment.
#include "pb_common.cuh"

namespace {

constexpr uint32_t kWireMagic = 0x56464250u;  // bytes 'P' 'B' 'F' 'V'
constexpr uint32_t kWireVersion = PB_WIRE_VERSION;

__device__ __forceinline__ int ref_to_dev(int i, int T) {  // reference index -> device address
  return ((i & 31) >> 2) * 4 * T + (i >> 5) * 4 + (i & 3);
}
// Shared-memory index of device address a: each of the 8 segments of N/8
// words (the v of the device order) is padded by 4 words, so the
// reference-order gather/scatter (a warp spans all 8 segments at one
// offset) hits 32 distinct banks instead of 4.
__device__ __forceinline__ int padded(int a, int ls) { return a + ((a >> ls) << 2); }

__global__ void __launch_bounds__(256) k_wire_serialize(PbDev P, const uint32_t* __restrict__ polys, int64_t n_rows,
                                                        int rows_per_frame, int form, int reorder,
                                                        int64_t frame_bytes, uint8_t* __restrict__ out) {
  extern __shared__ uint4 sm4[];
  const uint32_t* sm = reinterpret_cast<const uint32_t*>(sm4);
  const int N = P.N, T = N >> 5, ls = reorder ? P.logN - 3 : 30;
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    const int64_t p = r / rows_per_frame;
    const int rr = (int)(r - p * rows_per_frame);
    const uint4* src = reinterpret_cast<const uint4*>(polys + r * N);
    for (int i = threadIdx.x; i < N / 4; i += blockDim.x) sm4[padded(4 * i, ls) >> 2] = __ldg(src + i);
    __syncthreads();
    uint8_t* fbase = out + p * frame_bytes;
    if (rr == 0 && threadIdx.x == 0) {
      uint32_t* h = reinterpret_cast<uint32_t*>(fbase);
      h[0] = kWireMagic;
      h[1] = kWireVersion | ((uint32_t)N << 16);
      h[2] = ((uint32_t)N >> 16) | ((uint32_t)P.L << 16) | ((uint32_t)form << 24);
    }
    // The row as 2N u32 words: word 2i = residue of reference index i, 2i+1 = 0.
    uint32_t* w = reinterpret_cast<uint32_t*>(fbase + 12 + (int64_t)rr * N * 8);
    auto word = [&](int j) -> uint32_t {
      if (j & 1) return 0u;
      const int i = j >> 1;
      return sm[padded(reorder ? ref_to_dev(i, T) : i, ls)];
    };
    const int mis = (int)((reinterpret_cast<uintptr_t>(w) & 15) >> 2);
    const int pro = mis ? 4 - mis : 0;
    if (threadIdx.x < pro) w[threadIdx.x] = word(threadIdx.x);
    const int nvec = (2 * N - pro) >> 2;
    uint4* wv = reinterpret_cast<uint4*>(w + pro);
    for (int k = threadIdx.x; k < nvec; k += blockDim.x) {
      const int j = pro + 4 * k;
      wv[k] = make_uint4(word(j), word(j + 1), word(j + 2), word(j + 3));
    }
    const int tail0 = pro + 4 * nvec;
    if (threadIdx.x < 2 * N - tail0) w[tail0 + threadIdx.x] = word(tail0 + threadIdx.x);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_wire_deserialize(PbDev P, const uint8_t* __restrict__ in, int64_t n_rows,
                                                          int rows_per_frame, int form, int reorder,
                                                          int64_t frame_bytes, uint32_t* __restrict__ polys,
                                                          int32_t* bad) {
  extern __shared__ uint4 sm4[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(sm4);
  const int N = P.N, T = N >> 5, ls = reorder ? P.logN - 3 : 30;
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    const int64_t p = r / rows_per_frame;
    const int rr = (int)(r - p * rows_per_frame);
    const uint8_t* fbase = in + p * frame_bytes;
    if (rr == 0 && threadIdx.x == 0) {
      const uint32_t* h = reinterpret_cast<const uint32_t*>(fbase);
      int32_t f = 0;
      if (h[0] != kWireMagic || (h[1] & 0xffffu) != kWireVersion) f |= PB_WIRE_BAD_HEADER;
      const uint32_t n = (h[1] >> 16) | ((h[2] & 0xffffu) << 16);
      if (n != (uint32_t)N || ((h[2] >> 16) & 0xffu) != (uint32_t)P.L) f |= PB_WIRE_BAD_PARAMS;
      if ((int)(h[2] >> 24) != form) f |= PB_WIRE_BAD_FORM;
      if (f) atomicOr(bad, f);
    }
    const uint32_t* w = reinterpret_cast<const uint32_t*>(fbase + 12 + (int64_t)rr * N * 8);
    const uint32_t q = P.q[rr % P.L];
    int out_of_range = 0;
    // 8-byte loads either way: an 8-aligned row reads (lo_i, hi_i) pairs; a
    // row at 4 mod 8 (every other frame) reads (hi_{i-1}, lo_i) from one word
    // earlier and checks its last high word separately.
    // kU loads in flight per thread before any is consumed (the kernel is
    // load-latency bound otherwise: ncu long_scoreboard 82%).
    constexpr int kU = 8;
    const bool al8 = (reinterpret_cast<uintptr_t>(w) & 7) == 0;
    const uint2* w2 = reinterpret_cast<const uint2*>(al8 ? w : w - 1);
    for (int i0 = threadIdx.x; i0 < N; i0 += kU * blockDim.x) {
      uint2 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * blockDim.x;
        v[u] = i < N ? w2[i] : make_uint2(0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i >= N) break;
        const uint32_t lo = al8 ? v[u].x : v[u].y, hi = al8 ? v[u].y : (i > 0 ? v[u].x : 0u);
        out_of_range |= (hi != 0u) | (lo >= q);
        sm[padded(reorder ? ref_to_dev(i, T) : i, ls)] = lo;
      }
    }
    if (!al8 && threadIdx.x == 0) out_of_range |= w[2 * N - 1] != 0u;
    if (__syncthreads_or(out_of_range) && threadIdx.x == 0) atomicOr(bad, PB_WIRE_BAD_RESIDUE);
    uint32_t* dst = polys + r * N;
    for (int a = threadIdx.x; a < N; a += blockDim.x) dst[a] = sm[padded(a, ls)];
    __syncthreads();
  }
}

int wire_geometry(const pb_ctx* ctx, int64_t P, int32_t n_polys, int32_t form, int64_t* frame_bytes) {
  if (!ctx) return pb_set_error(PB_ERR_ARG, "null context");
  if (P < 0 || n_polys < 1 || n_polys > 2) return pb_set_error(PB_ERR_SHAPE, "PBFV frames hold 1 or 2 polynomials");
  if (form != PB_WIRE_COEFF && form != PB_WIRE_NTT) return pb_set_error(PB_ERR_FORM, "unknown PBFV form");
  *frame_bytes = PB_WIRE_FRAME_SIZE(ctx->dev.N, ctx->dev.L, n_polys);
  return PB_OK;
}

int wire_grid(int64_t n_rows) {
  const int64_t cap = 148 * 8;
  return (int)(n_rows < cap ? n_rows : cap);
}

}  // namespace

extern "C" int pb_wire_frame_bytes(const pb_ctx* ctx, int32_t n_polys, int64_t* out_host) {
  if (!out_host) return pb_set_error(PB_ERR_ARG, "null output");
  return wire_geometry(ctx, 0, n_polys, PB_WIRE_NTT, out_host);
}

extern "C" int pb_wire_serialize(const pb_ctx* ctx, const uint32_t* polys, int64_t P, int32_t n_polys, int32_t form,
                                 uint8_t* out, void* stream) {
  int64_t fb = 0;
  int s = wire_geometry(ctx, P, n_polys, form, &fb);
  if (s) return s;
  if (P == 0) return PB_OK;
  if (!polys || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if ((reinterpret_cast<uintptr_t>(polys) & 15) || (reinterpret_cast<uintptr_t>(out) & 3))
    return pb_set_error(PB_ERR_ARG, "polys must be 16-byte and out 4-byte aligned");
  const int N = ctx->dev.N;
  const size_t smem = (size_t)N * 4 + 8 * 4 * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_wire_serialize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t n_rows = P * n_polys * ctx->dev.L;
  const int reorder = form == PB_WIRE_NTT && ctx->dev.logN >= 11;
  k_wire_serialize<<<wire_grid(n_rows), 256, smem, pb_stream_of(stream)>>>(ctx->dev, polys, n_rows,
                                                                          n_polys * ctx->dev.L, form, reorder, fb, out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_wire_deserialize(const pb_ctx* ctx, const uint8_t* in, int64_t P, int32_t n_polys, int32_t form,
                                   uint32_t* polys, int32_t* bad, void* stream) {
  int64_t fb = 0;
  int s = wire_geometry(ctx, P, n_polys, form, &fb);
  if (s) return s;
  if (!bad) return pb_set_error(PB_ERR_ARG, "null status word");
  cudaStream_t st = pb_stream_of(stream);
  cudaMemsetAsync(bad, 0, sizeof(int32_t), st);
  if (P == 0) {
    PB_CHECK_LAUNCH();
    return PB_OK;
  }
  if (!polys || !in) return pb_set_error(PB_ERR_ARG, "null argument");
  if (reinterpret_cast<uintptr_t>(in) & 3) return pb_set_error(PB_ERR_ARG, "in must be 4-byte aligned");
  const int N = ctx->dev.N;
  const size_t smem = (size_t)N * 4 + 8 * 4 * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_wire_deserialize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t n_rows = P * n_polys * ctx->dev.L;
  const int reorder = form == PB_WIRE_NTT && ctx->dev.logN >= 11;
  k_wire_deserialize<<<wire_grid(n_rows), 256, smem, st>>>(ctx->dev, in, n_rows, n_polys * ctx->dev.L, form, reorder,
                                                          fb, polys, bad);
  PB_CHECK_LAUNCH();
  return PB_OK;
}
