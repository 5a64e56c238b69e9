// pb_modswitch.cu — response compaction by modulus switching (SPEC:196:
// "dropping one RNS level before sending masked results back", OFF by
// default).  A ciphertext under Q = q_0..q_{L-1} becomes one under
// Q' = Q / q_{L-1}:  c'_i = (c_i - [c]_{q_{L-1}}) * q_{L-1}^-1 mod q_i, with
// [c]_{q_{L-1}} the centered coefficient-form residue of the dropped limb —
// the rounding of c * Q'/Q.  Everything stays in the NTT domain except the
// dropped limb's rows, which go through one inverse NTT (1-limb context),
// a centered lift into the L-1 remaining limbs and their forward NTT.
// Bound: HBM; per polynomial L rows read, L-1 rows written, plus the
// scratch rows the NTTs stream (L2-resident at reply sizes).
#include "pb_common.cuh"

namespace {

// x[p][i][n] = centered(a[p][n]) mod q_i, a in [0, q_last).  One CTA per
// polynomial (grid-stride), 16-byte loads and stores.
__device__ __forceinline__ uint32_t ms_center(uint32_t v, uint32_t q_last, uint32_t q) {
  const bool neg = v > (q_last >> 1);
  const uint32_t mag = neg ? q_last - v : v;  // |centered value| < q_last / 2
  const uint32_t r = mag >= q ? mag % q : mag;
  return (neg && r) ? q - r : r;
}

__global__ void __launch_bounds__(256) k_ms_lift(PbDev P, const uint32_t* __restrict__ a, uint32_t q_last,
                                                 int64_t n_polys, uint32_t* __restrict__ x) {
  const int N4 = P.N >> 2, L = P.L;
  for (int64_t p = blockIdx.x; p < n_polys; p += gridDim.x) {
    const uint4* a4 = reinterpret_cast<const uint4*>(a) + p * N4;
    uint4* x4 = reinterpret_cast<uint4*>(x) + p * L * N4;
    for (int k = threadIdx.x; k < N4; k += blockDim.x) {
      const uint4 v = a4[k];
      for (int i = 0; i < L; ++i) {
        const uint32_t q = P.q[i];
        x4[(int64_t)i * N4 + k] =
            make_uint4(ms_center(v.x, q_last, q), ms_center(v.y, q_last, q), ms_center(v.z, q_last, q),
                       ms_center(v.w, q_last, q));
      }
    }
  }
}

uint32_t inv_mod(uint32_t a, uint32_t m) {  // a^-1 mod m, gcd(a, m) = 1
  int64_t t = 0, nt = 1, r = m, nr = a % m;
  while (nr) {
    const int64_t qq = r / nr, tt = t - qq * nt, rr = r - qq * nr;
    t = nt, nt = tt, r = nr, nr = rr;
  }
  return (uint32_t)(t < 0 ? t + m : t);
}

struct MsConsts {
  uint32_t qinv[PB_MAXL], qinv_sh[PB_MAXL];
};

// out[p][i] = (c[p][i] - x[p][i]) * q_last^-1 mod q_i, x (NTT form) in place
// in out.  One CTA per output row (grid-stride), 16-byte accesses.
__device__ __forceinline__ uint32_t ms_fin(uint32_t cv, uint32_t xv, uint32_t w, uint32_t ws, uint32_t q) {
  return mul_shoup(cv >= xv ? cv - xv : cv + q - xv, w, ws, q);
}

__global__ void __launch_bounds__(256) k_ms_finish_v(PbDev P, const uint32_t* __restrict__ c, int c_limbs,
                                                     int64_t n_polys, MsConsts k, uint32_t* out) {
  const int N4 = P.N >> 2, L = P.L;
  for (int64_t row = blockIdx.x; row < n_polys * L; row += gridDim.x) {
    const int64_t p = row / L;
    const int i = (int)(row - p * L);
    const uint32_t q = P.q[i], w = k.qinv[i], ws = k.qinv_sh[i];
    const uint4* c4 = reinterpret_cast<const uint4*>(c) + (p * c_limbs + i) * N4;
    uint4* o4 = reinterpret_cast<uint4*>(out) + row * N4;
    for (int j = threadIdx.x; j < N4; j += blockDim.x) {
      const uint4 cv = c4[j], xv = o4[j];
      o4[j] = make_uint4(ms_fin(cv.x, xv.x, w, ws, q), ms_fin(cv.y, xv.y, w, ws, q), ms_fin(cv.z, xv.z, w, ws, q),
                         ms_fin(cv.w, xv.w, w, ws, q));
    }
  }
}

int ms_rows_grid(int64_t rows) {  // one CTA per row, up to 8 resident per SM
  const int64_t cap = 148 * 8;
  return (int)(rows < cap ? rows : cap);
}

}  // namespace

extern "C" int pb_mod_switch_drop(const pb_ctx* ctx_low, const pb_ctx* ctx_last, const uint32_t* ct, int64_t n_polys,
                                  uint32_t* out, uint32_t* scratch, void* stream) {
  if (!ctx_low || !ctx_last) return pb_set_error(PB_ERR_ARG, "null context");
  if (ctx_last->dev.L != 1 || ctx_last->dev.N != ctx_low->dev.N)
    return pb_set_error(PB_ERR_PARAMS, "ctx_last must be the 1-limb context of the dropped modulus, same N");
  if (n_polys < 0) return pb_set_error(PB_ERR_SHAPE, "negative polynomial count");
  if (n_polys == 0) return PB_OK;
  if (!ct || !out || !scratch) return pb_set_error(PB_ERR_ARG, "null argument");
  if ((reinterpret_cast<uintptr_t>(ct) | reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(scratch)) & 15)
    return pb_set_error(PB_ERR_ARG, "ct, out and scratch must be 16-byte aligned");
  if (ctx_low->dev.N < 4) return pb_set_error(PB_ERR_PARAMS, "N >= 4");
  const int N = ctx_low->dev.N, Ll = ctx_low->dev.L, Lc = Ll + 1;
  const uint32_t q_last = ctx_last->dev.q[0];
  for (int i = 0; i < Ll; ++i)
    if (ctx_low->dev.q[i] == q_last) return pb_set_error(PB_ERR_PARAMS, "dropped modulus is still in ctx_low");
  cudaStream_t st = pb_stream_of(stream);
  // the dropped limb's rows -> scratch [n][N], then to coefficient form
  cudaMemcpy2DAsync(scratch, (size_t)N * 4, ct + (size_t)(Lc - 1) * N, (size_t)Lc * N * 4, (size_t)N * 4,
                    (size_t)n_polys, cudaMemcpyDeviceToDevice, st);
  PB_CHECK_LAUNCH();
  int s = pb_ntt_inverse(ctx_last, scratch, n_polys, nullptr, st);
  if (s) return s;
  k_ms_lift<<<ms_rows_grid(n_polys), 256, 0, st>>>(ctx_low->dev, scratch, q_last, n_polys, out);
  PB_CHECK_LAUNCH();
  s = pb_ntt_forward(ctx_low, out, n_polys * Ll, nullptr, st);
  if (s) return s;
  MsConsts k{};
  for (int i = 0; i < Ll; ++i) {
    const uint32_t q = ctx_low->dev.q[i];
    k.qinv[i] = inv_mod(q_last % q, q);
    k.qinv_sh[i] = (uint32_t)(((uint64_t)k.qinv[i] << 32) / q);
  }
  k_ms_finish_v<<<ms_rows_grid(n_polys * Ll), 256, 0, st>>>(ctx_low->dev, ct, Lc, n_polys, k, out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}
