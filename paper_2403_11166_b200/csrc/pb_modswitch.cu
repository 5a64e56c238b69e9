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

// x[p][i][n] = centered(a[p][n]) mod q_i, a in [0, q_last).
__global__ void k_ms_lift(PbDev P, const uint32_t* __restrict__ a, uint32_t q_last, int64_t n_polys,
                          uint32_t* __restrict__ x) {
  const int N = P.N, L = P.L;
  const int64_t total = n_polys * (int64_t)N;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = g / N;
    const int n = (int)(g - p * N);
    const uint32_t v = a[g];
    const bool neg = v > (q_last >> 1);
    const uint32_t mag = neg ? q_last - v : v;  // |centered value| < q_last / 2
    for (int i = 0; i < L; ++i) {
      const uint32_t q = P.q[i];
      const uint32_t r = mag >= q ? mag % q : mag;
      x[(p * L + i) * N + n] = (neg && r) ? q - r : r;
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

// out[p][i] = (c[p][i] - x[p][i]) * q_last^-1 mod q_i, x (NTT form) in place in out.
__global__ void k_ms_finish_v(PbDev P, const uint32_t* __restrict__ c, int c_limbs, int64_t n_polys, MsConsts k,
                              uint32_t* out) {
  const int N = P.N, L = P.L;
  const int64_t total = n_polys * (int64_t)L * N;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = g / N;
    const int n = (int)(g - row * N);
    const int64_t p = row / L;
    const int i = (int)(row - p * L);
    const uint32_t q = P.q[i];
    const uint32_t cv = c[(p * c_limbs + i) * N + n], xv = out[g];
    const uint32_t d = cv >= xv ? cv - xv : cv + q - xv;
    out[g] = mul_shoup(d, k.qinv[i], k.qinv_sh[i], q);
  }
}

int ms_grid(int64_t n) {
  const int64_t b = (n + 255) / 256, cap = 148 * 16;
  return (int)(b < 1 ? 1 : (b < cap ? b : cap));
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
  k_ms_lift<<<ms_grid(n_polys * N), 256, 0, st>>>(ctx_low->dev, scratch, q_last, n_polys, out);
  PB_CHECK_LAUNCH();
  s = pb_ntt_forward(ctx_low, out, n_polys * Ll, nullptr, st);
  if (s) return s;
  MsConsts k{};
  for (int i = 0; i < Ll; ++i) {
    const uint32_t q = ctx_low->dev.q[i];
    k.qinv[i] = inv_mod(q_last % q, q);
    k.qinv_sh[i] = (uint32_t)(((uint64_t)k.qinv[i] << 32) / q);
  }
  k_ms_finish_v<<<ms_grid(n_polys * Ll * N), 256, 0, st>>>(ctx_low->dev, ct, Lc, n_polys, k, out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}
