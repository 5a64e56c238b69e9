// pb_common.cuh — device-side parameter block, modular arithmetic and RNG
// shared by every sm_100a kernel of the Pencil HE linear-layer engine.
//
// Residues are u32 (moduli q < 2^30, so lazy values in [0, 4q) fit u32;
// SURVEY §0 fact 3 set A).  Z_{2^ell} share elements are u64 bit patterns.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pencil_b200.h"

#define PB_MAXL PB_MAX_LIMBS

// Everything a kernel needs about the parameter set, passed by value
// (kernel parameter space) so it is served from the constant bank.
struct PbDev {
  int N, logN, L, ell;
  uint64_t t_mask;
  uint32_t q[PB_MAXL];
  uint32_t ninv[PB_MAXL], ninv_sh[PB_MAXL];    // N^-1 mod q and its Shoup quotient
  uint32_t w0n[PB_MAXL], w0n_sh[PB_MAXL];      // last inverse stage's twiddle psi^-brv(1) * N^-1 (+ Shoup)
  uint32_t delta[PB_MAXL], delta_sh[PB_MAXL];  // floor(Q/t) mod q_i
  uint64_t mu[PB_MAXL];                        // floor(2^64 / q) (Barrett)
  double inv_q32[PB_MAXL];                     // 2^32 / q (Shoup quotient estimate)
  uint32_t qn[PB_MAXL];                        // -q^-1 mod 2^32 (Montgomery)
  uint32_t r2[PB_MAXL], r2_sh[PB_MAXL];        // 2^32 mod q (to Montgomery form) + Shoup
  uint32_t tmod[PB_MAXL];                      // t mod q_i (centered lift)
  uint32_t pinv[PB_MAXL], pinv_sh[PB_MAXL];    // Garner (q_0..q_{i-1})^-1 mod q_i
  uint32_t pmod[PB_MAXL][PB_MAXL];             // pmod[i][k] = (q_0..q_{k-1}) mod q_i
  uint32_t pmod_sh[PB_MAXL][PB_MAXL];          // their Shoup companions (Garner's inner products)
  uint64_t sc_int[PB_MAXL];                    // floor(t P_{i-1} / Q) mod 2^64
  double sc_frac[PB_MAXL];                     // frac(t P_{i-1} / Q)
  const uint2* tw_fwd;                         // [L][N] {psi^brv(i), shoup}
  const uint2* tw_inv;                         // [L][N] {psi^-brv(i), shoup}
  const uint2* tw3_fwd;                        // [L][31*N/32] P3-stage twiddles, interleaved
  const uint2* tw3_inv;
  int tw3_stride;                              // uint2 per limb in tw3_* (0 when N < 2048)
  // N = 32768 only: the two independent N/2-point transforms the rows split into
  // after the cross-half stage (2-CTA cluster NTT): half b's tables [2][L][N/2]
  // with entry I = psi^brv(I + (1 + b) 2^floor(log2 I)), and their P3 tables
  const uint2* tws_fwd;
  const uint2* tws_inv;
  const uint2* tw3s_fwd;
  const uint2* tw3s_inv;
  int tw3s_stride;
};

struct pb_ctx {
  PbDev dev;        // device pointers inside point at the buffers below
  uint2* d_tw_fwd;
  uint2* d_tw_inv;
  uint2* d_tw3_fwd;
  uint2* d_tw3_inv;
  uint2* d_tws;  // [fwd | inv] half-transform tables (N = 32768), one allocation
  pb_params host;   // the descriptor the context was created from
};

// ------------------------------------------- TMA bulk copies + mbarriers ---
// 1-D bulk async copies (cp.async.bulk, the TMA engine without a tensor map)
// into shared memory, completion tracked by an mbarrier transaction count.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n PB_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra PB_WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// The same on precomputed shared-space addresses (hot loops: no cvta per
// call), and a wait that lets the thread sleep until the phase completes
// (suspend-time hint) instead of re-issuing try_wait -- spinning warps take
// issue slots from the math warps of the same SM sub-partition.
__device__ __forceinline__ void mbar_expect_tx_a(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n PB_WAITA_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra PB_WAITA_%=;\n}\n" ::"r"(bar),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s_a(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// generic-proxy accesses to shared memory before async-proxy (TMA) writes to it
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------ mod arith ---

// Shoup multiplication: a * w mod q given ws = floor(w * 2^32 / q).
// Valid for any a < 2^32; result in [0, 2q).
__device__ __forceinline__ uint32_t mul_shoup_lazy(uint32_t a, uint32_t w, uint32_t ws, uint32_t q) {
  const uint32_t hi = __umulhi(a, ws);
  return a * w - hi * q;
}

__device__ __forceinline__ uint32_t csub(uint32_t x, uint32_t m) {  // x in [0, 2m) -> [0, m)
  return min(x, x - m);
}

__device__ __forceinline__ uint32_t mul_shoup(uint32_t a, uint32_t w, uint32_t ws, uint32_t q) {
  return csub(mul_shoup_lazy(a, w, ws, q), q);
}

// Exact Shoup quotient floor(w * 2^32 / q) for w < q, from a float64 estimate.
__device__ __forceinline__ uint32_t shoup_of(uint32_t w, uint32_t q, double inv_q32) {
  const uint64_t num = (uint64_t)w << 32;
  uint32_t est = (uint32_t)__double2uint_rz(__dmul_rn((double)w, inv_q32));
  int64_t r = (int64_t)(num - (uint64_t)est * q);
  while (r < 0) { --est; r += q; }
  while (r >= (int64_t)q) { ++est; r -= q; }
  return est;
}

// Barrett reduction of a 64-bit value: x mod q, mu = floor(2^64/q).
__device__ __forceinline__ uint32_t reduce64(uint64_t x, uint32_t q, uint64_t mu) {
  const uint64_t qh = __umul64hi(x, mu);
  uint64_t r = x - qh * (uint64_t)q;  // r < 3q
  uint32_t rr = (uint32_t)r;
  rr = min(rr, rr - q);
  rr = min(rr, rr - q);
  return rr;
}

// Generic a*b mod q for a, b < 2^32.
__device__ __forceinline__ uint32_t mulmod(uint32_t a, uint32_t b, uint32_t q, uint64_t mu) {
  return reduce64((uint64_t)a * b, q, mu);
}

// a*b mod q for a, b < q (so ab < 2^2k, k = bit length of q <= 30): Barrett
// with 32-bit operands -- floor(2^2k / q) is a shift of mu = floor(2^64 / q)
// (both hoisted out of loops over one limb) -- two IMAD.WIDE instead of the
// 64x64-bit high product of reduce64.  Result == mulmod(a, b, q, mu).
__device__ __forceinline__ uint32_t mulmod_lt(uint32_t a, uint32_t b, uint32_t q, uint64_t mu) {
  const int k = 32 - __clz(q);
  const uint32_t m = (uint32_t)(mu >> (64 - 2 * k));  // < 2^(k+1)
  const uint64_t x = (uint64_t)a * b;
  const uint32_t b1 = (uint32_t)(x >> (k - 1));       // < 2^(k+1)
  const uint32_t qh = (uint32_t)(((uint64_t)b1 * m) >> (k + 1));
  uint32_t r = (uint32_t)x - qh * q;                  // [0, 3q): floor(ab/q) - qh in {0,1,2}
  r = min(r, r - q);
  return min(r, r - q);
}

__device__ __forceinline__ uint32_t addmod(uint32_t a, uint32_t b, uint32_t q) {  // a,b < q
  return csub(a + b, q);
}
__device__ __forceinline__ uint32_t submod(uint32_t a, uint32_t b, uint32_t q) {  // a,b < q
  return csub(a + q - b, q);
}

// Centered lift of a Z_t value (t = 2^ell) into Z_q: v >= t/2 -> v - t.
__device__ __forceinline__ uint32_t lift_centered(uint64_t v, int ell, uint32_t q, uint64_t mu,
                                                  uint32_t tmod) {
  const uint32_t r = reduce64(v, q, mu);
  const bool neg = (v >> (ell - 1)) & 1ull;
  return neg ? submod(r, tmod, q) : r;
}

// ---------------------------------------------------------------- Philox ---
// Philox4x64-10 exactly as numpy's PhiloxGenerator (R:52-55 uses
// np.random.Philox(key=[seed, stream])): counter words pre-incremented, so
// raw output r of a fresh stream comes from block ctr=(r/4 + 1, 0, 0, 0),
// lane r % 4 (pinned by tests/test_gpu_rng.py).
struct u64x4 {
  uint64_t v[4];
};

__device__ __forceinline__ u64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                               uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t hi0 = __umul64hi(c0, M0), lo0 = c0 * M0;
    const uint64_t hi1 = __umul64hi(c2, M1), lo1 = c2 * M1;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0; k1 += W1;
  }
  u64x4 o;
  o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
  return o;
}

// Raw 64-bit output #idx (0-based) of numpy Philox(key=[seed, stream]).
__device__ __forceinline__ uint64_t philox_np_raw(uint64_t seed, uint64_t stream, uint64_t idx) {
  const uint64_t blk = (idx >> 2) + 1;
  const u64x4 o = philox4x64_10(blk, 0, 0, 0, seed, stream);
  return o.v[idx & 3];
}

// Philox4x32-10 for device-only randomness (encryption noise, mask filler):
// independent of numpy, domain-separated by the key words.
struct u32x4 {
  uint32_t v[4];
};
__device__ __forceinline__ u32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(c0, M0), lo0 = c0 * M0;
    const uint32_t hi1 = __umulhi(c2, M1), lo1 = c2 * M1;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0; k1 += W1;
  }
  u32x4 o;
  o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
  return o;
}

// Four uniform residues mod q (q < 2^30) from one Philox4x32 call at counter
// (jq | l << 24, pp, domain): each word is masked to bitlen(q) bits and kept
// when < q (exactly uniform; rejection probability < 2^-10 for the 30-bit NTT
// primes, < 1/2 for any q); a rejected word is redrawn as a 64-bit
// multiply-high sample from its own domain-separated call (statistical
// distance 2^-34).  Half the Philox work of one 64-bit draw per residue.
// The rejected words' redraws (probability < 2^-8 per quad): out of line, so
// the callers' unrolled loops carry one Philox body per draw, not five
// (k_encrypt_sk: 5960 -> ~2400 SASS instructions, instruction-cache stalls).
static __device__ __noinline__ uint4 uniform_quad_redraw(uint64_t seed, uint64_t pp, uint32_t c0, uint32_t q,
                                                  uint32_t domain, uint4 x) {
  uint32_t v[4] = {x.x, x.y, x.z, x.w};
  for (int i = 0; i < 4; ++i) {
    if (v[i] < q) continue;
    const u32x4 s = philox4x32_10(c0, (uint32_t)pp, (uint32_t)(pp >> 32), domain ^ (0x80000000u | (uint32_t)i),
                                  (uint32_t)seed, (uint32_t)(seed >> 32));
    v[i] = (uint32_t)__umul64hi(((uint64_t)s.v[1] << 32) | s.v[0], q);
  }
  return make_uint4(v[0], v[1], v[2], v[3]);
}

__device__ __forceinline__ void uniform_quad(uint64_t seed, uint64_t pp, int l, int jq, uint32_t q, uint32_t domain,
                                             uint32_t (&x)[4]) {
  const uint32_t c0 = (uint32_t)jq | ((uint32_t)l << 24);
  const u32x4 r = philox4x32_10(c0, (uint32_t)pp, (uint32_t)(pp >> 32), domain, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint32_t mask = (2u << (31 - __clz(q))) - 1u;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[i] = r.v[i] & mask;
    bad |= x[i] >= q;
  }
  if (bad) {
    const uint4 f = uniform_quad_redraw(seed, pp, c0, q, domain, make_uint4(x[0], x[1], x[2], x[3]));
    x[0] = f.x; x[1] = f.y; x[2] = f.z; x[3] = f.w;
  }
}

// Centred binomial CBD(20) samples: three per Philox4x32 output (120 of its
// 128 bits, disjoint 20-bit halves).
__device__ __forceinline__ void cbd20x3(const u32x4& r, int (&s)[3]) {
  s[0] = __popc(r.v[0] & 0xFFFFFu) - __popc(r.v[1] & 0xFFFFFu);
  s[1] = __popc(r.v[2] & 0xFFFFFu) - __popc(r.v[3] & 0xFFFFFu);
  s[2] = __popc(((r.v[0] >> 20) | (r.v[1] >> 20) << 12) & 0xFFFFFu) -
         __popc(((r.v[2] >> 20) | (r.v[3] >> 20) << 12) & 0xFFFFFu);
}

// ------------------------------------------------------- seed indirection ---
// A CUDA graph replays kernels with frozen arguments, so every RNG-consuming
// entry point also accepts `seed_dev`: when non-NULL the per-step seed S is
// read from device memory at run time.
//   numpy-identical streams:  key word 0 = S + seed            (np_seed)
//   device-only streams:      key = fmix64(S * G + seed)       (dev_key)
// With seed_dev == NULL the host passes the final value (eager mode); the
// host-side SeededRng.device_key uses the same mixing, so both modes agree.
__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t np_seed(uint64_t seed, const uint64_t* seed_dev) {
  return seed_dev ? *seed_dev + seed : seed;
}
__device__ __forceinline__ uint64_t dev_key(uint64_t seed, const uint64_t* seed_dev) {
  return seed_dev ? fmix64(*seed_dev * 0x9E3779B97F4A7C15ull + seed) : seed;
}

// ---------------------------------------------------------- launch glue ---

#define PB_CHECK_LAUNCH()                                      \
  do {                                                         \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return pb_set_cuda_error(_e);       \
  } while (0)

int pb_set_cuda_error(cudaError_t e);
int pb_set_error(int code, const char* msg);

static inline cudaStream_t pb_stream_of(void* s) { return (cudaStream_t)s; }

// Grid of a one-CTA-per-row kernel: all rows, or at most the cap set by
// pb_set_launch_cap (background work that must leave SMs to the critical
// path; the kernels loop over rows with a grid stride).
int64_t pb_row_grid(int64_t rows);

static inline int pb_grid_1d(int64_t n, int threads, int64_t cap = 148 * 32) {
  int64_t g = (n + threads - 1) / threads;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}
