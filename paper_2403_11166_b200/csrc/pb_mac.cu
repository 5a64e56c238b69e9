// pb_mac.cu — MO-side evaluation of the packed matmul/conv products, tiled.
//
// The MO's work for one protocol message (Alg.1 step 2-3, Alg.2 step 2) is
//   out[b,o] = sum_k ctA[b,k] (*) ptA[o,k]  (+ sum_k ctB[o,k] (*) ptB[b,k])  -  Delta*NTT(mask[b,o])
// over an (nB x nO) grid of output ciphertexts with nI input blocks.  It is
// split into two kernels:
//   k_mask_ntt    one CTA per (output, limb): builds Delta*(mask + filler) in
//                 shared memory, forward NTT in registers, writes -mask into
//                 the output's c0 row (device order);
//   k_mac_ws      (nI >= 3) a 2x2 (or 1x2) tile of outputs per CTA and a
//                 512-coefficient slice of one limb: per input block the
//                 operand row slices are copied into a 4-stage shared-memory
//                 ring by a producer warp driving the TMA engine
//                 (cp.async.bulk + mbarrier), every ct / pt vector is reused
//                 across the tile, products accumulate lazily in u64 (one
//                 IMAD.WIDE per mod-MAC), written once;
//   k_mac_eager   (nI <= 2) the same tile from registers with per-term
//                 Montgomery reduction (nothing to amortise a lazy reduction).
// Plaintexts are stored in Montgomery form (pt*2^32 mod q), so no Shoup
// companion row is streamed.
#include "pb_pack.cuh"

#include <stdlib.h>

namespace {

using pbk::mont_lazy;

__device__ __forceinline__ uint32_t delta_m(const PbDev& P, int l, uint64_t m) {
  const uint32_t q = P.q[l];
  return mul_shoup(reduce64(m, q, P.mu[l]), P.delta[l], P.delta_sh[l], q);
}

// ------------------------------------------------ plaintexts, Montgomery ---
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5))
    k_encode_plain_mont(PbDev P, pbk::Pack src, int64_t nP, uint32_t* pt) {
  using Nt = pb::Ntt<LOGN>;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  const int L = P.L;
  const int ell = P.ell;
  for (int64_t row = blockIdx.x; row < nP * L; row += gridDim.x) {  // one row per CTA unless capped
    if (row != blockIdx.x) __syncthreads();  // shared memory of the previous row is free
    const int l = (int)(row / nP);  // limb-major: co-resident CTAs share one limb's twiddles
    const int64_t p = row % nP;
    const uint32_t q = P.q[l];
    const uint64_t mu = P.mu[l];
    const uint32_t tm = P.tmod[l];
    uint32_t a[32];
    // x 2^32 (Montgomery form) applied to the source values before the NTT
    // (linear): once per occupied slot of a packed source instead of once per
    // output coefficient
    const uint32_t r2 = P.r2[l], r2s = P.r2_sh[l];
    const int bits =  // OR of the occupied indices: structurally trivial NTT stages are skipped
        pbk::load_source<Nt>(a, sm, src, p, tid,
                             [&](uint64_t v) { return mul_shoup(lift_centered(v, ell, q, mu, tm), r2, r2s, q); });
    Nt::forward(a, sm, P.tw_fwd + (size_t)l * Nt::N, P.tw3_fwd + (size_t)l * P.tw3_stride, tid, q, bits);
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = pb::canon4(a[c], q);
    Nt::gst3(pt + (p * L + l) * Nt::N, a, tid);
  }
}

// ----------------------------------------------------------- mask NTT ----
// -Delta * NTT(pi_y(mask) + filler) of output row (p, l) into m[] (P3 layout =
// device order): the uniform filler on the unused slots, Delta * mask on the
// useful ones (pi_y through out_pos / out_dst), forward NTT in registers.
template <class Nt>
__device__ __forceinline__ void neg_mask_ntt(uint32_t (&m)[32], uint32_t* sm, const PbDev& P, int l, int64_t p,
                                             const int32_t* out_pos, const int64_t* out_dst, int U,
                                             const uint64_t* mask_vals, int filler, uint64_t fseed, int tid) {
  constexpr int N = Nt::N;
  const uint32_t q = P.q[l];
  if (filler) {
    for (int jq = tid; jq < N / 4; jq += Nt::T) {
      uint32_t x[4];
      uniform_quad(fseed, (uint64_t)p, l, jq, q, 0x4d41534cu /* "MASL" */, x);
#pragma unroll
      for (int i = 0; i < 4; ++i) sm[Nt::pad(4 * jq + i)] = x[i];
    }
  } else {
    for (int j = tid; j < N; j += Nt::T) sm[Nt::pad(j)] = 0u;
  }
  __syncthreads();
  if (mask_vals) {
    const int32_t* pos = out_pos + p * U;
    const int64_t* dst = out_dst + p * U;
    for (int u0 = tid; u0 < U; u0 += 8 * Nt::T) {  // batched: index loads before value loads
      int j[8];
      int64_t d[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int u = u0 + k * Nt::T;
        j[k] = u < U ? __ldg(pos + u) : -1;
        d[k] = u < U ? __ldg(dst + u) : 0;
      }
      uint64_t v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = j[k] >= 0 ? __ldg(mask_vals + d[k]) : 0ull;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (j[k] >= 0) sm[Nt::pad(j[k])] = delta_m(P, l, v[k]);
    }
  }
  __syncthreads();
  Nt::ld1(sm, m, tid);
  __syncthreads();
  Nt::forward(m, sm, P.tw_fwd + (size_t)l * N, P.tw3_fwd + (size_t)l * P.tw3_stride, tid, q);
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const uint32_t v = pb::canon4(m[c], q);
    m[c] = v ? q - v : 0u;
  }
}

template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5))
    k_mask_ntt(PbDev P, int64_t nP, const int32_t* out_pos, const int64_t* out_dst, int U, const uint64_t* mask_vals,
               int filler, uint64_t filler_arg, const uint64_t* seed_dev, uint32_t* ct_out) {
  using Nt = pb::Ntt<LOGN>;
  extern __shared__ uint32_t sm[];
  const int l = (int)(blockIdx.x / nP);  // limb-major: co-resident CTAs share one limb's twiddles
  const int64_t p = blockIdx.x % nP;
  uint32_t m[32];
  neg_mask_ntt<Nt>(m, sm, P, l, p, out_pos, out_dst, U, mask_vals, filler,
                   filler ? dev_key(filler_arg, seed_dev) : 0ull, threadIdx.x);
  Nt::gst3(ct_out + ((size_t)p * 2 * P.L + l) * Nt::N, m, threadIdx.x);  // -mask, added to by the MAC
}

// The MO's whole evaluation of a streaming shape (nI <= 2) in one pass: per
// output row (p = b * nO + o, limb l) the -Delta NTT(mask) row is built in
// registers as in k_mask_ntt, then the 128-bit device-order vectors of the
// MAC terms sum_k ctA[b,k] (*) ptA[o,k] (+ ctB[o,k] (*) ptB[b,k]) are added
// and both output rows written once -- no -mask row written and re-read by a
// separate MAC kernel (1.46x -> 1.0x of the algorithmic traffic at K = 1).
// Bit-identical to k_mask_ntt + k_mac_* (same filler stream, same reductions).
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5))
    k_mask_mac(PbDev P, const uint32_t* __restrict__ ctA, const uint32_t* __restrict__ ptA,
               const uint32_t* __restrict__ ctB, const uint32_t* __restrict__ ptB, int nO, int nI, int64_t nP,
               const int32_t* out_pos, const int64_t* out_dst, int U, const uint64_t* mask_vals, int filler,
               uint64_t filler_arg, const uint64_t* seed_dev, uint32_t* ct_out) {
  using Nt = pb::Ntt<LOGN>;
  constexpr int N = Nt::N;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  const int L = P.L;
  const int l = (int)(blockIdx.x / nP);
  const int64_t p = blockIdx.x % nP;
  const int b = (int)(p / nO), o = (int)(p - (int64_t)b * nO);
  const uint32_t q = P.q[l], qn = P.qn[l];
  uint32_t m[32];
  neg_mask_ntt<Nt>(m, sm, P, l, p, out_pos, out_dst, U, mask_vals, filler,
                   filler ? dev_key(filler_arg, seed_dev) : 0ull, tid);
  const size_t rs = (size_t)L * N / 4;  // uint4 per polynomial
  const size_t lo = (size_t)l * N / 4 + tid;
  uint4* o0 = reinterpret_cast<uint4*>(ct_out) + (size_t)p * 2 * rs + lo;
  auto mac = [&](uint32_t& a, uint32_t x, uint32_t w) { a = addmod(a, csub(mont_lazy(x, w, q, qn), q), q); };
#pragma unroll 2
  for (int v = 0; v < 8; ++v) {
    uint32_t a0[4] = {m[4 * v], m[4 * v + 1], m[4 * v + 2], m[4 * v + 3]}, a1[4] = {0u, 0u, 0u, 0u};
    const size_t vo = lo + (size_t)v * Nt::T;
    for (int k = 0; k < nI; ++k) {
      if (ctA) {
        const uint4* c = reinterpret_cast<const uint4*>(ctA) + (size_t)(b * nI + k) * 2 * rs + vo;
        const uint4 x0 = __ldg(c), x1 = __ldg(c + rs);
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(ptA) + (size_t)(o * nI + k) * rs + vo);
        mac(a0[0], x0.x, w.x); mac(a0[1], x0.y, w.y); mac(a0[2], x0.z, w.z); mac(a0[3], x0.w, w.w);
        mac(a1[0], x1.x, w.x); mac(a1[1], x1.y, w.y); mac(a1[2], x1.z, w.z); mac(a1[3], x1.w, w.w);
      }
      if (ctB) {
        const uint4* c = reinterpret_cast<const uint4*>(ctB) + (size_t)(o * nI + k) * 2 * rs + vo;
        const uint4 x0 = __ldg(c), x1 = __ldg(c + rs);
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(ptB) + (size_t)(b * nI + k) * rs + vo);
        mac(a0[0], x0.x, w.x); mac(a0[1], x0.y, w.y); mac(a0[2], x0.z, w.z); mac(a0[3], x0.w, w.w);
        mac(a1[0], x1.x, w.x); mac(a1[1], x1.y, w.y); mac(a1[2], x1.z, w.z); mac(a1[3], x1.w, w.w);
      }
    }
    o0[(size_t)v * Nt::T] = make_uint4(a0[0], a0[1], a0[2], a0[3]);
    o0[rs + (size_t)v * Nt::T] = make_uint4(a1[0], a1[1], a1[2], a1[3]);
  }
}

// ------------------------------------------------------------ tiled MAC ---
constexpr int MAC_THREADS = 128;  // one uint4 (4 coefficients) per thread per row slice

// Vector of V consecutive coefficients (V = 2: uint2, V = 4: uint4).
template <int V> struct Vec;
template <> struct Vec<4> {
  using T = uint4;
  __device__ __forceinline__ static uint32_t get(const T& x, int e) { return e == 0 ? x.x : e == 1 ? x.y : e == 2 ? x.z : x.w; }
  __device__ __forceinline__ static T make(const uint32_t (&a)[4]) { return make_uint4(a[0], a[1], a[2], a[3]); }
  __device__ __forceinline__ static T zero() { return make_uint4(0, 0, 0, 0); }
};
template <> struct Vec<2> {
  using T = uint2;
  __device__ __forceinline__ static uint32_t get(const T& x, int e) { return e == 0 ? x.x : x.y; }
  __device__ __forceinline__ static T make(const uint32_t (&a)[2]) { return make_uint2(a[0], a[1]); }
  __device__ __forceinline__ static T zero() { return make_uint2(0, 0); }
};

// Lazy 64-bit accumulation (k_mac_ws): a product x * w~ (x < q,
// w~ = w 2^32 mod q, both < 2^30) is < 2^60, so 14 products plus a reduced
// residue (< 2^30) fit a u64 -- a mod-MAC is ONE IMAD.WIDE.U32 (fma pipe)
// instead of a Montgomery multiply + two conditional subtractions (alu pipe,
// which bound the eager kernel: ncu alu 56%, math-pipe-throttle stalls).  The
// accumulator is Barrett-reduced every MAC_CHUNK input blocks and once at the
// end, where one Montgomery step removes the plaintexts' 2^32 factor.
constexpr int MAC_CHUNK = 7;  // k-steps per reduction (2 terms x 7 = 14 products)
// k_mac_ws folds with ONE IMAD.WIDE per accumulator instead of a Barrett
// reduction: a = lo + hi * (2^32 mod q) < q 2^32, after which m more products
// (< q^2 each) keep a < q (2^32 + m q) < 2^64 for m <= 12 (q < 2^30).
constexpr int MAC_FOLD1 = 12;  // k-steps between folds, one term
constexpr int MAC_FOLD2 = 6;   // two terms (two products per k-step)

// TMA-pipelined lazy MAC.  A CTA owns a 2x2 output tile and a 512-coefficient
// slice of one limb; per input block k its operands are 2-KB contiguous row
// slices (ct c0/c1 per batch block, pt per output block, and the same for the
// second cross term), copied into a STAGES-deep shared-memory ring by the TMA
// engine (cp.async.bulk + mbarrier) while the CTA multiplies the previous
// stages -- the L2 latency that bounded the register-load kernel is off the
// critical path, and the math is one IMAD.WIDE.U32 per mod-MAC.

template <int TB, int TO, int V, int CT = MAC_THREADS>
struct PipeCfg {
  static constexpr int SLOT = CT * V * 4;  // bytes per operand slice
  static constexpr int SLOTS_A = 2 * TB + TO;       // ct c0/c1 per batch block + pt per output block
  static constexpr int SLOTS_B = 2 * TO + TB;
};

// Warp-specialised TMA-pipelined MAC: a fifth warp only issues the TMA
// copies (per-copy address = base + k * stride, precomputed), gated per stage
// by an "empty" mbarrier the four consumer warps arrive on, so the consumers
// never wait for the issuing thread at a CTA barrier (ncu on the round-1
// single-role kernel: 26%
// of stall samples were the per-k __syncthreads behind thread 0's issue work).
// TERMS: 1 = cross term A only, 2 = B only (compile-time: the consumer loop
// carries no per-k term branches and the slot layout is constant; single-term
// evaluations 6-8 % faster); 0 = both, taken at run time -- the compile-time
// two-term body spills at the 96-register budget (and measured 6-10 % slower).
template <int TB, int TO, int V, int STAGES, int MINB = 1, int CT = MAC_THREADS, int TERMS = 3>
__global__ void __launch_bounds__(CT + 32, MINB)
    k_mac_ws(PbDev P, const uint32_t* ctA, const uint32_t* ptA, const uint32_t* ctB, const uint32_t* ptB, int nB,
             int nO, int nI, uint32_t* ct_out) {
  using C = PipeCfg<TB, TO, V, CT>;
  using VT = typename Vec<V>::T;
  const bool HA = TERMS ? (TERMS & 1) != 0 : ctA != nullptr, HB = TERMS ? (TERMS & 2) != 0 : ctB != nullptr;
  extern __shared__ __align__(128) uint8_t pipe_sm[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int CA = 0, PA = 2 * TB, CB = HA ? C::SLOTS_A : 0, PB = CB + 2 * TO;
  const int nslots = (HA ? C::SLOTS_A : 0) + (HB ? C::SLOTS_B : 0);
  const int N = P.N, L = P.L;
  const int slices = N / (V * CT);
  const int tilesO = (nO + TO - 1) / TO;
  const int tb = blockIdx.x / tilesO, to = blockIdx.x % tilesO;
  const int l = blockIdx.y / slices, sl = blockIdx.y % slices;
  const int tid = threadIdx.x;
  bool okb[TB], oko[TO];
#pragma unroll
  for (int i = 0; i < TB; ++i) okb[i] = tb * TB + i < nB;
#pragma unroll
  for (int o = 0; o < TO; ++o) oko[o] = to * TO + o < nO;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CT / 32);
    }
    mbar_init_fence();
  }
  __syncthreads();

  if (tid >= CT) {  // ---- producer warp (one thread; slot table in registers)
    if (tid != CT) return;
    constexpr int NS = C::SLOTS_A + C::SLOTS_B;
    const size_t rowb = (size_t)N * 4;
    const size_t off = (size_t)sl * C::SLOT + (size_t)l * rowb;
    const size_t ct_k = 2 * (size_t)L * rowb, pt_k = (size_t)L * rowb;  // bytes per k step
    const uint8_t* base[NS];
    uint32_t dsto[NS];
    bool on[NS];
    uint32_t bytes = 0;
#pragma unroll
    for (int i = 0; i < TB; ++i) {
      const size_t bi = (size_t)(tb * TB + i) * nI;
      const uint8_t* a = reinterpret_cast<const uint8_t*>(ctA) + bi * ct_k + off;
      base[2 * i] = a, base[2 * i + 1] = a + (size_t)L * rowb;
      dsto[2 * i] = (CA + 2 * i) * C::SLOT, dsto[2 * i + 1] = (CA + 2 * i + 1) * C::SLOT;
      on[2 * i] = on[2 * i + 1] = HA && okb[i];
      base[C::SLOTS_A + 2 * TO + i] = reinterpret_cast<const uint8_t*>(ptB) + bi * pt_k + off;
      dsto[C::SLOTS_A + 2 * TO + i] = (PB + i) * C::SLOT;
      on[C::SLOTS_A + 2 * TO + i] = HB && okb[i];
    }
#pragma unroll
    for (int o = 0; o < TO; ++o) {
      const size_t oi = (size_t)(to * TO + o) * nI;
      base[2 * TB + o] = reinterpret_cast<const uint8_t*>(ptA) + oi * pt_k + off;
      dsto[2 * TB + o] = (PA + o) * C::SLOT;
      on[2 * TB + o] = HA && oko[o];
      const uint8_t* b = reinterpret_cast<const uint8_t*>(ctB) + oi * ct_k + off;
      base[C::SLOTS_A + 2 * o] = b, base[C::SLOTS_A + 2 * o + 1] = b + (size_t)L * rowb;
      dsto[C::SLOTS_A + 2 * o] = (CB + 2 * o) * C::SLOT, dsto[C::SLOTS_A + 2 * o + 1] = (CB + 2 * o + 1) * C::SLOT;
      on[C::SLOTS_A + 2 * o] = on[C::SLOTS_A + 2 * o + 1] = HB && oko[o];
    }
#pragma unroll
    for (int c = 0; c < NS; ++c) bytes += on[c] ? (uint32_t)C::SLOT : 0u;
    const uint32_t sm0 = smem_addr(pipe_sm), full0 = smem_addr(full), empty0 = smem_addr(empty);
    for (int k = 0; k < nI; ++k) {
      const int s = k % STAGES;
      const uint32_t fb = full0 + 8u * s;
      if (k >= STAGES) mbar_wait_a(empty0 + 8u * s, (uint32_t)((k / STAGES - 1) & 1));
      mbar_expect_tx_a(fb, bytes);
      const uint32_t st = sm0 + (uint32_t)(s * nslots * C::SLOT);
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        // slots [2TB ct | TO pt] of term A advance by ct_k / pt_k, term B [2TO ct | TB pt] likewise
        const size_t stride = (c < 2 * TB || (c >= C::SLOTS_A && c < C::SLOTS_A + 2 * TO)) ? ct_k : pt_k;
        if (on[c]) bulk_g2s_a(st + dsto[c], base[c] + (size_t)k * stride, C::SLOT, fb);
      }
    }
    return;
  }

  // ---- consumer warps
  const uint32_t q = P.q[l], qn = P.qn[l];
  const uint64_t mu = P.mu[l];
  uint64_t acc[TB][TO][2][V];
#pragma unroll
  for (int i = 0; i < TB; ++i)
#pragma unroll
    for (int o = 0; o < TO; ++o)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = 0; e < V; ++e) acc[i][o][c][e] = 0ull;
  auto mac = [&](uint64_t (&a)[V], const VT& x, const VT& w) {
#pragma unroll
    for (int e = 0; e < V; ++e) a[e] += (uint64_t)Vec<V>::get(x, e) * Vec<V>::get(w, e);
  };
  constexpr int SV = C::SLOT / (4 * V);
  const int chunk = (HA && HB) ? MAC_FOLD2 : MAC_FOLD1;  // k-steps between folds
  const uint32_t r32 = reduce64(1ull << 32, q, mu);            // 2^32 mod q
  int since = 0;
  const uint32_t full0 = smem_addr(full), empty0 = smem_addr(empty);
  const VT* st0 = reinterpret_cast<const VT*>(pipe_sm) + tid;
  const bool lane0 = (tid & 31) == 0;
  uint32_t ph = 0;
  // the stage ring unrolled: stage s is a compile-time offset from one base
  // (no per-k address arithmetic or shared-window re-derivation)
  for (int k0 = 0; k0 < nI; k0 += STAGES, ph ^= 1u) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      const int k = k0 + s;
      if (k >= nI) break;
      mbar_wait_a(full0 + 8u * s, ph);
      const VT* st = st0 + s * (nslots * SV);
      if (HA) {
        VT w[TO];
#pragma unroll
        for (int o = 0; o < TO; ++o) w[o] = st[(PA + o) * SV];
#pragma unroll
        for (int i = 0; i < TB; ++i) {
          const VT x0 = st[(CA + 2 * i) * SV], x1 = st[(CA + 2 * i + 1) * SV];
#pragma unroll
          for (int o = 0; o < TO; ++o) { mac(acc[i][o][0], x0, w[o]); mac(acc[i][o][1], x1, w[o]); }
        }
      }
      if (HB) {
        VT u[TB];
#pragma unroll
        for (int i = 0; i < TB; ++i) u[i] = st[(PB + i) * SV];
#pragma unroll
        for (int o = 0; o < TO; ++o) {
          const VT y0 = st[(CB + 2 * o) * SV], y1 = st[(CB + 2 * o + 1) * SV];
#pragma unroll
          for (int i = 0; i < TB; ++i) { mac(acc[i][o][0], y0, u[i]); mac(acc[i][o][1], y1, u[i]); }
        }
      }
      __syncwarp();
      if (lane0) mbar_arrive_a(empty0 + 8u * s);  // this warp is done reading stage s
      if (++since == chunk && k + 1 < nI) {
        since = 0;
#pragma unroll
        for (int i = 0; i < TB; ++i)
#pragma unroll
          for (int o = 0; o < TO; ++o)
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int e = 0; e < V; ++e) {
                const uint64_t a = acc[i][o][c][e];
                acc[i][o][c][e] = (uint64_t)(uint32_t)(a >> 32) * r32 + (uint32_t)a;
              }
      }
    }
  }
  auto fin = [&](uint64_t a) { return csub(mont_lazy(reduce64(a, q, mu), 1u, q, qn), q); };
  VT* out = reinterpret_cast<VT*>(ct_out);
  const size_t row = (size_t)N / V;
  const size_t v = (size_t)sl * CT + tid;
#pragma unroll
  for (int i = 0; i < TB; ++i)
#pragma unroll
    for (int o = 0; o < TO; ++o) {
      if (!(okb[i] && oko[o])) continue;
      const size_t r = (size_t)(tb * TB + i) * nO + (to * TO + o);
      const size_t b0 = (r * 2 * L + l) * row + v;
      const VT m = out[b0];
      uint32_t c0[V], c1[V];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        c0[e] = addmod(fin(acc[i][o][0][e]), Vec<V>::get(m, e), q);
        c1[e] = fin(acc[i][o][1][e]);
      }
      out[b0] = Vec<V>::make(c0);
      out[b0 + (size_t)L * row] = Vec<V>::make(c1);
    }
}

template <int TB, int TO, int V, int STAGES, int MINB, int CT, int TERMS>
void launch_ws_t(const PbDev& P, const uint32_t* ctA, const uint32_t* ptA, const uint32_t* ctB, const uint32_t* ptB,
                 int nB, int nO, int nI, uint32_t* out, cudaStream_t st) {
  using C = PipeCfg<TB, TO, V, CT>;
  const size_t smem = (size_t)STAGES * ((ctA ? C::SLOTS_A : 0) + (ctB ? C::SLOTS_B : 0)) * C::SLOT;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_mac_ws<TB, TO, V, STAGES, MINB, CT, TERMS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  dim3 grid((unsigned)(((nB + TB - 1) / TB) * ((nO + TO - 1) / TO)), (unsigned)(P.L * (P.N / (V * CT))));
  k_mac_ws<TB, TO, V, STAGES, MINB, CT, TERMS><<<grid, CT + 32, smem, st>>>(P, ctA, ptA, ctB, ptB, nB, nO, nI, out);
}

template <int TB, int TO, int V, int STAGES, int MINB = 1, int CT = MAC_THREADS>
void launch_ws(const PbDev& P, const uint32_t* ctA, const uint32_t* ptA, const uint32_t* ctB, const uint32_t* ptB,
               int nB, int nO, int nI, uint32_t* out, cudaStream_t st) {
  if (ctA && ctB) launch_ws_t<TB, TO, V, STAGES, MINB, CT, 0>(P, ctA, ptA, ctB, ptB, nB, nO, nI, out, st);
  else if (ctA) launch_ws_t<TB, TO, V, STAGES, MINB, CT, 1>(P, ctA, ptA, ctB, ptB, nB, nO, nI, out, st);
  else launch_ws_t<TB, TO, V, STAGES, MINB, CT, 2>(P, ctA, ptA, ctB, ptB, nB, nO, nI, out, st);
}

// Eager variant (Montgomery multiply + reduce per term, u32 accumulators,
// 96 registers): faster than the lazy kernel when nI <= 2 (no reduction to
// amortise; the K=1 FC shape is HBM/latency-bound).
template <int TB, int TO>
__global__ void __launch_bounds__(MAC_THREADS)
    k_mac_eager(PbDev P, const uint32_t* ctA, const uint32_t* ptA, const uint32_t* ctB, const uint32_t* ptB, int nB,
                int nO, int nI, uint32_t* ct_out) {
  const int N = P.N, L = P.L;
  const int slices = N / (4 * MAC_THREADS);
  const int tilesO = (nO + TO - 1) / TO;
  const int tb = blockIdx.x / tilesO, to = blockIdx.x % tilesO;
  const int l = blockIdx.y / slices, sl = blockIdx.y % slices;
  const uint32_t q = P.q[l], qn = P.qn[l];
  const size_t row = (size_t)N / 4;  // uint4 per row
  const size_t v = (size_t)sl * MAC_THREADS + threadIdx.x;
  const uint4* cA = reinterpret_cast<const uint4*>(ctA);
  const uint4* pA = reinterpret_cast<const uint4*>(ptA);
  const uint4* cB = reinterpret_cast<const uint4*>(ctB);
  const uint4* pB = reinterpret_cast<const uint4*>(ptB);
  uint32_t acc[TB][TO][2][4];
#pragma unroll
  for (int i = 0; i < TB; ++i)
#pragma unroll
    for (int o = 0; o < TO; ++o)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][o][c][e] = 0u;
  bool okb[TB], oko[TO];
#pragma unroll
  for (int i = 0; i < TB; ++i) okb[i] = tb * TB + i < nB;
#pragma unroll
  for (int o = 0; o < TO; ++o) oko[o] = to * TO + o < nO;

  auto mac4 = [&](uint32_t (&a)[4], const uint4& x, const uint4& w) {
    a[0] = addmod(a[0], csub(mont_lazy(x.x, w.x, q, qn), q), q);
    a[1] = addmod(a[1], csub(mont_lazy(x.y, w.y, q, qn), q), q);
    a[2] = addmod(a[2], csub(mont_lazy(x.z, w.z, q, qn), q), q);
    a[3] = addmod(a[3], csub(mont_lazy(x.w, w.w, q, qn), q), q);
  };
  const uint4 z4 = make_uint4(0, 0, 0, 0);
  for (int k = 0; k < nI; ++k) {
    if (cA) {  // term A: ctA[b-block] (*) ptA[o-block]
      uint4 x0[TB], x1[TB], w[TO];
#pragma unroll
      for (int i = 0; i < TB; ++i) {
        const size_t base = ((size_t)((tb * TB + i) * nI + k) * 2 * L + l) * row + v;
        x0[i] = okb[i] ? __ldg(cA + base) : z4;
        x1[i] = okb[i] ? __ldg(cA + base + (size_t)L * row) : z4;
      }
#pragma unroll
      for (int o = 0; o < TO; ++o) w[o] = oko[o] ? __ldg(pA + ((size_t)((to * TO + o) * nI + k) * L + l) * row + v) : z4;
#pragma unroll
      for (int i = 0; i < TB; ++i)
#pragma unroll
        for (int o = 0; o < TO; ++o) {
          mac4(acc[i][o][0], x0[i], w[o]);
          mac4(acc[i][o][1], x1[i], w[o]);
        }
    }
    if (cB) {  // term B: ctB[o-block] (*) ptB[b-block]
      uint4 y0[TO], y1[TO], u[TB];
#pragma unroll
      for (int o = 0; o < TO; ++o) {
        const size_t base = ((size_t)((to * TO + o) * nI + k) * 2 * L + l) * row + v;
        y0[o] = oko[o] ? __ldg(cB + base) : z4;
        y1[o] = oko[o] ? __ldg(cB + base + (size_t)L * row) : z4;
      }
#pragma unroll
      for (int i = 0; i < TB; ++i) u[i] = okb[i] ? __ldg(pB + ((size_t)((tb * TB + i) * nI + k) * L + l) * row + v) : z4;
#pragma unroll
      for (int i = 0; i < TB; ++i)
#pragma unroll
        for (int o = 0; o < TO; ++o) {
          mac4(acc[i][o][0], y0[o], u[i]);
          mac4(acc[i][o][1], y1[o], u[i]);
        }
    }
  }
  uint4* out = reinterpret_cast<uint4*>(ct_out);
#pragma unroll
  for (int i = 0; i < TB; ++i)
#pragma unroll
    for (int o = 0; o < TO; ++o) {
      if (!(okb[i] && oko[o])) continue;
      const size_t r = (size_t)(tb * TB + i) * nO + (to * TO + o);
      const size_t b0 = (r * 2 * L + l) * row + v;
      const uint4 m = out[b0];  // -mask written by k_mask_ntt
      out[b0] = make_uint4(addmod(acc[i][o][0][0], m.x, q), addmod(acc[i][o][0][1], m.y, q),
                           addmod(acc[i][o][0][2], m.z, q), addmod(acc[i][o][0][3], m.w, q));
      out[b0 + (size_t)L * row] = make_uint4(acc[i][o][1][0], acc[i][o][1][1], acc[i][o][1][2], acc[i][o][1][3]);
    }
}

template <typename KernelT>
void set_smem(KernelT k, size_t smem) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <int LOGN>
void launch_encode_mont(const PbDev& P, pbk::Pack src, int64_t nP, uint32_t* pt, cudaStream_t st) {
  using Nt = pb::Ntt<LOGN>;
  const size_t smem = Nt::SMEM_WORDS * 4;
  set_smem(k_encode_plain_mont<LOGN>, smem);
  k_encode_plain_mont<LOGN><<<(unsigned)pb_row_grid(nP * P.L), Nt::T, smem, st>>>(P, src, nP, pt);
}

template <int LOGN>
void launch_mask(const PbDev& P, int64_t nP, const int32_t* out_pos, const int64_t* out_dst, int U,
                 const uint64_t* mask_vals, int filler, uint64_t fseed, const uint64_t* seed_dev, uint32_t* ct_out,
                 cudaStream_t st) {
  using Nt = pb::Ntt<LOGN>;
  const size_t smem = Nt::SMEM_WORDS * 4;
  set_smem(k_mask_ntt<LOGN>, smem);
  k_mask_ntt<LOGN><<<(unsigned)(nP * P.L), Nt::T, smem, st>>>(P, nP, out_pos, out_dst, U, mask_vals, filler, fseed,
                                                              seed_dev, ct_out);
}

template <int LOGN>
void launch_mask_mac(const PbDev& P, const uint32_t* ctA, const uint32_t* ptA, const uint32_t* ctB,
                     const uint32_t* ptB, int nB, int nO, int nI, const int32_t* out_pos, const int64_t* out_dst,
                     int U, const uint64_t* mask_vals, int filler, uint64_t fseed, const uint64_t* seed_dev,
                     uint32_t* ct_out, cudaStream_t st) {
  using Nt = pb::Ntt<LOGN>;
  const size_t smem = Nt::SMEM_WORDS * 4;
  set_smem(k_mask_mac<LOGN>, smem);
  const int64_t nP = (int64_t)nB * nO;
  k_mask_mac<LOGN><<<(unsigned)(nP * P.L), Nt::T, smem, st>>>(P, ctA, ptA, ctB, ptB, nO, nI, nP, out_pos, out_dst, U,
                                                              mask_vals, filler, fseed, seed_dev, ct_out);
}

int check_ctx(const pb_ctx* ctx) {
  if (!ctx) return pb_set_error(PB_ERR_ARG, "null context");
  if (ctx->dev.logN < 11) return pb_set_error(PB_ERR_PARAMS, "fused BFV kernels need N >= 2048");
  return PB_OK;
}

}  // namespace

extern "C" int pb_encode_plain_mont(const pb_ctx* ctx, const uint64_t* vals, const int32_t* pack_pos,
                                    const int32_t* pack_src, int32_t Z, int64_t P, uint32_t* pt_mont, void* stream) {
  if (int s = check_ctx(ctx)) return s;
  if (P <= 0) return PB_OK;
  if (!vals || !pt_mont) return pb_set_error(PB_ERR_ARG, "null argument");
  if (pack_pos && (!pack_src || Z < 0)) return pb_set_error(PB_ERR_ARG, "packed source needs pos, src and Z");
  if (P > (int64_t)0x7fffffff / ctx->dev.L) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  pbk::Pack src{vals, pack_pos, pack_src, pack_pos ? Z : 0};
  PB_DISPATCH_LOGN(ctx->dev.logN, launch_encode_mont, ctx->dev, src, P, pt_mont, pb_stream_of(stream));
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_mask_ntt(const pb_ctx* ctx, int64_t P, const int32_t* out_pos, const int64_t* out_dst, int32_t U,
                           const uint64_t* mask_vals, int filler, uint64_t filler_seed, const uint64_t* seed_dev,
                           uint32_t* ct_out, void* stream) {
  if (int s = check_ctx(ctx)) return s;
  if (P <= 0) return PB_OK;
  if (!ct_out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (mask_vals && (!out_pos || !out_dst)) return pb_set_error(PB_ERR_ARG, "mask needs out_pos/out_dst");
  if (P > (int64_t)0x7fffffff / ctx->dev.L) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  PB_DISPATCH_LOGN(ctx->dev.logN, launch_mask, ctx->dev, P, out_pos, out_dst, U, mask_vals, filler, filler_seed,
                   seed_dev, ct_out, pb_stream_of(stream));
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_ctpt_mac_tiled(const pb_ctx* ctx, const uint32_t* ctA, const uint32_t* ptA_mont, const uint32_t* ctB,
                                 const uint32_t* ptB_mont, int32_t nB, int32_t nO, int32_t nI, uint32_t* ct_out,
                                 void* stream) {
  if (int s = check_ctx(ctx)) return s;
  if (nB <= 0 || nO <= 0) return PB_OK;
  if (!ct_out || (!ctA && !ctB)) return pb_set_error(PB_ERR_ARG, "null argument");
  if ((ctA && !ptA_mont) || (ctB && !ptB_mont)) return pb_set_error(PB_ERR_ARG, "each term needs ct and pt");
  if (nI < 1) return pb_set_error(PB_ERR_SHAPE, "nI must be >= 1");
  const int N = ctx->dev.N, L = ctx->dev.L;
  cudaStream_t st = pb_stream_of(stream);
  if (nI <= 2) {  // streaming shapes: 1x1 tiles (96 -> fewer registers, more resident warps);
                  // FC-like K=1: 0.174 -> 0.131 ms, 4.5 TB/s of actual DRAM traffic
    dim3 grid((unsigned)(nB * nO), (unsigned)(L * (N / (4 * MAC_THREADS))));
    k_mac_eager<1, 1><<<grid, MAC_THREADS, 0, st>>>(ctx->dev, ctA, ptA_mont, ctB, ptB_mont, nB, nO, nI, ct_out);
  } else {
    // Warp-specialised TMA-pipelined lazy MAC (B200, graph-timed): FC 784x128 fwd
    // 52.7 -> 39.3 us, its grad-W 51.1 -> 45.7 us, conv-like K=16 646 -> 587 us vs
    // a single-role pipelined kernel (round 1, removed).
    // Tiles 2x2 (single-role kernels and 1x2 / 2x4 / 4x4 / grouped tiles
    // measured slower, profiles/r02_mac_tiles.jsonl); one batch block (nB = 1):
    // 1x1, no idle half tile (MLP fwd2 4.0 -> 3.2 us, grad-W2 5.4 -> 4.0 us).
    // Two cross terms (Alg. 2) stage twice the operands per k-step: a 2-deep
    // ring (48 KB) keeps 4 CTAs per SM where 4 stages (96 KB) fit only 2 --
    // conv-like K=16 two-term 1236 -> 802 us, MLP grad-W0 79 -> 63 us (round 1
    // used 1x2 tiles at 4 stages for these).
    if (nB == 1)
      launch_ws<1, 1, 4, 4, 4>(ctx->dev, ctA, ptA_mont, ctB, ptB_mont, nB, nO, nI, ct_out, st);
    else if (ctA && ctB)
      launch_ws<2, 2, 4, 2, 4>(ctx->dev, ctA, ptA_mont, ctB, ptB_mont, nB, nO, nI, ct_out, st);
    else
      launch_ws<2, 2, 4, 4, 4>(ctx->dev, ctA, ptA_mont, ctB, ptB_mont, nB, nO, nI, ct_out, st);
  }
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_mask_mac(const pb_ctx* ctx, const uint32_t* ctA, const uint32_t* ptA_mont, const uint32_t* ctB,
                           const uint32_t* ptB_mont, int32_t nB, int32_t nO, int32_t nI, const int32_t* out_pos,
                           const int64_t* out_dst, int32_t U, const uint64_t* mask_vals, int filler,
                           uint64_t filler_seed, const uint64_t* seed_dev, uint32_t* ct_out, void* stream) {
  if (int s = check_ctx(ctx)) return s;
  if (nB <= 0 || nO <= 0) return PB_OK;
  if (!ct_out || (!ctA && !ctB)) return pb_set_error(PB_ERR_ARG, "null argument");
  if ((ctA && !ptA_mont) || (ctB && !ptB_mont)) return pb_set_error(PB_ERR_ARG, "each term needs ct and pt");
  if (nI < 1 || nI > 2) return pb_set_error(PB_ERR_SHAPE, "pb_mask_mac takes the streaming shapes nI <= 2");
  if (mask_vals && (!out_pos || !out_dst)) return pb_set_error(PB_ERR_ARG, "mask needs out_pos/out_dst");
  if ((int64_t)nB * nO > (int64_t)0x7fffffff / ctx->dev.L) return pb_set_error(PB_ERR_SHAPE, "too many outputs");
  PB_DISPATCH_LOGN(ctx->dev.logN, launch_mask_mac, ctx->dev, ctA, ptA_mont, ctB, ptB_mont, nB, nO, nI, out_pos,
                   out_dst, U, mask_vals, filler, filler_seed, seed_dev, ct_out, pb_stream_of(stream));
  PB_CHECK_LAUNCH();
  return PB_OK;
}
