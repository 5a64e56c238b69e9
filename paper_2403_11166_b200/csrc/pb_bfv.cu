// pb_bfv.cu — fused RNS-BFV kernels for the Pencil linear-layer protocol.
//
//   encode_plain     centered lift + NTT + Shoup companions   (he_plain_mul operand)
//   encrypt_pk/_sk   lift/pack + Delta*m + NTT + key MAC
//   decrypt*         c0 + c1*s + INTT (+ Garner/scale-round, + pi_y^-1 gather)
//   ctpt_mac_mask    sum_k ct (*) pt - Delta*NTT(mask)        (Alg.1 steps 2-3, Alg.2 step 2)
//
// One CTA per (polynomial, limb); the NTT lives in registers/shared memory
// (pb_ntt.cuh) so every kernel reads its operands once from HBM and writes
// its result once.
#include "pb_ntt.cuh"

#include <cooperative_groups.h>
#include <cstdlib>

namespace {

// A plaintext source: `vals` is a flat Z_t tensor.  With `pos` set, poly p
// has coefficient pos[p][z] = vals[src[p][z]] for z < Z (pos < 0: unused
// slot) and zeros elsewhere -- the compact form of the packing maps pi_v /
// pi_W.  With pos == NULL, vals is a dense [P][N] array.
struct PbPack {
  const uint64_t* vals;
  const int32_t* pos;
  const int32_t* src;
  int Z;
};

// Loads the lifted source polynomial p into a[] in the NTT's P1 layout.
// The packed path builds the row in shared memory (zero + scatter) and
// leaves `sm` free (synchronised) for the NTT that follows.
template <class Nt, class Lift>
__device__ __forceinline__ void load_source(uint32_t (&a)[32], uint32_t* sm, const PbPack& s, int64_t p, int tid,
                                            Lift lift) {
  if (s.pos) {
    for (int j = tid; j < Nt::N; j += Nt::T) sm[Nt::pad(j)] = 0u;
    __syncthreads();
    const int32_t* pp = s.pos + p * s.Z;
    const int32_t* ps = s.src + p * s.Z;
    // batches of 8 slots per thread: all position / source loads are issued
    // before the dependent value loads (a per-slot pos -> src -> value chain
    // serialises three L2 round trips per slot)
    for (int z0 = tid; z0 < s.Z; z0 += 8 * Nt::T) {
      int j[8], si[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int z = z0 + u * Nt::T;
        j[u] = z < s.Z ? __ldg(pp + z) : -1;
        si[u] = z < s.Z ? __ldg(ps + z) : 0;
      }
      uint64_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = j[u] >= 0 ? __ldg(s.vals + si[u]) : 0ull;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j[u] >= 0) sm[Nt::pad(j[u])] = lift(v[u]);
    }
    __syncthreads();
    Nt::ld1(sm, a, tid);
    __syncthreads();
  } else {
    const uint64_t* v = s.vals + p * Nt::N;
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = lift(__ldg(v + Nt::j1(tid, c)));
  }
}

__device__ __forceinline__ uint32_t lift_small(int v, uint32_t q) { return v < 0 ? q - (uint32_t)(-v) : (uint32_t)v; }

// Delta * m mod q for a Z_t value m.
__device__ __forceinline__ uint32_t delta_m(const PbDev& P, int l, uint64_t m) {
  const uint32_t q = P.q[l];
  return mul_shoup(reduce64(m, q, P.mu[l]), P.delta[l], P.delta_sh[l], q);
}

// --------------------------------------------------------------- encode ---
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5))
    k_encode_plain(PbDev P, PbPack src, int64_t nP, uint32_t* pt, uint32_t* pt_sh) {
  using Nt = pb::Ntt<LOGN>;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  const int L = P.L;
  const int l = (int)(blockIdx.x / nP);  // limb-major: co-resident CTAs share one limb's twiddles
  const int64_t p = blockIdx.x % nP;
  const uint32_t q = P.q[l];
  const uint64_t mu = P.mu[l];
  const uint32_t tm = P.tmod[l];
  const int ell = P.ell;
  uint32_t a[32];
  load_source<Nt>(a, sm, src, p, tid, [&](uint64_t v) { return lift_centered(v, ell, q, mu, tm); });
  Nt::forward(a, sm, P.tw_fwd + (size_t)l * Nt::N, P.tw3_fwd + (size_t)l * P.tw3_stride, tid, q);
  uint32_t* row = pt + (p * L + l) * Nt::N;
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = pb::canon4(a[c], q);
  Nt::gst3(row, a, tid);
  if (pt_sh) {
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = shoup_of(a[c], q, P.inv_q32[l]);
    Nt::gst3(pt_sh + (p * L + l) * Nt::N, a, tid);
  }
}

// Dense lift (coefficient form): out[p][l][j] = lift(vals[p][j]).
__global__ void k_lift(PbDev P, const uint64_t* vals, int64_t nP, int centered, uint32_t* out) {
  const int N = P.N, L = P.L;
  const int64_t total = nP * L * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % N);
    const int64_t pl = e / N;
    const int l = (int)(pl % L);
    const int64_t p = pl / L;
    const uint64_t v = vals[p * N + j];
    out[e] = centered ? lift_centered(v, P.ell, P.q[l], P.mu[l], P.tmod[l]) : reduce64(v, P.q[l], P.mu[l]);
  }
}

// Packed scatter into a zeroed dense Z_t array (used by pb_lift with a map).
__global__ void k_unpack(PbPack s, int N, int64_t nP, uint64_t* dense) {
  const int64_t total = nP * s.Z;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = s.pos[e];
    if (j >= 0) dense[(e / s.Z) * N + j] = s.vals[s.src[e]];
  }
}

// ----------------------------------------------------------------- noise ---
// Device-only encryption randomness (fact 5: decrypted values do not depend
// on it): ternary u and centred-binomial(eta=20) e from Philox4x32-10 keyed by
// (seed, domain) with counter (coefficient, poly).
__device__ __forceinline__ int cbd20(uint32_t x, uint32_t y) {
  return __popc(x & 0xFFFFFu) - __popc(y & 0xFFFFFu);
}

__global__ void k_sample_noise(int N, int64_t nP, uint64_t seed_arg, const uint64_t* seed_dev, uint64_t nonce,
                               int with_u, int8_t* u, int8_t* e1, int8_t* e2) {
  const uint64_t seed = dev_key(seed_arg, seed_dev);
  const int64_t total = nP * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / N;
    const uint32_t j = (uint32_t)(e - p * N);
    const uint64_t pp = (uint64_t)p + nonce;
    const u32x4 r = philox4x32_10(j, (uint32_t)pp, (uint32_t)(pp >> 32), 0x454e4331u /* "ENC1" */, (uint32_t)seed,
                                  (uint32_t)(seed >> 32));
    if (with_u) {
      const u32x4 r2 = philox4x32_10(j, (uint32_t)pp, (uint32_t)(pp >> 32), 0x454e4332u, (uint32_t)seed,
                                     (uint32_t)(seed >> 32));
      u[e] = (int8_t)((int)(((uint64_t)r2.v[0] * 3ull) >> 32) - 1);
      e2[e] = (int8_t)cbd20(r2.v[1], r2.v[2]);
    }
    e1[e] = (int8_t)cbd20(r.v[0], r.v[1]);
  }
}

// --------------------------------------------------------------- encrypt ---
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5))
    k_encrypt_pk(PbDev P, const uint32_t* pk, PbPack src, int64_t nP, const int8_t* u, const int8_t* e1,
                 const int8_t* e2, uint32_t* ct) {
  using Nt = pb::Ntt<LOGN>;
  constexpr int N = Nt::N;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  const int L = P.L;
  const int l = (int)(blockIdx.x / nP);  // limb-major: co-resident CTAs share one limb's twiddles
  const int64_t p = blockIdx.x % nP;
  const uint32_t q = P.q[l];
  const uint64_t mu = P.mu[l];
  const uint2* tw = P.tw_fwd + (size_t)l * N;
  const uint2* t3 = P.tw3_fwd + (size_t)l * P.tw3_stride;
  const int8_t* up = u + p * N;
  const int8_t* e1p = e1 + p * N;
  const int8_t* e2p = e2 + p * N;

  uint32_t U[32], b[32], k[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) U[c] = lift_small(up[Nt::j1(tid, c)], q);
  Nt::forward(U, sm, tw, t3, tid, q);
#pragma unroll
  for (int c = 0; c < 32; ++c) U[c] = pb::canon4(U[c], q);  // mulmod_lt needs operands < q
  __syncthreads();
  // c1 = pk1 * U + NTT(e2)
#pragma unroll
  for (int c = 0; c < 32; ++c) b[c] = lift_small(e2p[Nt::j1(tid, c)], q);
  Nt::forward(b, sm, tw, t3, tid, q);
  Nt::gld3(pk + ((size_t)1 * L + l) * N, k, tid);
#pragma unroll
  for (int c = 0; c < 32; ++c) b[c] = addmod(mulmod_lt(k[c], U[c], q, mu), pb::canon4(b[c], q), q);
  Nt::gst3(ct + ((p * 2 + 1) * L + l) * N, b, tid);
  __syncthreads();
  // c0 = pk0 * U + NTT(e1 + Delta m)
  load_source<Nt>(b, sm, src, p, tid, [&](uint64_t v) { return delta_m(P, l, v); });
#pragma unroll
  for (int c = 0; c < 32; ++c) b[c] = addmod(lift_small(e1p[Nt::j1(tid, c)], q), b[c], q);
  Nt::forward(b, sm, tw, t3, tid, q);
  Nt::gld3(pk + (size_t)l * N, k, tid);
#pragma unroll
  for (int c = 0; c < 32; ++c) b[c] = addmod(mulmod_lt(k[c], U[c], q, mu), pb::canon4(b[c], q), q);
  Nt::gst3(ct + ((p * 2 + 0) * L + l) * N, b, tid);
}

// Uniform residue mod q for (poly, limb, coefficient-pair) from Philox4x32.
__device__ __forceinline__ void uniform_pair(uint64_t seed, uint64_t nonce, int64_t p, int l, int jpair, uint32_t q,
                                             uint32_t domain, uint32_t& x0, uint32_t& x1) {
  const uint64_t pp = (uint64_t)p + nonce;
  const u32x4 r = philox4x32_10((uint32_t)jpair | ((uint32_t)l << 24), (uint32_t)pp, (uint32_t)(pp >> 32), domain,
                                (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t a = ((uint64_t)r.v[1] << 32) | r.v[0];
  const uint64_t b = ((uint64_t)r.v[3] << 32) | r.v[2];
  x0 = (uint32_t)__umul64hi(a, q);
  x1 = (uint32_t)__umul64hi(b, q);
}

// The encryption noise e ~ CBD(20) of P polynomials, int8 [P][N], drawn ONCE
// per polynomial (it is the same integer polynomial in every RNS limb).
// Coefficient tid + T c (T = N/32, c < 32) comes from Philox4x32-10 keyed
// (seed, "ENC5") at counter ((tid << 4) | g, p + nonce), g = c / 3, three
// samples per call; one thread per call, consecutive threads consecutive tid
// (coalesced byte stores).  k_encrypt_sk's L limb CTAs then read it from L2
// instead of each redrawing it (7x less RNG work for the noise at L = 7).
__global__ void __launch_bounds__(256) k_enc_noise(int logN, int64_t nP, uint64_t seed_arg, const uint64_t* seed_dev,
                                                   uint64_t nonce, int8_t* __restrict__ e) {
  const uint64_t seed = dev_key(seed_arg, seed_dev);
  const int T = 1 << (logN - 5);
  const int64_t total = nP * 11 * T;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int tid = (int)(x & (T - 1));
    const int64_t pg = x >> (logN - 5);
    const int64_t p = pg / 11;
    const int g = (int)(pg - p * 11);
    const uint64_t pp = (uint64_t)p + nonce;
    const u32x4 r = philox4x32_10(((uint32_t)tid << 4) | (uint32_t)g, (uint32_t)pp, (uint32_t)(pp >> 32),
                                  0x454e4335u /* "ENC5" */, (uint32_t)seed, (uint32_t)(seed >> 32));
    int sv[3];
    cbd20x3(r, sv);
    int8_t* ep = e + (p << logN) + tid;
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (3 * g + i < 32) ep[(size_t)(3 * g + i) * T] = (int8_t)sv[i];
  }
}

// Symmetric encryption, one CTA per (polynomial, limb) row: c0 = NTT(e +
// Delta m) - a s, c1 = a, with e from k_enc_noise (or the caller's noise in
// the bit-exact oracle runs) and a uniform in the NTT domain drawn here (four
// residues per Philox call).  Under a launch cap (background preparation) a
// CTA loops over R consecutive rows in polynomial-major order.
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5), NTT_MINB(LOGN))
    k_encrypt_sk(PbDev P, const uint32_t* sk, const uint32_t* sk_sh, PbPack src, int64_t nP, const uint32_t* a_in,
                 const int8_t* e, uint64_t seed_arg, const uint64_t* seed_dev, uint64_t nonce, uint32_t* ct) {
  using Nt = pb::Ntt<LOGN>;
  const uint64_t seed = dev_key(seed_arg, seed_dev);
  constexpr int N = Nt::N;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  const int L = P.L;
  const int64_t rows = nP * L;
  const int64_t R = (rows + gridDim.x - 1) / gridDim.x;
  for (int64_t it = 0; it < R; ++it) {
  int l;
  int64_t p;
  if (R == 1) {
    l = (int)(blockIdx.x / nP);  // limb-major: co-resident CTAs share one limb's twiddles
    p = blockIdx.x % nP;
  } else {
    const int64_t row = blockIdx.x * R + it;
    if (row >= rows) break;
    p = row / L;
    l = (int)(row - p * L);
    if (it) __syncthreads();  // shared memory of the previous row is free
  }
  const uint32_t q = P.q[l];
  const uint64_t mu = P.mu[l];
  const int8_t* ep = e + p * N;
  uint32_t b[32];
  load_source<Nt>(b, sm, src, p, tid, [&](uint64_t v) { return delta_m(P, l, v); });
  // + e with |e| <= 20 as e + q: Delta m + e + q < 3q stays inside the NTT's lazy input range [0, 4q)
#pragma unroll
  for (int c = 0; c < 32; ++c) b[c] += (uint32_t)((int)q + ep[Nt::j1(tid, c)]);
  Nt::forward(b, sm, P.tw_fwd + (size_t)l * N, P.tw3_fwd + (size_t)l * P.tw3_stride, tid, q);
  // c1 = a, c0 = NTT(e + Delta m) - a*s, one 128-bit device-order vector at a
  // time (keeps a and s out of the register file: 32 live residues, not 96)
  const uint4* s4 = reinterpret_cast<const uint4*>(sk + (size_t)l * N) + tid;
  const uint4* h4 = sk_sh ? reinterpret_cast<const uint4*>(sk_sh + (size_t)l * N) + tid : nullptr;
  const uint4* a4 = a_in ? reinterpret_cast<const uint4*>(a_in + (p * L + l) * N) + tid : nullptr;
  uint4* c0 = reinterpret_cast<uint4*>(ct + ((p * 2 + 0) * L + l) * N) + tid;
  uint4* c1 = reinterpret_cast<uint4*>(ct + ((p * 2 + 1) * L + l) * N) + tid;
  const uint32_t q2 = 2 * q;
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    uint32_t a[4];
    if (a4) {
      const uint4 x = __ldg(a4 + v * Nt::T);
      a[0] = x.x; a[1] = x.y; a[2] = x.z; a[3] = x.w;
    } else {
      uniform_quad(seed, (uint64_t)p + nonce, l, (tid << 3) + v, q, 0x53454e44u /* "SEND" */, a);
    }
    const uint4 sv = __ldg(s4 + v * Nt::T);
    const uint32_t sk_[4] = {sv.x, sv.y, sv.z, sv.w};
    uint32_t o[4];
    if (h4) {  // Shoup with the key's companion row: c0 = b - a s over lazy ranges, one canonicalisation
      const uint4 hv = __ldg(h4 + v * Nt::T);
      const uint32_t sh_[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t bb = min(b[4 * v + k], b[4 * v + k] - q2);           // [0, 2q)
        const uint32_t t = mul_shoup_lazy(a[k], sk_[k], sh_[k], q);          // [0, 2q)
        o[k] = pb::canon4(bb - t + q2, q);                                    // (0, 4q) -> [0, q)
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = submod(pb::canon4(b[4 * v + k], q), mulmod_lt(a[k], sk_[k], q, mu), q);
    }
    c0[v * Nt::T] = make_uint4(o[0], o[1], o[2], o[3]);
    c1[v * Nt::T] = make_uint4(a[0], a[1], a[2], a[3]);
  }
  }
}

// Split symmetric encryption.  The message-independent part of
// k_encrypt_sk -- a (uniform, NTT domain), -a*s and the noise e -- is
// precomputed elementwise by k_encrypt_pre (no NTT: one thread per 128-bit
// device-order quad, e drawn once per polynomial instead of once per limb);
// k_encrypt_add then does the message-dependent rest on the critical path:
// c0 = -a*s + NTT(e + Delta m).  Same a as k_encrypt_sk under (seed, nonce),
// so k_encrypt_add(pre) == k_encrypt_sk with caller noise (a, e) bit for bit.
// grid (ceil(N/4 / 256), L, nP): one thread per 128-bit device-order quad.
__global__ void __launch_bounds__(256) k_encrypt_pre(PbDev P, const uint32_t* sk, uint64_t seed_arg,
                                                     const uint64_t* seed_dev, uint64_t nonce, uint32_t* ct,
                                                     int8_t* e) {
  const uint64_t seed = dev_key(seed_arg, seed_dev);
  const int N = P.N, L = P.L, T = N >> 5;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;  // quad k = v*T + tid of the row, as k_encrypt_sk's stores
  if (k >= (N >> 2)) return;
  const int l = blockIdx.y;
  const int64_t p = blockIdx.z;
  const int v = k / T, tid = k - v * T;
  const uint32_t q = P.q[l];
  const uint64_t mu = P.mu[l];
  const uint64_t pp = (uint64_t)p + nonce;
  uint32_t a[4];
  uniform_quad(seed, pp, l, (tid << 3) + v, q, 0x53454e44u /* "SEND" */, a);
  const uint4 sv = __ldg(reinterpret_cast<const uint4*>(sk + (size_t)l * N) + k);
  const uint32_t sk_[4] = {sv.x, sv.y, sv.z, sv.w};
  uint32_t o[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) o[c] = submod(0u, mulmod_lt(a[c], sk_[c], q, mu), q);
  reinterpret_cast<uint4*>(ct + ((p * 2 + 0) * L + l) * N)[k] = make_uint4(o[0], o[1], o[2], o[3]);
  reinterpret_cast<uint4*>(ct + ((p * 2 + 1) * L + l) * N)[k] = make_uint4(a[0], a[1], a[2], a[3]);
  if (l == 0 && k < (N + 11) / 12) {  // e ~ CBD(20), once per polynomial: coefficients 12k .. 12k+11
    int8_t* ep = e + p * N + 12 * k;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const u32x4 r = philox4x32_10(4u * k + g, (uint32_t)pp, (uint32_t)(pp >> 32), 0x454e4334u /* "ENC4" */,
                                    (uint32_t)seed, (uint32_t)(seed >> 32));
      int sv[3];
      cbd20x3(r, sv);
#pragma unroll
      for (int i = 0; i < 3; ++i)
        if (12 * k + 3 * g + i < N) ep[3 * g + i] = (int8_t)sv[i];
    }
  }
}

template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5), NTT_MINB(LOGN))
    k_encrypt_add(PbDev P, PbPack src, int64_t nP, const int8_t* e, uint32_t* ct) {
  using Nt = pb::Ntt<LOGN>;
  constexpr int N = Nt::N;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  const int L = P.L;
  const int l = (int)(blockIdx.x / nP);  // limb-major: co-resident CTAs share one limb's twiddles
  const int64_t p = blockIdx.x % nP;
  const uint32_t q = P.q[l];
  uint4* c0 = reinterpret_cast<uint4*>(ct + ((p * 2 + 0) * L + l) * N) + tid;
#pragma unroll
  for (int v = 0; v < 8; ++v) asm volatile("prefetch.global.L2 [%0];" ::"l"(c0 + v * Nt::T));
  const int8_t* ep = e + p * N;
  uint32_t b[32];
  load_source<Nt>(b, sm, src, p, tid, [&](uint64_t v) { return delta_m(P, l, v); });
#pragma unroll
  for (int c = 0; c < 32; ++c) b[c] = addmod(lift_small(ep[Nt::j1(tid, c)], q), b[c], q);
  Nt::forward(b, sm, P.tw_fwd + (size_t)l * N, P.tw3_fwd + (size_t)l * P.tw3_stride, tid, q);
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const uint4 x = c0[v * Nt::T];
    c0[v * Nt::T] = make_uint4(addmod(x.x, pb::canon4(b[4 * v], q), q), addmod(x.y, pb::canon4(b[4 * v + 1], q), q),
                               addmod(x.z, pb::canon4(b[4 * v + 2], q), q),
                               addmod(x.w, pb::canon4(b[4 * v + 3], q), q));
  }
}

// Number of low index bits (<= 5) that are 1 in every useful slot of a ciphertext:
// its inverse NTT can be output-pruned by that many stages (Ntt::inverse_pruned).
// Block-wide AND over the slot list; `flag` is a shared int (synchronised).
template <class Nt>
__device__ __forceinline__ int common_low_ones(const int32_t* pos, int U, int tid, int* flag) {
  if (tid == 0) *flag = -1;
  __syncthreads();
  int acc = -1;
  for (int u0 = tid; u0 < U; u0 += 8 * Nt::T) {  // batched: eight independent loads in flight
    int j[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) j[k] = u0 + k * Nt::T < U ? __ldg(pos + u0 + k * Nt::T) : -1;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (j[k] >= 0) acc &= j[k];
  }
  if (acc != -1) atomicAnd(flag, acc);
  __syncthreads();
  const int v = *flag;
  __syncthreads();
  int t = 0;
  while (t < 5 && ((v >> t) & 1)) ++t;
  // one pruned stage leaves N/2 values for the shared-memory stages: slower than
  // the register inverse (B200: U = 4096 x 2 cts 11.7 -> 15.1 us); from two on it pays
  return t >= 2 ? t : 0;
}

// inverse_scaled, or the output-pruned inverse for TT common low one-bits:
// returns TT (0: full inverse, result in a[] in P1 layout; else the compact
// array A[n >> TT] in sm).
template <class Nt>
__device__ __forceinline__ int inverse_for_slots(uint32_t (&a)[32], uint32_t* sm, const PbDev& P, int l, int tid,
                                                 uint32_t q, int tt) {
  const uint2* tw = P.tw_inv + (size_t)l * Nt::N;
  const uint2* t3 = P.tw3_inv + (size_t)l * P.tw3_stride;
  const uint32_t ni = P.ninv[l], nis = P.ninv_sh[l], wn = P.w0n[l], wns = P.w0n_sh[l];
  switch (tt) {
    case 1: Nt::template inverse_pruned<1>(a, sm, tw, t3, tid, q, ni, nis, wn, wns); return 1;
    case 2: Nt::template inverse_pruned<2>(a, sm, tw, t3, tid, q, ni, nis, wn, wns); return 2;
    case 3: Nt::template inverse_pruned<3>(a, sm, tw, t3, tid, q, ni, nis, wn, wns); return 3;
    case 4: Nt::template inverse_pruned<4>(a, sm, tw, t3, tid, q, ni, nis, wn, wns); return 4;
    case 5: Nt::template inverse_pruned<5>(a, sm, tw, t3, tid, q, ni, nis, wn, wns); return 5;
    default: Nt::inverse_scaled(a, sm, tw, t3, tid, q, ni, nis, wn, wns); return 0;
  }
}

// --------------------------------------------------------------- decrypt ---
// mode 0: write x = INTT(c0 + c1 s) for all coefficients to out32 [P][L][N].
// mode 1: write only the useful slots out_pos[p][u] to out32 [P][L][U].
// (MODE a template parameter: one inverse-NTT body per kernel in the
// instruction stream, not both.)
template <int LOGN, int MODE>
__global__ void __launch_bounds__(1 << (LOGN - 5))
    k_decrypt_inv(PbDev P, const uint32_t* sk, const uint32_t* ct, int64_t nP, const int32_t* out_pos,
                  int U, uint32_t* out32) {
  using Nt = pb::Ntt<LOGN>;
  constexpr int N = Nt::N;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  const int L = P.L;
  const int l = (int)(blockIdx.x / nP);  // limb-major: co-resident CTAs share one limb's twiddles
  const int64_t p = blockIdx.x % nP;
  const uint32_t q = P.q[l];
  const uint64_t mu = P.mu[l];
  uint32_t a[32], b[32];
  Nt::gld3(ct + ((p * 2 + 1) * L + l) * N, a, tid);
  Nt::gld3(sk + (size_t)l * N, b, tid);
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = mulmod_lt(a[c], b[c], q, mu);
  Nt::gld3(ct + ((p * 2 + 0) * L + l) * N, b, tid);
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = addmod(a[c], b[c], q);
  if constexpr (MODE == 0) {
    const uint32_t ni = P.ninv[l], nis = P.ninv_sh[l];
    Nt::inverse_scaled(a, sm, P.tw_inv + (size_t)l * N, P.tw3_inv + (size_t)l * P.tw3_stride, tid, q, ni, nis,
                       P.w0n[l], P.w0n_sh[l]);
    Nt::gst1(out32 + (p * L + l) * N, a, tid);
  } else {
    const int32_t* pos = out_pos + p * U;
    const int tt = inverse_for_slots<Nt>(a, sm, P, l, tid, q,
                                         common_low_ones<Nt>(pos, U, tid, reinterpret_cast<int*>(sm + Nt::TW_OFF)));
    if (tt == 0) {
      __syncthreads();
      Nt::st1(sm, a, tid);
    }
    __syncthreads();
    uint32_t* dst = out32 + (p * L + l) * U;
    for (int u0 = tid; u0 < U; u0 += 8 * Nt::T) {  // batched position loads
      int j[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) j[k] = u0 + k * Nt::T < U ? __ldg(pos + u0 + k * Nt::T) : -1;
#pragma unroll
      for (int k = 0; k < 8; ++k)  // already scaled by N^-1
        if (j[k] >= 0) dst[u0 + k * Nt::T] = tt ? sm[j[k] >> tt] : sm[Nt::pad(j[k])];
    }
  }
}

__device__ __forceinline__ void garner_dev(const PbDev& P, const uint32_t* x, int64_t xs, uint32_t (&d)[PB_MAXL]) {
#pragma unroll
  for (int i = 0; i < PB_MAXL; ++i) {
    if (i < P.L) {
      const uint32_t qi = P.q[i];
      const uint64_t mu = P.mu[i];
      uint32_t acc = 0;
#pragma unroll
      for (int k = 0; k < PB_MAXL; ++k)
        if (k < i) acc = addmod(acc, mul_shoup(d[k], P.pmod[i][k], P.pmod_sh[i][k], qi), qi);
      const uint32_t xv = reduce64(x[i * xs], qi, mu);
      d[i] = mul_shoup(submod(xv, acc, qi), P.pinv[i], P.pinv_sh[i], qi);
    }
  }
}

__device__ __forceinline__ uint64_t scale_round_dev(const PbDev& P, const uint32_t (&d)[PB_MAXL]) {
  uint64_t acc_i = 0;
  double acc_f = 0.0;
#pragma unroll
  for (int i = 0; i < PB_MAXL; ++i) {
    if (i < P.L) {
      acc_i += (uint64_t)d[i] * P.sc_int[i];
      acc_f = __dadd_rn(acc_f, __dmul_rn((double)d[i], P.sc_frac[i]));
    }
  }
  return (acc_i + (uint64_t)floor(__dadd_rn(acc_f, 0.5))) & P.t_mask;
}

// Garner + scale-round on the gathered slots, scattered into the share tensor.
__global__ void k_decode_gather(PbDev P, const uint32_t* x, int64_t nP, int U, const int32_t* out_pos,
                                const int64_t* out_dst, uint64_t* share) {
  const int L = P.L;
  const int64_t total = nP * U;
  if (total < (1ll << 31)) {  // 32-bit slot arithmetic (a 64-bit division per slot was a large share of the kernel)
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < (uint32_t)total; e += gridDim.x * blockDim.x) {
      if (out_pos[e] < 0) continue;
      const uint32_t p = e / (uint32_t)U, u = e - p * (uint32_t)U;
      uint32_t d[PB_MAXL];
      garner_dev(P, x + (uint64_t)p * L * U + u, U, d);
      share[out_dst[e]] = scale_round_dev(P, d);
    }
    return;
  }
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    if (out_pos[e] < 0) continue;
    const int64_t p = e / U;
    const int u = (int)(e - p * U);
    uint32_t d[PB_MAXL];
    garner_dev(P, x + p * L * U + u, U, d);
    share[out_dst[e]] = scale_round_dev(P, d);
  }
}

// Fused decrypt-to-share: one thread-block CLUSTER of L CTAs per output
// ciphertext, CTA l = limb l.  Each CTA computes x_l = INTT(c0 + c1 s) * N^-1
// for its limb and leaves the row in its shared memory; after a cluster
// barrier every CTA decodes a 1/L share of the useful slots, reading the L
// residues of a coefficient straight from the L CTAs' shared memory (DSMEM),
// Garner + scale-round (K:158-199), and writes the share element (pi_y^-1).
// Replaces k_decrypt_inv (mode 1) + k_decode_gather: one launch, no scratch.
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5))
    k_decrypt_share_cluster(PbDev P, const uint32_t* sk, const uint32_t* ct, int64_t nP, const int32_t* out_pos,
                            const int64_t* out_dst, int U, uint64_t* share) {
  namespace cg = cooperative_groups;
  using Nt = pb::Ntt<LOGN>;
  constexpr int N = Nt::N;
  extern __shared__ uint32_t sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x;
  const int L = P.L;
  const int l = (int)cluster.block_rank();
  const int64_t p = blockIdx.x / L;
  const uint32_t q = P.q[l];
  const uint64_t mu = P.mu[l];
  uint32_t a[32], b[32];
  Nt::gld3(ct + ((p * 2 + 1) * L + l) * N, a, tid);
  Nt::gld3(sk + (size_t)l * N, b, tid);
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = mulmod_lt(a[c], b[c], q, mu);
  Nt::gld3(ct + ((p * 2 + 0) * L + l) * N, b, tid);
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = addmod(a[c], b[c], q);
  const int32_t* pos = out_pos + p * U;
  const int tt = inverse_for_slots<Nt>(a, sm, P, l, tid, q,
                                       common_low_ones<Nt>(pos, U, tid, reinterpret_cast<int*>(sm + Nt::TW_OFF)));
  if (tt == 0) {
    __syncthreads();
    Nt::st1(sm, a, tid);
  }
  cluster.sync();  // every limb's row (or its compact useful part) is in its CTA's shared memory
  const uint32_t* rows[PB_MAXL];
#pragma unroll
  for (int k = 0; k < PB_MAXL; ++k) rows[k] = k < L ? cluster.map_shared_rank(sm, k) : nullptr;
  const int64_t* dst = out_dst + p * U;
  // CTA l decodes the contiguous block [u0, u1) of the useful slots (balanced
  // across the cluster: a strided split left the remainder to one CTA, whose
  // peers then idled at the closing barrier), two slots per thread per pass
  // with both slots' loads in flight together
  const int per = (U + L - 1) / L;
  const int u0 = l * per, u1 = min(U, u0 + per);
  for (int u = u0 + tid; u < u1; u += 2 * Nt::T) {
    const int ub = u + Nt::T;
    const int ja = __ldg(pos + u), jb = ub < u1 ? __ldg(pos + ub) : -1;
    const int64_t da = __ldg(dst + u), db = ub < u1 ? __ldg(dst + ub) : 0;
    uint32_t xa[PB_MAXL], xb[PB_MAXL], d[PB_MAXL];
    const int ia = ja < 0 ? 0 : (tt ? ja >> tt : Nt::pad(ja)), ib = jb < 0 ? 0 : (tt ? jb >> tt : Nt::pad(jb));
#pragma unroll
    for (int k = 0; k < PB_MAXL; ++k) {
      xa[k] = (k < L && ja >= 0) ? rows[k][ia] : 0u;
      xb[k] = (k < L && jb >= 0) ? rows[k][ib] : 0u;
    }
    if (ja >= 0) {
      garner_dev(P, xa, 1, d);
      share[da] = scale_round_dev(P, d);
    }
    if (jb >= 0) {
      garner_dev(P, xb, 1, d);
      share[db] = scale_round_dev(P, d);
    }
  }
  cluster.sync();  // peers may still be reading this CTA's shared memory
}

__global__ void k_decode_dense(PbDev P, const uint32_t* x, int64_t nP, uint64_t* out) {
  const int N = P.N, L = P.L;
  const int64_t total = nP * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / N;
    const int j = (int)(e - p * N);
    uint32_t d[PB_MAXL];
    garner_dev(P, x + p * L * N + j, N, d);
    out[e] = scale_round_dev(P, d);
  }
}

// ------------------------------------------------------------- MO: MAC ---
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5))
    k_ctpt_mac_mask(PbDev P, const uint32_t* ct_in, const uint32_t* pt, const uint32_t* pt_sh, const int32_t* terms,
                    int K, int64_t nP, const int32_t* out_pos, const int64_t* out_dst, int U, const uint64_t* mask_vals,
                    int filler, uint64_t filler_arg, const uint64_t* seed_dev, uint32_t* ct_out) {
  using Nt = pb::Ntt<LOGN>;
  const uint64_t filler_seed = dev_key(filler_arg, seed_dev);
  constexpr int N = Nt::N;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  const int L = P.L;
  const int l = (int)(blockIdx.x / nP);  // limb-major: co-resident CTAs share one limb's twiddles
  const int64_t p = blockIdx.x % nP;
  const uint32_t q = P.q[l];

  // 1. Delta * mask polynomial (coefficient form) in shared memory.
  if (filler) {
    for (int jp = tid; jp < N / 2; jp += Nt::T) {
      uint32_t x0, x1;
      uniform_pair(filler_seed, 0, p, l, jp, q, 0x4d41534bu /* "MASK" */, x0, x1);
      sm[Nt::pad(2 * jp)] = x0;
      sm[Nt::pad(2 * jp + 1)] = x1;
    }
  } else {
    for (int j = tid; j < N; j += Nt::T) sm[Nt::pad(j)] = 0u;
  }
  __syncthreads();
  if (mask_vals) {
    const int32_t* pos = out_pos + p * U;
    const int64_t* dst = out_dst + p * U;
    for (int u = tid; u < U; u += Nt::T) {
      const int j = pos[u];
      if (j >= 0) sm[Nt::pad(j)] = delta_m(P, l, __ldg(mask_vals + dst[u]));
    }
  }
  __syncthreads();
  uint32_t m[32];
  Nt::ld1(sm, m, tid);
  __syncthreads();
  Nt::forward(m, sm, P.tw_fwd + (size_t)l * N, P.tw3_fwd + (size_t)l * P.tw3_stride, tid, q);

  // 2. MAC over the K (ct, pt) terms, one 128-bit device-order vector at a
  //    time (P3 register v <-> uint4 #(v*T + tid) of the row), then
  //    subtract the mask and store.
  const size_t rowoff = (size_t)l * N;
  uint4* o0 = reinterpret_cast<uint4*>(ct_out + ((size_t)p * 2 + 0) * L * N + rowoff) + tid;
  uint4* o1 = reinterpret_cast<uint4*>(ct_out + ((size_t)p * 2 + 1) * L * N + rowoff) + tid;
  const int32_t* tp = terms + p * K * 2;
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    uint32_t a0[4] = {0u, 0u, 0u, 0u}, a1[4] = {0u, 0u, 0u, 0u};
    for (int kk = 0; kk < K; ++kk) {
      const int ci = __ldg(tp + 2 * kk), pi = __ldg(tp + 2 * kk + 1);
      if (ci < 0) continue;
      const size_t vo = (size_t)v * Nt::T + tid;
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(pt + (size_t)pi * L * N + rowoff) + vo);
      const uint4 ws = __ldg(reinterpret_cast<const uint4*>(pt_sh + (size_t)pi * L * N + rowoff) + vo);
      const uint4 x0 = __ldg(reinterpret_cast<const uint4*>(ct_in + ((size_t)ci * 2 + 0) * L * N + rowoff) + vo);
      const uint4 x1 = __ldg(reinterpret_cast<const uint4*>(ct_in + ((size_t)ci * 2 + 1) * L * N + rowoff) + vo);
      a0[0] = addmod(a0[0], mul_shoup(x0.x, w.x, ws.x, q), q);
      a0[1] = addmod(a0[1], mul_shoup(x0.y, w.y, ws.y, q), q);
      a0[2] = addmod(a0[2], mul_shoup(x0.z, w.z, ws.z, q), q);
      a0[3] = addmod(a0[3], mul_shoup(x0.w, w.w, ws.w, q), q);
      a1[0] = addmod(a1[0], mul_shoup(x1.x, w.x, ws.x, q), q);
      a1[1] = addmod(a1[1], mul_shoup(x1.y, w.y, ws.y, q), q);
      a1[2] = addmod(a1[2], mul_shoup(x1.z, w.z, ws.z, q), q);
      a1[3] = addmod(a1[3], mul_shoup(x1.w, w.w, ws.w, q), q);
    }
    o0[v * Nt::T] = make_uint4(submod(a0[0], pb::canon4(m[4 * v + 0], q), q), submod(a0[1], pb::canon4(m[4 * v + 1], q), q),
                               submod(a0[2], pb::canon4(m[4 * v + 2], q), q), submod(a0[3], pb::canon4(m[4 * v + 3], q), q));
    o1[v * Nt::T] = make_uint4(a1[0], a1[1], a1[2], a1[3]);
  }
}

// ------------------------------------------------------------- launchers ---
template <typename KernelT>
static void set_smem(KernelT k, size_t smem) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <int LOGN>
void launch_encode_plain(const PbDev& P, PbPack src, int64_t nP, uint32_t* pt, uint32_t* pt_sh, cudaStream_t st) {
  using Nt = pb::Ntt<LOGN>;
  const size_t smem = Nt::SMEM_WORDS * 4;
  set_smem(k_encode_plain<LOGN>, smem);
  k_encode_plain<LOGN><<<(unsigned)(nP * P.L), Nt::T, smem, st>>>(P, src, nP, pt, pt_sh);
}

template <int LOGN>
void launch_encrypt_pk(const PbDev& P, const uint32_t* pk, PbPack src, int64_t nP, const int8_t* u, const int8_t* e1,
                       const int8_t* e2, uint32_t* ct, cudaStream_t st) {
  using Nt = pb::Ntt<LOGN>;
  const size_t smem = Nt::SMEM_WORDS * 4;
  set_smem(k_encrypt_pk<LOGN>, smem);
  k_encrypt_pk<LOGN><<<(unsigned)(nP * P.L), Nt::T, smem, st>>>(P, pk, src, nP, u, e1, e2, ct);
}

template <int LOGN>
void launch_encrypt_sk(const PbDev& P, const uint32_t* sk, const uint32_t* sk_sh, PbPack src, int64_t nP,
                       const uint32_t* a_in, const int8_t* e, uint64_t seed, const uint64_t* seed_dev, uint64_t nonce,
                       uint32_t* ct, cudaStream_t st) {
  using Nt = pb::Ntt<LOGN>;
  const int64_t grid = pb_row_grid(nP * P.L);
  const size_t smem = Nt::SMEM_WORDS * 4;
  set_smem(k_encrypt_sk<LOGN>, smem);
  k_encrypt_sk<LOGN><<<(unsigned)grid, Nt::T, smem, st>>>(P, sk, sk_sh, src, nP, a_in, e, seed, seed_dev, nonce, ct);
}

template <int LOGN>
void launch_encrypt_add(const PbDev& P, PbPack src, int64_t nP, const int8_t* e, uint32_t* ct, cudaStream_t st) {
  using Nt = pb::Ntt<LOGN>;
  const size_t smem = Nt::SMEM_WORDS * 4;
  set_smem(k_encrypt_add<LOGN>, smem);
  k_encrypt_add<LOGN><<<(unsigned)(nP * P.L), Nt::T, smem, st>>>(P, src, nP, e, ct);
}

template <int LOGN>
int launch_decrypt_share_cluster(const PbDev& P, const uint32_t* sk, const uint32_t* ct, int64_t nP,
                                 const int32_t* out_pos, const int64_t* out_dst, int U, uint64_t* share,
                                 cudaStream_t st) {
  using Nt = pb::Ntt<LOGN>;
  const size_t smem = Nt::SMEM_WORDS * 4;
  set_smem(k_decrypt_share_cluster<LOGN>, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nP * P.L));
  cfg.blockDim = dim3(Nt::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)P.L;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, k_decrypt_share_cluster<LOGN>, P, sk, ct, nP, out_pos, out_dst, U, share);
}

template <int LOGN>
void launch_decrypt_inv(const PbDev& P, const uint32_t* sk, const uint32_t* ct, int64_t nP, int mode,
                        const int32_t* out_pos, int U, uint32_t* out32, cudaStream_t st) {
  using Nt = pb::Ntt<LOGN>;
  const size_t smem = Nt::SMEM_WORDS * 4;
  if (mode == 0) {
    set_smem(k_decrypt_inv<LOGN, 0>, smem);
    k_decrypt_inv<LOGN, 0><<<(unsigned)(nP * P.L), Nt::T, smem, st>>>(P, sk, ct, nP, out_pos, U, out32);
  } else {
    set_smem(k_decrypt_inv<LOGN, 1>, smem);
    k_decrypt_inv<LOGN, 1><<<(unsigned)(nP * P.L), Nt::T, smem, st>>>(P, sk, ct, nP, out_pos, U, out32);
  }
}

template <int LOGN>
void launch_mac(const PbDev& P, const uint32_t* ct_in, const uint32_t* pt, const uint32_t* pt_sh, const int32_t* terms,
                int K, int64_t nP, const int32_t* out_pos, const int64_t* out_dst, int U, const uint64_t* mask_vals,
                int filler, uint64_t filler_seed, const uint64_t* seed_dev, uint32_t* ct_out, cudaStream_t st) {
  using Nt = pb::Ntt<LOGN>;
  const size_t smem = Nt::SMEM_WORDS * 4;
  set_smem(k_ctpt_mac_mask<LOGN>, smem);
  k_ctpt_mac_mask<LOGN><<<(unsigned)(nP * P.L), Nt::T, smem, st>>>(P, ct_in, pt, pt_sh, terms, K, nP, out_pos, out_dst,
                                                                   U, mask_vals, filler, filler_seed, seed_dev, ct_out);
}

int need_big_n(const pb_ctx* ctx) {
  if (!ctx) return pb_set_error(PB_ERR_ARG, "null context");
  if (ctx->dev.logN < 11) return pb_set_error(PB_ERR_PARAMS, "fused BFV kernels need N >= 2048");
  return PB_OK;
}

int64_t max_grid_polys(const pb_ctx* ctx) { return (int64_t)0x7fffffff / ctx->dev.L; }

int make_pack(const uint64_t* vals, const int32_t* pos, const int32_t* src, int32_t Z, PbPack* out) {
  if (!vals) return pb_set_error(PB_ERR_ARG, "null plaintext source");
  if (pos && (!src || Z < 0)) return pb_set_error(PB_ERR_ARG, "packed source needs pos, src and Z >= 0");
  out->vals = vals;
  out->pos = pos;
  out->src = src;
  out->Z = pos ? Z : 0;
  return PB_OK;
}

// Scratch for device-sampled noise: a per-thread cached buffer reused
// across calls (stream-ordered use only).
}  // namespace

// ================================================================ C ABI ===
#define PB_PACK_OR_RETURN(pk, vals, pos, src, Z) \
  PbPack pk;                                     \
  if (int _s = make_pack(vals, pos, src, Z, &pk)) return _s

extern "C" int pb_encode_plain(const pb_ctx* ctx, const uint64_t* vals, const int32_t* pack_pos,
                               const int32_t* pack_src, int32_t Z, int64_t nP, uint32_t* pt, uint32_t* pt_shoup,
                               void* stream) {
  if (int s = need_big_n(ctx)) return s;
  if (nP <= 0) return PB_OK;
  if (!pt) return pb_set_error(PB_ERR_ARG, "null argument");
  if (nP > max_grid_polys(ctx)) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  PB_PACK_OR_RETURN(src, vals, pack_pos, pack_src, Z);
  PB_DISPATCH_LOGN(ctx->dev.logN, launch_encode_plain, ctx->dev, src, nP, pt, pt_shoup, pb_stream_of(stream));
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_lift(const pb_ctx* ctx, const uint64_t* vals, int64_t nP, int centered, uint32_t* out, void* stream) {
  if (!ctx) return pb_set_error(PB_ERR_ARG, "null context");
  if (nP <= 0) return PB_OK;
  if (!vals || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  k_lift<<<pb_grid_1d(nP * ctx->dev.L * ctx->dev.N, 256), 256, 0, pb_stream_of(stream)>>>(ctx->dev, vals, nP, centered,
                                                                                          out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_unpack(const uint64_t* vals, const int32_t* pack_pos, const int32_t* pack_src, int32_t Z, int32_t N,
                         int64_t nP, uint64_t* dense, void* stream) {
  if (nP <= 0 || Z <= 0) return PB_OK;
  if (!dense || N <= 0) return pb_set_error(PB_ERR_ARG, "null argument");
  PB_PACK_OR_RETURN(src, vals, pack_pos, pack_src, Z);
  if (!pack_pos) return pb_set_error(PB_ERR_ARG, "pb_unpack needs a packed source");
  k_unpack<<<pb_grid_1d(nP * Z, 256), 256, 0, pb_stream_of(stream)>>>(src, N, nP, dense);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_encrypt_pk_noise(const pb_ctx* ctx, const uint32_t* pk, const uint64_t* vals,
                                   const int32_t* pack_pos, const int32_t* pack_src, int32_t Z, int64_t nP,
                                   const int8_t* u, const int8_t* e1, const int8_t* e2, uint32_t* ct, void* stream) {
  if (int s = need_big_n(ctx)) return s;
  if (nP <= 0) return PB_OK;
  if (!pk || !u || !e1 || !e2 || !ct) return pb_set_error(PB_ERR_ARG, "null argument");
  if (nP > max_grid_polys(ctx)) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  PB_PACK_OR_RETURN(src, vals, pack_pos, pack_src, Z);
  PB_DISPATCH_LOGN(ctx->dev.logN, launch_encrypt_pk, ctx->dev, pk, src, nP, u, e1, e2, ct, pb_stream_of(stream));
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_encrypt_pk(const pb_ctx* ctx, const uint32_t* pk, const uint64_t* vals, const int32_t* pack_pos,
                             const int32_t* pack_src, int32_t Z, int64_t nP, uint64_t seed, const uint64_t* seed_dev,
                             uint64_t nonce, uint32_t* ct, void* stream) {
  if (int s = need_big_n(ctx)) return s;
  if (nP <= 0) return PB_OK;
  const int N = ctx->dev.N;
  cudaStream_t st = pb_stream_of(stream);
  int8_t* buf = nullptr;  // stream-ordered scratch: safe under concurrent streams and graph capture
  if (cudaMallocAsync((void**)&buf, (size_t)nP * N * 3, st) != cudaSuccess)
    return pb_set_error(PB_ERR_CUDA, "noise scratch allocation failed");
  int8_t *u = buf, *e1 = buf + nP * N, *e2 = buf + 2 * nP * N;
  k_sample_noise<<<pb_grid_1d(nP * N, 256), 256, 0, st>>>(N, nP, seed, seed_dev, nonce, 1, u, e1, e2);
  PB_CHECK_LAUNCH();
  const int rc = pb_encrypt_pk_noise(ctx, pk, vals, pack_pos, pack_src, Z, nP, u, e1, e2, ct, stream);
  cudaFreeAsync(buf, st);
  return rc;
}

extern "C" int pb_encrypt_sk_noise(const pb_ctx* ctx, const uint32_t* sk, const uint64_t* vals,
                                   const int32_t* pack_pos, const int32_t* pack_src, int32_t Z, int64_t nP,
                                   const uint32_t* a, const int8_t* e, uint32_t* ct, void* stream) {
  if (int s = need_big_n(ctx)) return s;
  if (nP <= 0) return PB_OK;
  if (!sk || !e || !ct) return pb_set_error(PB_ERR_ARG, "null argument");
  if (nP > max_grid_polys(ctx)) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  PB_PACK_OR_RETURN(src, vals, pack_pos, pack_src, Z);
  PB_DISPATCH_LOGN(ctx->dev.logN, launch_encrypt_sk, ctx->dev, sk, (const uint32_t*)nullptr, src, nP, a, e, 0ull,
                   (const uint64_t*)nullptr, 0ull, ct, pb_stream_of(stream));
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_encrypt_sk(const pb_ctx* ctx, const uint32_t* sk, const uint32_t* sk_shoup, const uint64_t* vals,
                             const int32_t* pack_pos, const int32_t* pack_src, int32_t Z, int64_t nP, uint64_t seed,
                             const uint64_t* seed_dev, uint64_t nonce, uint32_t* ct, void* stream) {
  if (int s = need_big_n(ctx)) return s;
  if (nP <= 0) return PB_OK;
  if (!sk || !ct) return pb_set_error(PB_ERR_ARG, "null argument");
  if (nP > max_grid_polys(ctx)) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  PB_PACK_OR_RETURN(src, vals, pack_pos, pack_src, Z);
  cudaStream_t st = pb_stream_of(stream);
  // the noise polynomials first (stream-ordered scratch, graph-capturable)
  int8_t* e = nullptr;
  if (cudaMallocAsync((void**)&e, (size_t)nP << ctx->dev.logN, st) != cudaSuccess)
    return pb_set_error(PB_ERR_CUDA, "encryption noise scratch allocation failed");
  const int64_t thr = (nP * 11) << (ctx->dev.logN - 5);
  k_enc_noise<<<pb_row_grid((thr + 255) / 256), 256, 0, st>>>(ctx->dev.logN, nP, seed, seed_dev, nonce, e);
  PB_DISPATCH_LOGN(ctx->dev.logN, launch_encrypt_sk, ctx->dev, sk, sk_shoup, src, nP, (const uint32_t*)nullptr,
                   (const int8_t*)e, seed, seed_dev, nonce, ct, st);
  cudaFreeAsync(e, st);
  PB_CHECK_LAUNCH();
  return PB_OK;
}
extern "C" int pb_encrypt_sk_zero(const pb_ctx* ctx, const uint32_t* sk, int64_t nP, uint64_t seed,
                                  const uint64_t* seed_dev, uint64_t nonce, uint32_t* ct, int8_t* e, void* stream) {
  if (int s = need_big_n(ctx)) return s;
  if (nP <= 0) return PB_OK;
  if (!sk || !ct || !e) return pb_set_error(PB_ERR_ARG, "null argument");
  if (nP > max_grid_polys(ctx)) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  if (nP > 65535) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  const dim3 grid((unsigned)((ctx->dev.N / 4 + 255) / 256), (unsigned)ctx->dev.L, (unsigned)nP);
  k_encrypt_pre<<<grid, 256, 0, pb_stream_of(stream)>>>(ctx->dev, sk, seed, seed_dev, nonce, ct, e);
  PB_CHECK_LAUNCH();
  return PB_OK;
}
extern "C" int pb_encrypt_sk_add(const pb_ctx* ctx, const uint64_t* vals, const int32_t* pack_pos,
                                 const int32_t* pack_src, int32_t Z, int64_t nP, const int8_t* e, uint32_t* ct,
                                 void* stream) {
  if (int s = need_big_n(ctx)) return s;
  if (nP <= 0) return PB_OK;
  if (!ct || !e) return pb_set_error(PB_ERR_ARG, "null argument");
  if (nP > max_grid_polys(ctx)) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  PB_PACK_OR_RETURN(src, vals, pack_pos, pack_src, Z);
  PB_DISPATCH_LOGN(ctx->dev.logN, launch_encrypt_add, ctx->dev, src, nP, e, ct, pb_stream_of(stream));
  PB_CHECK_LAUNCH();
  return PB_OK;
}
extern "C" int pb_decrypt_coeffs(const pb_ctx* ctx, const uint32_t* sk, const uint32_t* ct, int64_t nP, uint32_t* x,
                                 void* stream) {
  if (int s = need_big_n(ctx)) return s;
  if (!sk || !ct || !x) return pb_set_error(PB_ERR_ARG, "null argument");
  if (nP <= 0) return PB_OK;
  if (nP > max_grid_polys(ctx)) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  PB_DISPATCH_LOGN(ctx->dev.logN, launch_decrypt_inv, ctx->dev, sk, ct, nP, 0, (const int32_t*)nullptr, 0, x,
                   pb_stream_of(stream));
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_decrypt(const pb_ctx* ctx, const uint32_t* sk, const uint32_t* ct, int64_t nP, uint64_t* m,
                          uint32_t* scratch, void* stream) {
  if (int s = pb_decrypt_coeffs(ctx, sk, ct, nP, scratch, stream)) return s;
  if (nP <= 0) return PB_OK;
  if (!m) return pb_set_error(PB_ERR_ARG, "null argument");
  k_decode_dense<<<pb_grid_1d(nP * ctx->dev.N, 256), 256, 0, pb_stream_of(stream)>>>(ctx->dev, scratch, nP, m);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_decrypt_to_share(const pb_ctx* ctx, const uint32_t* sk, const uint32_t* ct, int64_t nP,
                                   const int32_t* out_pos, const int64_t* out_dst, int32_t U, uint64_t* share_out,
                                   uint32_t* scratch, void* stream) {
  if (int s = need_big_n(ctx)) return s;
  if (!sk || !ct || !out_pos || !out_dst || !share_out || !scratch) return pb_set_error(PB_ERR_ARG, "null argument");
  if (nP <= 0 || U <= 0) return PB_OK;
  if (nP > max_grid_polys(ctx)) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  cudaStream_t st = pb_stream_of(stream);
  // fused cluster kernel (one launch, DSMEM limb exchange) when the decode is
  // light; with many useful slots per ciphertext the separate decode kernel's
  // parallelism wins (B200, graph-timed: U = 256 x 32 cts 12.3 vs 13.9 us,
  // U = 512 x 16 cts 12.2 vs 10.7 us, U = 2041 x 50 cts 27.5 vs 19.2 us)
  if (U < 384 && ctx->dev.logN == 13 && ctx->dev.L >= 2) {
    const int rc = launch_decrypt_share_cluster<13>(ctx->dev, sk, ct, nP, out_pos, out_dst, U, share_out, st);
    if (rc != 0) return pb_set_error(PB_ERR_CUDA, cudaGetErrorString((cudaError_t)rc));
    PB_CHECK_LAUNCH();
    return PB_OK;
  }
  PB_DISPATCH_LOGN(ctx->dev.logN, launch_decrypt_inv, ctx->dev, sk, ct, nP, 1, out_pos, U, scratch, st);
  PB_CHECK_LAUNCH();
  k_decode_gather<<<pb_grid_1d(nP * U, 128), 128, 0, st>>>(ctx->dev, scratch, nP, U, out_pos, out_dst, share_out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_ctpt_mac_mask(const pb_ctx* ctx, const uint32_t* ct_in, const uint32_t* pt, const uint32_t* pt_shoup,
                                const int32_t* terms, int32_t K, int64_t nP, const int32_t* out_pos,
                                const int64_t* out_dst, int32_t U, const uint64_t* mask_vals, int filler,
                                uint64_t filler_seed, const uint64_t* seed_dev, uint32_t* ct_out, void* stream) {
  if (int s = need_big_n(ctx)) return s;
  if (!ct_in || !pt || !pt_shoup || !terms || !ct_out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (mask_vals && (!out_pos || !out_dst)) return pb_set_error(PB_ERR_ARG, "mask needs out_pos/out_dst");
  if (K < 1) return pb_set_error(PB_ERR_SHAPE, "K must be >= 1");
  if (nP <= 0) return PB_OK;
  if (nP > max_grid_polys(ctx)) return pb_set_error(PB_ERR_SHAPE, "too many polynomials in one call");
  PB_DISPATCH_LOGN(ctx->dev.logN, launch_mac, ctx->dev, ct_in, pt, pt_shoup, terms, K, nP, out_pos, out_dst, U,
                   mask_vals, filler, filler_seed, seed_dev, ct_out, pb_stream_of(stream));
  PB_CHECK_LAUNCH();
  return PB_OK;
}

// Shoup companions of NTT-domain rows: out[r][j] = floor(in[r][j] 2^32 / q_l),
// row r on limb r % L (the secret key's companion row for pb_encrypt_sk).
namespace {
__global__ void k_shoup_rows(PbDev P, const uint32_t* in, uint32_t* out, int64_t n_rows) {
  const int64_t total = n_rows * P.N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int l = (int)((e / P.N) % P.L);
    out[e] = shoup_of(in[e], P.q[l], P.inv_q32[l]);
  }
}
}  // namespace

extern "C" int pb_shoup_rows(const pb_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n_rows, void* stream) {
  if (!ctx || !in || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (n_rows <= 0) return PB_OK;
  k_shoup_rows<<<pb_grid_1d(n_rows * ctx->dev.N, 256), 256, 0, pb_stream_of(stream)>>>(ctx->dev, in, out, n_rows);
  PB_CHECK_LAUNCH();
  return PB_OK;
}
