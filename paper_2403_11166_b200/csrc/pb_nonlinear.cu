// pb_nonlinear.cu — the OT-based non-linear protocols of SPEC:491-581 /
// PAPER:1248-1268 (CrypTFlow2-style) on the B200, with SPEC:479's dealer OT
// backend ("local correlated-randomness generator ... fast, insecure") as the
// oblivious-transfer functionality: the receiver obtains message[choice].
// Both parties run in this process, so every round of a protocol instance is
// evaluated by one thread per element -- each party's messages computed only
// from that party's inputs and randomness, the opened values from both
// parties' messages -- and the communication is counted by the caller's census.
//
//   secure comparison  1{a < b}, a at P0 (the MO), b at P1 (the DO): 4-bit
//                      blocks, per block one 1-of-16 OT of P0's (lt, eq) table
//                      masked with P0's random bits, the blocks combined in a
//                      tree lt = lt_hi ^ (eq_hi & lt_lo), eq = eq_hi & eq_lo
//                      with Beaver bit triples from the dealer (XOR shares)
//   DReLU              1{x >= 0} = 1 ^ MSB(x0) ^ MSB(x1) ^ carry, carry =
//                      1{2^(l-1) - 1 - x0' < x1'} over l-1 bits
//   MUX / bit inject   d * x from XOR-shared d with two 1-of-2 OTs (CrypTFlow2
//                      Alg. 6): z0 = r0 - r1 + d x1, z1 = r1 - r0 + d x0
//   faithful trunc     arith_shift(x, k) = ((x0' >> k) + (x1 >> k) + c
//                      - w 2^(l-k)) - 2^(l-1-k), x0' = x0 + 2^(l-1): wrap w and
//                      low carry c by two comparisons, B2A by the MUX
//
// Every random word comes from the numpy-identical Philox4x64 stream
// (seed, stream_id) at raw index elem * WORDS + k, so oracle/nonlinear.py
// restates each protocol bit for bit.
#include "pb_common.cuh"

namespace {

// An element's W random words: raw draws base .. base+W-1 of the numpy
// Philox4x64 stream, from the 4-word counter blocks covering them (each
// computed once, not once per word as philox_np_raw would), placed by the
// element's phase base mod 4 with selects -- compile-time indices only, so
// the words stay in registers.
template <int W>
struct Rng {
  uint64_t v[W];
  __device__ __forceinline__ uint64_t w(int k) const { return v[k]; }
  __device__ __forceinline__ void fill(uint64_t seed, uint64_t stream, uint64_t base) {
    constexpr int NB = (W + 3) / 4 + 1;
    const uint64_t b0 = base >> 2;
    const int ph = (int)(base & 3);
    const int nb = (ph + W + 3) >> 2;  // blocks this element needs (NB - 1 or NB)
    uint64_t t[4 * NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (b < nb) {
        const u64x4 o = philox4x64_10(b0 + b + 1, 0, 0, 0, seed, stream);  // numpy pre-increments the counter
#pragma unroll
        for (int j = 0; j < 4; ++j) t[4 * b + j] = o.v[j];
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) t[4 * b + j] = 0ull;
      }
    }
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = ph == 0 ? t[k] : ph == 1 ? t[k + 1] : ph == 2 ? t[k + 2] : t[k + 3];
  }
};

// Beaver AND of XOR-shared bits with triple (u0, u1, v0, v1, w0): the parties
// open d = x ^ u and e = y ^ v.
__device__ __forceinline__ void and_gate(uint32_t x0, uint32_t x1, uint32_t y0, uint32_t y1, uint32_t t,
                                         uint32_t& z0, uint32_t& z1) {
  const uint32_t u0 = t & 1, u1 = (t >> 1) & 1, v0 = (t >> 2) & 1, v1 = (t >> 3) & 1, w0 = (t >> 4) & 1;
  const uint32_t w1 = ((u0 ^ u1) & (v0 ^ v1)) ^ w0;  // the dealer's second triple share
  const uint32_t d = (x0 ^ u0) ^ (x1 ^ u1), e = (y0 ^ v0) ^ (y1 ^ v1);  // opened
  z0 = w0 ^ (d & v0) ^ (e & u0) ^ (d & e);
  z1 = w1 ^ (d & v1) ^ (e & u1);
}

// 5 triple bits number t from the little-endian bit string of words tw[0..3]
__device__ __forceinline__ uint32_t triple_bits(const uint64_t (&tw)[4], int t) {
  const int bit = 5 * t, i = bit >> 6, o = bit & 63;
  uint64_t v = tw[i] >> o;
  if (o > 59) v |= tw[i + 1] << (64 - o);
  return (uint32_t)(v & 31u);
}

// The comparison tree for a compile-time leaf count: every node's shares in
// its own registers, every triple's bit offset a constant (the runtime-q
// version below spends most of its ALU work on variable shifts and loop
// control; k_nl is ALU-bound).  Level CNT -> (CNT + 1) / 2, pairs (2i, 2i+1)
// combined in place into node i with triples T + 2i, T + 2i + 1.
template <int CNT, int T>
struct CmpTree {
  __device__ __forceinline__ static void run(uint32_t (&L0)[16], uint32_t (&L1)[16], uint32_t (&E0)[16],
                                             uint32_t (&E1)[16], const uint64_t (&tw)[4]) {
#pragma unroll
    for (int i = 0; i < CNT / 2; ++i) {
      uint32_t a0, a1, b0, b1;
      and_gate(E0[2 * i + 1], E1[2 * i + 1], L0[2 * i], L1[2 * i], triple_bits(tw, T + 2 * i), a0, a1);
      and_gate(E0[2 * i + 1], E1[2 * i + 1], E0[2 * i], E1[2 * i], triple_bits(tw, T + 2 * i + 1), b0, b1);
      L0[i] = L0[2 * i + 1] ^ a0;
      L1[i] = L1[2 * i + 1] ^ a1;
      E0[i] = b0;
      E1[i] = b1;
    }
    if constexpr (CNT & 1) {
      L0[CNT / 2] = L0[CNT - 1];
      L1[CNT / 2] = L1[CNT - 1];
      E0[CNT / 2] = E0[CNT - 1];
      E1[CNT / 2] = E1[CNT - 1];
    }
    CmpTree<(CNT + 1) / 2, T + 2 * (CNT / 2)>::run(L0, L1, E0, E1, tw);
  }
};
template <int T>
struct CmpTree<1, T> {
  __device__ __forceinline__ static void run(uint32_t (&)[16], uint32_t (&)[16], uint32_t (&)[16], uint32_t (&)[16],
                                             const uint64_t (&)[4]) {}
};

template <int Q>
__device__ __forceinline__ void cmp_lt_q(uint64_t a, uint64_t b, uint32_t lt0m, uint32_t eq0m,
                                         const uint64_t (&tw)[4], uint32_t& c0, uint32_t& c1) {
  uint32_t L0[16], L1[16], E0[16], E1[16];
#pragma unroll
  for (int j = 0; j < Q; ++j) {  // leaf OTs: P1 (choice b_j) learns P0's table entry
    const uint32_t aj = (uint32_t)(a >> (4 * j)) & 15u, bj = (uint32_t)(b >> (4 * j)) & 15u;
    L0[j] = (lt0m >> j) & 1u;
    E0[j] = (eq0m >> j) & 1u;
    L1[j] = L0[j] ^ (uint32_t)(aj < bj);
    E1[j] = E0[j] ^ (uint32_t)(aj == bj);
  }
  CmpTree<Q, 0>::run(L0, L1, E0, E1, tw);
  c0 = L0[0];
  c1 = L1[0];
}

// XOR shares (c0 at P0, c1 at P1) of 1{a < b} over nbits <= 64 bits.
// lt0 / eq0: P0's random leaf masks (bit j = block j); tw: triple words.
// Every leaf count is a compile-time instance (pb_nl_op: nbits <= 61).
__device__ __forceinline__ void cmp_lt(uint64_t a, uint64_t b, int nbits, uint32_t lt0m, uint32_t eq0m,
                                       const uint64_t (&tw)[4], uint32_t& c0, uint32_t& c1) {
#define PB_CMPQ(Q) \
  case Q: cmp_lt_q<Q>(a, b, lt0m, eq0m, tw, c0, c1); return;
  switch ((nbits + 3) >> 2) {
    PB_CMPQ(1) PB_CMPQ(2) PB_CMPQ(3) PB_CMPQ(4) PB_CMPQ(5) PB_CMPQ(6) PB_CMPQ(7) PB_CMPQ(8)
    PB_CMPQ(9) PB_CMPQ(10) PB_CMPQ(11) PB_CMPQ(12) PB_CMPQ(13) PB_CMPQ(14) PB_CMPQ(15) PB_CMPQ(16)
    default: c0 = c1 = 0u; return;
  }
#undef PB_CMPQ
}

__device__ __forceinline__ uint64_t lmask(int ell) { return ell >= 64 ? ~0ull : ((1ull << ell) - 1); }

// DReLU (4 words: leaf masks, 3 triple words): XOR shares of 1{x >= 0}.
template <class R>
__device__ __forceinline__ void drelu(uint64_t x0, uint64_t x1, int ell, const R& r, int off, uint32_t& d0,
                                      uint32_t& d1) {
  const int h = ell - 1;
  const uint64_t hm = (1ull << h) - 1;
  const uint64_t lw = r.w(off);
  const uint64_t tw[4] = {r.w(off + 1), r.w(off + 2), r.w(off + 3), 0ull};
  uint32_t c0, c1;
  cmp_lt(hm - (x0 & hm), x1 & hm, h, (uint32_t)(lw & 0xFFFFu), (uint32_t)((lw >> 16) & 0xFFFFu), tw, c0, c1);
  d0 = 1u ^ (uint32_t)((x0 >> h) & 1u) ^ c0;
  d1 = (uint32_t)((x1 >> h) & 1u) ^ c1;
}

// MUX (2 words: r0, r1): arithmetic shares of d * x from XOR-shared d.
template <class R>
__device__ __forceinline__ void mux(uint32_t d0, uint32_t d1, uint64_t x0, uint64_t x1, uint64_t m, const R& r,
                                    int off, uint64_t& z0, uint64_t& z1) {
  const uint64_t r0 = r.w(off) & m, r1 = r.w(off + 1) & m;
  const uint64_t m00 = (uint64_t)(0 - r0) + (d0 ? x0 : 0ull), m01 = (uint64_t)(0 - r0) + (d0 ? 0ull : x0);  // P0 sends
  const uint64_t m10 = (uint64_t)(0 - r1) + (d1 ? x1 : 0ull), m11 = (uint64_t)(0 - r1) + (d1 ? 0ull : x1);  // P1 sends
  const uint64_t y1 = d1 ? m01 : m00, y0 = d0 ? m11 : m10;  // 1-of-2 OTs: P1 chooses with d1, P0 with d0
  z0 = (r0 + y0) & m;
  z1 = (r1 + y1) & m;
}

// Faithful arithmetic shift by k (9 words: leaves, 3 + 1 triple words, 2 x 2 MUX words).
template <class R>
__device__ __forceinline__ void trunc(uint64_t x0, uint64_t x1, int ell, int k, const R& r, int off, uint64_t& y0,
                                      uint64_t& y1) {
  const uint64_t m = lmask(ell), km = (1ull << k) - 1;
  const uint64_t xb = (x0 + (1ull << (ell - 1))) & m;  // P0's biased share: signed -> unsigned order
  const uint64_t lw = r.w(off);
  const uint64_t tw1[4] = {r.w(off + 1), r.w(off + 2), r.w(off + 3), 0ull};
  const uint64_t tw2[4] = {r.w(off + 4), 0ull, 0ull, 0ull};
  uint32_t w0, w1, c0, c1;
  cmp_lt(m - xb, x1, ell, (uint32_t)(lw & 0xFFFFu), (uint32_t)((lw >> 16) & 0xFFFFu), tw1, w0, w1);  // wrap
  cmp_lt(km - (xb & km), x1 & km, k, (uint32_t)((lw >> 32) & 0xFFFFu), (uint32_t)((lw >> 48) & 0xFFFFu), tw2, c0,
         c1);  // low carry
  uint64_t C0, C1, W0, W1;
  mux(c0, c1, 1ull, 0ull, m, r, off + 5, C0, C1);                // B2A(c)
  mux(w0, w1, 1ull << (ell - k), 0ull, m, r, off + 7, W0, W1);   // B2A(w) * 2^(l-k)
  y0 = ((xb >> k) + C0 - W0 - (1ull << (ell - 1 - k))) & m;
  y1 = ((x1 >> k) + C1 - W1) & m;
}

constexpr int W_DRELU = 4, W_MUX = 2, W_TRUNC = 9;

// op: 0 DReLU (d out), 1 MUX (d in), 2 TRUNC, 3 RELU + TRUNC (d out), 4 TRUNC + MUX (d in)
template <int OP>
struct NlWords;
template <> struct NlWords<0> { static constexpr int W = W_DRELU; };
template <> struct NlWords<1> { static constexpr int W = W_MUX; };
template <> struct NlWords<2> { static constexpr int W = W_TRUNC; };
template <> struct NlWords<3> { static constexpr int W = W_DRELU + W_MUX + W_TRUNC; };
template <> struct NlWords<4> { static constexpr int W = W_TRUNC + W_MUX; };

template <int OP>
__global__ void __launch_bounds__(256) k_nl(const uint64_t* __restrict__ x0, const uint64_t* __restrict__ x1,
                                            int64_t n, int ell, int k, const uint8_t* __restrict__ d_in,
                                            uint8_t* __restrict__ d_out, uint64_t seed_arg, const uint64_t* seed_dev,
                                            uint64_t stream_id, uint64_t raw_offset,
                                            uint64_t* __restrict__ y0, uint64_t* __restrict__ y1) {
  constexpr int W = NlWords<OP>::W;
  const uint64_t seed = np_seed(seed_arg, seed_dev);
  const uint64_t m = lmask(ell);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Rng<W> r;
    r.fill(seed, stream_id, raw_offset + (uint64_t)i * W);
    const uint64_t a = x0[i] & m, b = x1[i] & m;
    uint32_t d0 = 0, d1 = 0;
    uint64_t z0 = a, z1 = b;
    if constexpr (OP == 1 || OP == 4) {
      d0 = d_in[i] & 1u;
      d1 = (d_in[i] >> 1) & 1u;
    }
    if constexpr (OP == 0) {
      drelu(a, b, ell, r, 0, d0, d1);
    } else if constexpr (OP == 1) {
      mux(d0, d1, a, b, m, r, 0, z0, z1);
    } else if constexpr (OP == 2) {
      trunc(a, b, ell, k, r, 0, z0, z1);
    } else if constexpr (OP == 3) {
      drelu(a, b, ell, r, 0, d0, d1);
      uint64_t u0, u1;
      mux(d0, d1, a, b, m, r, W_DRELU, u0, u1);
      trunc(u0, u1, ell, k, r, W_DRELU + W_MUX, z0, z1);
    } else {
      uint64_t u0, u1;
      trunc(a, b, ell, k, r, 0, u0, u1);
      mux(d0, d1, u0, u1, m, r, W_TRUNC, z0, z1);
    }
    if constexpr (OP == 0 || OP == 3) d_out[i] = (uint8_t)(d0 | (d1 << 1));
    if constexpr (OP != 0) {
      y0[i] = z0;
      y1[i] = z1;
    }
  }
}

}  // namespace

// Random words per element of each op (the caller reserves n * words raw draws).
extern "C" int pb_nl_words(int op) {
  switch (op) {
    case PB_NL_DRELU: return W_DRELU;
    case PB_NL_MUX: return W_MUX;
    case PB_NL_TRUNC: return W_TRUNC;
    case PB_NL_RELU_TRUNC: return W_DRELU + W_MUX + W_TRUNC;
    case PB_NL_TRUNC_MUX: return W_TRUNC + W_MUX;
    default: return -1;
  }
}

extern "C" int pb_nl_op(int op, const uint64_t* x0, const uint64_t* x1, int64_t n, int32_t ell, int32_t k,
                        const uint8_t* d_in, uint8_t* d_out, uint64_t seed, const uint64_t* seed_dev,
                        uint64_t stream_id, uint64_t raw_offset, uint64_t* y0, uint64_t* y1, void* stream) {
  const int words = pb_nl_words(op);
  if (words < 0) return pb_set_error(PB_ERR_ARG, "bad non-linear op");
  if (ell < 4 || ell > 62) return pb_set_error(PB_ERR_ARG, "ell must be in [4, 62]");
  const bool tr = op == PB_NL_TRUNC || op == PB_NL_RELU_TRUNC || op == PB_NL_TRUNC_MUX;
  // the low-carry comparison's 2 (ceil(k/4) - 1) triples live in one 64-bit word
  if (tr && (k < 1 || k >= ell - 1 || k > 28)) return pb_set_error(PB_ERR_ARG, "truncation bits must be in [1, 28]");
  if (n <= 0) return PB_OK;
  if (!x0 || !x1) return pb_set_error(PB_ERR_ARG, "null argument");
  if ((op == PB_NL_MUX || op == PB_NL_TRUNC_MUX) && !d_in) return pb_set_error(PB_ERR_ARG, "MUX needs d shares");
  if ((op == PB_NL_DRELU || op == PB_NL_RELU_TRUNC) && !d_out) return pb_set_error(PB_ERR_ARG, "null d_out");
  if (op != PB_NL_DRELU && (!y0 || !y1)) return pb_set_error(PB_ERR_ARG, "null output");
  cudaStream_t st = pb_stream_of(stream);
#define PB_NL(OP) k_nl<OP><<<pb_grid_1d(n, 256), 256, 0, st>>>(x0, x1, n, ell, k, d_in, d_out, seed, seed_dev, \
                                                              stream_id, raw_offset, y0, y1)
  switch (op) {
    case 0: PB_NL(0); break;
    case 1: PB_NL(1); break;
    case 2: PB_NL(2); break;
    case 3: PB_NL(3); break;
    default: PB_NL(4); break;
  }
#undef PB_NL
  PB_CHECK_LAUNCH();
  return PB_OK;
}
