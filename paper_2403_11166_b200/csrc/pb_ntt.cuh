// pb_ntt.cuh — register-blocked negacyclic NTT building blocks for sm_100a.
//
// Same transform as the reference ntt_forward / ntt_inverse (K:31-77):
// Cooley-Tukey with psi^bitrev twiddles, natural -> bit-reversed order, and
// the Gentleman-Sande inverse back to natural order.  The arithmetic is
// Harvey's lazy butterfly with Shoup twiddles over u32 residues (q < 2^30,
// values kept in [0,4q) forward / [0,2q) inverse, canonicalised once at the
// end), so results are bit-identical to K's fully reduced `%` version.
//
// Layout: one CTA of T = N/32 threads owns a row; every thread holds 32
// residues in registers.  The log2(N) stages are done in three register
// passes separated by two shared-memory exchanges:
//   P1  stages 0..4        (index bits N-1..N-5)   j = tid + T*c
//   P2  stages 5..logN-6   (middle bits)           j = lane | mid(c)<<5 | top(c,warp)
//   P3  stages logN-5..    (bits 4..0)             j = tid*32 + c
// Shared memory is padded (word j lives at j + j/32), which makes all three
// access patterns bank-conflict free with compile-time immediate offsets.
#pragma once

#include "pb_common.cuh"

// Min CTAs per SM for a row-per-CTA NTT kernel so that its register budget is
// 64 (32 residues + 16 twiddle pairs per thread fit; more registers cost
// occupancy -- measured slower on B200).
#define NTT_MINB(LOGN) ((1 << ((LOGN) - 5)) >= 1024 ? 1 : 1024 / (1 << ((LOGN) - 5)))

namespace pb {

__device__ __forceinline__ void ct_bfly(uint32_t& x, uint32_t& y, uint2 w, uint32_t q, uint32_t q2) {
  const uint32_t xx = min(x, x - q2);          // [0, 2q)
  const uint32_t tt = mul_shoup_lazy(y, w.x, w.y, q);  // [0, 2q)
  x = xx + tt;                                 // [0, 4q)
  y = xx - tt + q2;                            // (0, 4q)
}

__device__ __forceinline__ void gs_bfly(uint32_t& x, uint32_t& y, uint2 w, uint32_t q, uint32_t q2) {
  uint32_t s = x + y;                          // inputs in [0, 2q)
  s = min(s, s - q2);                          // [0, 2q)
  const uint32_t d = x - y + q2;               // (0, 4q)
  y = mul_shoup_lazy(d, w.x, w.y, q);          // [0, 2q)
  x = s;
}

template <int LOGN>
struct Ntt {
  static_assert(LOGN >= 11 && LOGN <= 15, "register NTT covers N = 2^11 .. 2^15");
  static constexpr int N = 1 << LOGN;
  static constexpr int T = N >> 5;
  static constexpr int M = LOGN - 10;
  // exchange area (padded row) + the staged twiddles of stages 0..LOGN-6
  // (tw[1 .. T-1], one uint2 per thread, shared by all threads of the row)
  static constexpr int TW_OFF = N + (N >> 5);
  static constexpr int SMEM_WORDS = TW_OFF + 2 * T;
  __device__ __forceinline__ static uint2* stw(uint32_t* sm) { return reinterpret_cast<uint2*>(sm + TW_OFF); }

  __device__ __forceinline__ static int pad(int j) { return j + (j >> 5); }

  // ---- index maps ----
  __device__ __forceinline__ static int fc2(int c) {  // compile-time part of the P2 index
    return ((c & ((1 << M) - 1)) << 5) | ((c >> M) << (LOGN - 5));
  }
  __device__ __forceinline__ static int j1(int tid, int c) { return tid + T * c; }
  __device__ __forceinline__ static int j2(int tid, int c) {
    return (tid & 31) + ((tid >> 5) << 10) + fc2(c);
  }
  __device__ __forceinline__ static int j3(int tid, int c) { return (tid << 5) + c; }

  // ---- shared memory exchanges (padded layout) ----
  __device__ __forceinline__ static void st1(uint32_t* sm, const uint32_t (&a)[32], int tid) {
    uint32_t* b = sm + pad(tid);
#pragma unroll
    for (int c = 0; c < 32; ++c) b[c * (T + T / 32)] = a[c];
  }
  __device__ __forceinline__ static void ld1(const uint32_t* sm, uint32_t (&a)[32], int tid) {
    const uint32_t* b = sm + pad(tid);
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = b[c * (T + T / 32)];
  }
  __device__ __forceinline__ static void st2(uint32_t* sm, const uint32_t (&a)[32], int tid) {
    uint32_t* b = sm + pad(j2(tid, 0));
#pragma unroll
    for (int c = 0; c < 32; ++c) b[pad(fc2(c))] = a[c];
  }
  __device__ __forceinline__ static void ld2(const uint32_t* sm, uint32_t (&a)[32], int tid) {
    const uint32_t* b = sm + pad(j2(tid, 0));
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = b[pad(fc2(c))];
  }
  __device__ __forceinline__ static void st3(uint32_t* sm, const uint32_t (&a)[32], int tid) {
    uint32_t* b = sm + tid * 33;
#pragma unroll
    for (int c = 0; c < 32; ++c) b[c] = a[c];
  }
  __device__ __forceinline__ static void ld3(const uint32_t* sm, uint32_t (&a)[32], int tid) {
    const uint32_t* b = sm + tid * 33;
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = b[c];
  }

  // ---- P3 twiddles: interleaved table, stage D at offset (2^D - 1)*T uint2,
  // entry [v][tid] = {w(2v), w(2v+1)} as one uint4, so every warp load is a
  // contiguous 512-byte line set (built by pb_ctx_create). ----
  template <int D>
  __device__ __forceinline__ static void tw3(const uint2* t3, int tid, uint2 (&w)[16]) {
    const uint2* base = t3 + ((1 << D) - 1) * T;
    if constexpr (D == 0) {
      w[0] = __ldg(base + tid);
    } else {
      const uint4* b4 = reinterpret_cast<const uint4*>(base);
#pragma unroll
      for (int v = 0; v < (1 << (D - 1)); ++v) {
        const uint4 x = __ldg(b4 + v * T + tid);
        w[2 * v] = make_uint2(x.x, x.y);
        w[2 * v + 1] = make_uint2(x.z, x.w);
      }
    }
  }

  // =========================== forward ===========================
  // bits: OR of the input's occupied indices.  Stage s butterflies index bit
  // logN-1-s; when that bit is 0 in every occupied position (earlier stages
  // only touch higher bits) the upper inputs are zero: (x, 0) -> (x, x).
  __device__ __forceinline__ static bool trivial(int bits, int s) { return !((bits >> (LOGN - 1 - s)) & 1); }
  __device__ __forceinline__ static void fwd_p1(uint32_t (&a)[32], const uint2* tw, uint32_t q, int bits = N - 1) {
    const uint32_t q2 = 2 * q;
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int tc = 16 >> s;
      if (trivial(bits, s)) {
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (!(c & tc)) a[c + tc] = a[c];
        continue;
      }
      uint2 w[16];
#pragma unroll
      for (int g = 0; g < (1 << s); ++g) w[g] = tw[(1 << s) + g];  // shared memory
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (!(c & tc)) ct_bfly(a[c], a[c + tc], w[c >> (5 - s)], q, q2);
    }
  }

  __device__ __forceinline__ static void fwd_p2(uint32_t (&a)[32], const uint2* tw, int tid, uint32_t q,
                                                int bits = N - 1) {
    const uint32_t q2 = 2 * q;
    const int warp = tid >> 5;
#pragma unroll
    for (int s = 5; s < 5 + M; ++s) {
      const int tc = 1 << (LOGN - 6 - s);
      if (trivial(bits, s)) {
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (!(c & tc)) a[c + tc] = a[c];
        continue;
      }
      const uint2* wb = tw + (1 << s) + (warp << (s + 10 - LOGN));
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (!(c & tc)) ct_bfly(a[c], a[c + tc], wb[fc2(c) >> (LOGN - s)], q, q2);
    }
  }
  template <int D>
  __device__ __forceinline__ static void fwd_p3_stage(uint32_t (&a)[32], const uint2* tw, int tid,
                                                      uint32_t q, uint32_t q2) {
    uint2 w[16];
    tw3<D>(tw, tid, w);
    const int tc = 16 >> D;
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (!(c & tc)) ct_bfly(a[c], a[c + tc], w[c >> (5 - D)], q, q2);
  }
  __device__ __forceinline__ static void fwd_p3(uint32_t (&a)[32], const uint2* tw, int tid, uint32_t q) {
    const uint32_t q2 = 2 * q;
    fwd_p3_stage<0>(a, tw, tid, q, q2);
    fwd_p3_stage<1>(a, tw, tid, q, q2);
    fwd_p3_stage<2>(a, tw, tid, q, q2);
    fwd_p3_stage<3>(a, tw, tid, q, q2);
    fwd_p3_stage<4>(a, tw, tid, q, q2);
  }

  // Full forward transform: a[] holds the row in P1 layout on entry and the
  // lazily reduced ([0,4q)) result in P3 layout on exit.  `sm` needs
  // SMEM_WORDS words; the caller syncs before reusing it.
  __device__ __forceinline__ static void forward(uint32_t (&a)[32], uint32_t* sm, const uint2* tw,
                                                 const uint2* t3, int tid, uint32_t q, int bits = N - 1) {
    // P1/P2 twiddles from shared memory: one coalesced load per thread instead of
    // just-in-time L1/L2 loads before every early stage (ncu: ~50% of the stall
    // samples sat in the P1 stages)
    uint2* st = stw(sm);
    st[tid] = __ldg(tw + tid);
    __syncthreads();
    fwd_p1(a, st, q, bits);
    st1(sm, a, tid);
    __syncthreads();
    ld2(sm, a, tid);
    fwd_p2(a, st, tid, q, bits);
    __syncthreads();
    st2(sm, a, tid);
    __syncthreads();
    ld3(sm, a, tid);
    fwd_p3(a, t3, tid, q);
  }

  // =========================== inverse ===========================
  template <int D>
  __device__ __forceinline__ static void inv_p3_stage(uint32_t (&a)[32], const uint2* tw, int tid,
                                                      uint32_t q, uint32_t q2) {
    uint2 w[16];
    tw3<D>(tw, tid, w);
    const int tc = 16 >> D;
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (!(c & tc)) gs_bfly(a[c], a[c + tc], w[c >> (5 - D)], q, q2);
  }
  __device__ __forceinline__ static void inv_p3(uint32_t (&a)[32], const uint2* tw, int tid, uint32_t q) {
    const uint32_t q2 = 2 * q;
    inv_p3_stage<4>(a, tw, tid, q, q2);
    inv_p3_stage<3>(a, tw, tid, q, q2);
    inv_p3_stage<2>(a, tw, tid, q, q2);
    inv_p3_stage<1>(a, tw, tid, q, q2);
    inv_p3_stage<0>(a, tw, tid, q, q2);
  }
  __device__ __forceinline__ static void inv_p2(uint32_t (&a)[32], const uint2* tw, int tid, uint32_t q) {
    const uint32_t q2 = 2 * q;
    const int warp = tid >> 5;
#pragma unroll
    for (int ss = 0; ss < M; ++ss) {
      const int s = 4 + M - ss;
      const int tc = 1 << (LOGN - 6 - s);
      const uint2* wb = tw + (1 << s) + (warp << (s + 10 - LOGN));
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (!(c & tc)) gs_bfly(a[c], a[c + tc], wb[fc2(c) >> (LOGN - s)], q, q2);
    }
  }
  __device__ __forceinline__ static void inv_p1(uint32_t (&a)[32], const uint2* tw, uint32_t q) {
    const uint32_t q2 = 2 * q;
#pragma unroll
    for (int ss = 0; ss < 5; ++ss) {
      const int s = 4 - ss;
      const int tc = 16 >> s;
      uint2 w[16];
#pragma unroll
      for (int g = 0; g < (1 << s); ++g) w[g] = tw[(1 << s) + g];  // shared memory
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (!(c & tc)) gs_bfly(a[c], a[c + tc], w[c >> (5 - s)], q, q2);
    }
  }

  // Full inverse (without the N^-1 scaling): a[] in P3 layout with values in
  // [0, 2q) on entry, P1 layout with values in [0, 2q) on exit.
  __device__ __forceinline__ static void inverse(uint32_t (&a)[32], uint32_t* sm, const uint2* tw,
                                                 const uint2* t3, int tid, uint32_t q) {
    uint2* st = stw(sm);
    st[tid] = __ldg(tw + tid);  // consumed after the next barrier (P2/P1)
    inv_p3(a, t3, tid, q);
    st3(sm, a, tid);
    __syncthreads();
    ld2(sm, a, tid);
    inv_p2(a, st, tid, q);
    __syncthreads();
    st2(sm, a, tid);
    __syncthreads();
    ld1(sm, a, tid);
    inv_p1(a, st, q);
  }

  // Inverse with the N^-1 scaling folded into the last (stage-0) GS butterfly:
  // x' = (x + y) N^-1, y' = (x - y) (w N^-1) -- 16 Shoup products per thread
  // instead of the 32 of a separate scaling pass.  Canonical [0, q) output in
  // P1 layout.  (wn, wns) = psi^-brv(1) N^-1 and its Shoup quotient.
  __device__ __forceinline__ static void inverse_scaled(uint32_t (&a)[32], uint32_t* sm, const uint2* tw,
                                                        const uint2* t3, int tid, uint32_t q, uint32_t ni,
                                                        uint32_t nis, uint32_t wn, uint32_t wns) {
    uint2* st = stw(sm);
    st[tid] = __ldg(tw + tid);
    inv_p3(a, t3, tid, q);
    st3(sm, a, tid);
    __syncthreads();
    ld2(sm, a, tid);
    inv_p2(a, st, tid, q);
    __syncthreads();
    st2(sm, a, tid);
    __syncthreads();
    ld1(sm, a, tid);
    const uint32_t q2 = 2 * q;
#pragma unroll
    for (int ss = 0; ss < 4; ++ss) {  // stages 4..1 as in inv_p1
      const int s = 4 - ss;
      const int tc = 16 >> s;
      uint2 w[16];
#pragma unroll
      for (int g = 0; g < (1 << s); ++g) w[g] = st[(1 << s) + g];
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (!(c & tc)) gs_bfly(a[c], a[c + tc], w[c >> (5 - s)], q, q2);
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) {  // stage 0 with the scaling folded in
      const uint32_t x = a[c], y = a[c + 16];  // [0, 2q)
      a[c] = mul_shoup(x + y, ni, nis, q);
      a[c + 16] = mul_shoup(x - y + q2, wn, wns, q);
    }
  }

  // ---- Output-pruned inverse.  The GS inverse decides output-index bit b in
  // its stage of distance 2^b (the difference branch makes bit b = 1).  When
  // only outputs n = 2^TT - 1 (mod 2^TT) are needed (the matmul packings'
  // useful slots), the first TT stages keep only the difference branch and
  // everything after runs on the N / 2^TT surviving values: the P3 stages on
  // the surviving registers, the remaining log N - 5 stages on a compact
  // shared-memory array A[m] = x[m 2^TT + 2^TT - 1] (same twiddles, same N^-1
  // folded into the last stage).  Result: canonical A[0 .. N >> TT) in sm. ----
  template <int TT, int D>
  __device__ __forceinline__ static void inv_p3_stage_pruned(uint32_t (&a)[32], const uint2* tw, int tid,
                                                             uint32_t q, uint32_t q2) {
    constexpr int b = 4 - D, tc = 1 << b;  // this stage butterflies index bit b
    uint2 w[16];
    tw3<D>(tw, tid, w);
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      if (c & tc) continue;
      if (b < TT) {  // keep the difference branch (upper register) of the surviving pairs
        if ((c & (tc - 1)) == tc - 1) a[c + tc] = mul_shoup_lazy(a[c] - a[c + tc] + q2, w[c >> (5 - D)].x,
                                                                 w[c >> (5 - D)].y, q);
      } else if ((c & ((1 << TT) - 1)) == (1 << TT) - 1) {
        gs_bfly(a[c], a[c + tc], w[c >> (5 - D)], q, q2);
      }
    }
  }
  template <int TT>
  __device__ __forceinline__ static void inverse_pruned(uint32_t (&a)[32], uint32_t* sm, const uint2* tw,
                                                        const uint2* t3, int tid, uint32_t q, uint32_t ni,
                                                        uint32_t nis, uint32_t wn, uint32_t wns) {
    static_assert(TT >= 1 && TT <= 5, "prune 1..5 stages");
    const uint32_t q2 = 2 * q;
    uint2* st = stw(sm);
    st[tid] = __ldg(tw + tid);  // stage twiddles tw[1 .. T) (the compact stages use indices < T)
    inv_p3_stage_pruned<TT, 4>(a, t3, tid, q, q2);
    inv_p3_stage_pruned<TT, 3>(a, t3, tid, q, q2);
    inv_p3_stage_pruned<TT, 2>(a, t3, tid, q, q2);
    inv_p3_stage_pruned<TT, 1>(a, t3, tid, q, q2);
    inv_p3_stage_pruned<TT, 0>(a, t3, tid, q, q2);
    constexpr int R = (1 << TT) - 1, NP = N >> TT;
#pragma unroll
    for (int c = R; c < 32; c += 1 << TT) sm[tid * (32 >> TT) + (c >> TT)] = a[c];  // compact index n >> TT
    __syncthreads();
#pragma unroll 1
    for (int bb = 5; bb < LOGN; ++bb) {  // remaining stages: index bits 5 .. logN-1
      const int d = 1 << (bb - TT);       // compact pair distance
      const int h = N >> (bb + 1);        // twiddle groups of this stage
      for (int k = tid; k < NP / 2; k += T) {
        const int m = ((k >> (bb - TT)) << (bb - TT + 1)) | (k & (d - 1));
        uint32_t x = sm[m], y = sm[m + d];
        if (bb < LOGN - 1) {
          gs_bfly(x, y, st[h + (m >> (bb + 1 - TT))], q, q2);
          sm[m] = x;
          sm[m + d] = y;
        } else {  // last stage with N^-1 folded in (as inverse_scaled)
          sm[m] = mul_shoup(x + y, ni, nis, q);
          sm[m + d] = mul_shoup(x - y + q2, wn, wns, q);
        }
      }
      __syncthreads();
    }
  }

  // ---- NTT-domain rows in DEVICE ORDER: bit-reversed index j = tid*32 + 4v + k
  // (the P3 layout) is stored at address v*4T + tid*4 + k, so a P3-layout
  // register file moves to/from HBM with fully coalesced 128-bit accesses.
  // (pb_ntt_reorder converts to/from the reference's bit-reversed order.) ----
  __device__ __forceinline__ static int dev_addr(int j) { return ((j & 31) >> 2) * 4 * T + (j >> 5) * 4 + (j & 3); }
  __device__ __forceinline__ static void gld3(const uint32_t* row, uint32_t (&a)[32], int tid) {
    const uint4* p = reinterpret_cast<const uint4*>(row) + tid;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const uint4 x = __ldg(p + v * T);
      a[4 * v] = x.x; a[4 * v + 1] = x.y; a[4 * v + 2] = x.z; a[4 * v + 3] = x.w;
    }
  }
  __device__ __forceinline__ static void gst3(uint32_t* row, const uint32_t (&a)[32], int tid) {
    uint4* p = reinterpret_cast<uint4*>(row) + tid;
#pragma unroll
    for (int v = 0; v < 8; ++v) p[v * T] = make_uint4(a[4 * v], a[4 * v + 1], a[4 * v + 2], a[4 * v + 3]);
  }
  __device__ __forceinline__ static void gld1(const uint32_t* row, uint32_t (&a)[32], int tid) {
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = __ldg(row + tid + T * c);
  }
  __device__ __forceinline__ static void gst1(uint32_t* row, const uint32_t (&a)[32], int tid) {
#pragma unroll
    for (int c = 0; c < 32; ++c) row[tid + T * c] = a[c];
  }
};

__device__ __forceinline__ uint32_t canon4(uint32_t x, uint32_t q) {  // [0,4q) -> [0,q)
  x = min(x, x - 2 * q);
  return min(x, x - q);
}

}  // namespace pb

// Dispatch a templated launcher over LOGN in [11, 15].
#define PB_DISPATCH_LOGN(logn, FN, ...)             \
  do {                                              \
    switch (logn) {                                 \
      case 11: FN<11>(__VA_ARGS__); break;          \
      case 12: FN<12>(__VA_ARGS__); break;          \
      case 13: FN<13>(__VA_ARGS__); break;          \
      case 14: FN<14>(__VA_ARGS__); break;          \
      case 15: FN<15>(__VA_ARGS__); break;          \
      default: break;                               \
    }                                               \
  } while (0)
