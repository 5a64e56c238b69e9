// pb_nttw.cuh — "wide" negacyclic NTT: V = 2^LOGV residues per thread and
// T = N/V threads per row (V = 8 or 16 vs the 32 of pb_ntt.cuh), for SMALL
// launches where the latency of one CTA, not throughput, bounds a kernel:
// a quarter of the per-thread work shortens the CTA's critical path at the
// cost of more shared-memory exchanges.
//
// Same transform, twiddle tables, lazy Harvey butterflies and canonical
// outputs as pb::Ntt (identical results bit-for-bit), and the same device
// order for NTT-domain rows, so kernels may mix the two freely.
//
// Pass p holds the index bits [lo_p, lo_p + LOGV), lo_p = max(0, LOGN - (p+1) LOGV):
// thread tid, slot c  ->  j = (tid & (2^lo - 1)) | c << lo | (tid >> lo) << (lo + LOGV)
// and runs the CT (forward, bits high -> low) / GS (inverse, low -> high)
// stages whose bit lies in the pass; stage s = LOGN-1-b on bit b uses the
// twiddle tw[2^s + (j >> (b+1))].  Shared memory is padded (j + j/32).
#pragma once

#include "pb_ntt.cuh"

namespace pb {

template <int LOGN, int LOGV>
struct NttW {
  static constexpr int N = 1 << LOGN;
  static constexpr int V = 1 << LOGV;
  static constexpr int T = N >> LOGV;
  static constexpr int P = (LOGN + LOGV - 1) / LOGV;
  static constexpr int SMEM_WORDS = N + (N >> 5);

  __device__ __forceinline__ static int pad(int j) { return j + (j >> 5); }
  __host__ __device__ static constexpr int lo_of(int p) {
    return LOGN - (p + 1) * LOGV > 0 ? LOGN - (p + 1) * LOGV : 0;
  }
  __device__ __forceinline__ static int jof(int lo, int tid, int c) {
    return (tid & ((1 << lo) - 1)) | (c << lo) | ((tid >> lo) << (lo + LOGV));
  }
  __device__ __forceinline__ static int j1(int tid, int c) { return tid + T * c; }  // pass-0 (natural) layout

  // stages on bits [bhi .. blo] (inclusive, descending) within held range lo
  template <int LO, int BHI, int BLO>
  __device__ __forceinline__ static void fwd_pass(uint32_t (&a)[V], const uint2* tw, int tid, uint32_t q) {
    const uint32_t q2 = 2 * q;
#pragma unroll
    for (int b = BHI; b >= BLO; --b) {
      const int s = LOGN - 1 - b;
      const int lb = b - LO;
      const int hi = (tid >> LO) << (LO + LOGV - b - 1);
#pragma unroll
      for (int c = 0; c < V; ++c)
        if (!(c & (1 << lb))) ct_bfly(a[c], a[c | (1 << lb)], __ldg(tw + (1 << s) + hi + (c >> (lb + 1))), q, q2);
    }
  }
  template <int LO, int BLO, int BHI>
  __device__ __forceinline__ static void inv_pass(uint32_t (&a)[V], const uint2* tw, int tid, uint32_t q) {
    const uint32_t q2 = 2 * q;
#pragma unroll
    for (int b = BLO; b <= BHI; ++b) {
      const int s = LOGN - 1 - b;
      const int lb = b - LO;
      const int hi = (tid >> LO) << (LO + LOGV - b - 1);
#pragma unroll
      for (int c = 0; c < V; ++c)
        if (!(c & (1 << lb))) gs_bfly(a[c], a[c | (1 << lb)], __ldg(tw + (1 << s) + hi + (c >> (lb + 1))), q, q2);
    }
  }
  __device__ __forceinline__ static void st(uint32_t* sm, const uint32_t (&a)[V], int lo, int tid) {
#pragma unroll
    for (int c = 0; c < V; ++c) sm[pad(jof(lo, tid, c))] = a[c];
  }
  __device__ __forceinline__ static void ld(const uint32_t* sm, uint32_t (&a)[V], int lo, int tid) {
#pragma unroll
    for (int c = 0; c < V; ++c) a[c] = sm[pad(jof(lo, tid, c))];
  }

  template <int p>
  __device__ __forceinline__ static void fwd_from(uint32_t (&a)[V], uint32_t* sm, const uint2* tw, int tid, uint32_t q) {
    if constexpr (p < P) {
      constexpr int LO = lo_of(p);
      constexpr int BHI = LOGN - 1 - p * LOGV;
      fwd_pass<LO, BHI, LO>(a, tw, tid, q);
      if constexpr (p + 1 < P) {
        st(sm, a, LO, tid);
        __syncthreads();
        ld(sm, a, lo_of(p + 1), tid);
        __syncthreads();
        fwd_from<p + 1>(a, sm, tw, tid, q);
      }
    }
  }
  // a[] in natural (pass-0) layout on entry; lazily reduced ([0,4q)) result in
  // the last pass's layout (j = c | tid << LOGV) on exit.  `sm` is free after.
  __device__ __forceinline__ static void forward(uint32_t (&a)[V], uint32_t* sm, const uint2* tw, int tid, uint32_t q) {
    fwd_from<0>(a, sm, tw, tid, q);
  }
  template <int p>
  __device__ __forceinline__ static void inv_from(uint32_t (&a)[V], uint32_t* sm, const uint2* tw, int tid, uint32_t q) {
    if constexpr (p >= 0) {
      constexpr int LO = lo_of(p);
      constexpr int BLO = (p == P - 1) ? 0 : LO;
      constexpr int BHI = LOGN - 1 - p * LOGV;
      inv_pass<LO, BLO, BHI>(a, tw, tid, q);
      if constexpr (p > 0) {
        st(sm, a, LO, tid);
        __syncthreads();
        ld(sm, a, lo_of(p - 1), tid);
        __syncthreads();
        inv_from<p - 1>(a, sm, tw, tid, q);
      }
    }
  }
  // a[] in the last pass's layout, values in [0,2q) on entry; natural layout,
  // [0,2q) on exit (no N^-1 scaling).
  __device__ __forceinline__ static void inverse(uint32_t (&a)[V], uint32_t* sm, const uint2* tw, int tid, uint32_t q) {
    inv_from<P - 1>(a, sm, tw, tid, q);
  }

  // ---- device order (pb_ntt.cuh): bit-reversed j = 32 t + 4 v + k at v*N/8 + 4 t + k.
  // The last-pass layout holds j = V*tid + c, c < V: uint4 groups of 4. ----
  __device__ __forceinline__ static int dev4(int tid, int g) {  // uint4 index of slots 4g..4g+3
    const int j = (tid << LOGV) + 4 * g;
    return ((j & 31) >> 2) * (N >> 5) + (j >> 5);
  }
  __device__ __forceinline__ static void gst_dev(uint32_t* row, const uint32_t (&a)[V], int tid) {
    uint4* p4 = reinterpret_cast<uint4*>(row);
#pragma unroll
    for (int g = 0; g < V / 4; ++g) p4[dev4(tid, g)] = make_uint4(a[4 * g], a[4 * g + 1], a[4 * g + 2], a[4 * g + 3]);
  }
  __device__ __forceinline__ static void gld_dev(const uint32_t* row, uint32_t (&a)[V], int tid) {
    const uint4* p4 = reinterpret_cast<const uint4*>(row);
#pragma unroll
    for (int g = 0; g < V / 4; ++g) {
      const uint4 x = __ldg(p4 + dev4(tid, g));
      a[4 * g] = x.x; a[4 * g + 1] = x.y; a[4 * g + 2] = x.z; a[4 * g + 3] = x.w;
    }
  }
  __device__ __forceinline__ static void gld1(const uint32_t* row, uint32_t (&a)[V], int tid) {
#pragma unroll
    for (int c = 0; c < V; ++c) a[c] = __ldg(row + tid + T * c);
  }
  __device__ __forceinline__ static void gst1(uint32_t* row, const uint32_t (&a)[V], int tid) {
#pragma unroll
    for (int c = 0; c < V; ++c) row[tid + T * c] = a[c];
  }
};

}  // namespace pb
