// pb_pack.cuh — packed plaintext sources (compact pi_v / pi_W maps) and
// Montgomery arithmetic shared by the MO-side kernels.
#pragma once

#include "pb_ntt.cuh"

namespace pbk {

// A plaintext source: `vals` is a flat Z_t tensor.  With `pos` set, poly p
// has coefficient pos[p][z] = vals[src[p][z]] for z < Z (pos < 0: unused
// slot) and zeros elsewhere -- the compact form of the packing maps pi_v /
// pi_W.  With pos == NULL, vals is a dense [P][N] array.
struct Pack {
  const uint64_t* vals;
  const int32_t* pos;
  const int32_t* src;
  int Z;
};

// Loads the lifted source polynomial p into a[] in the NTT's P1 layout; the
// packed path builds the row in shared memory and leaves `sm` free.  Returns
// the OR of the occupied coefficient indices (N - 1 when dense): a forward NTT
// stage whose index bit is 0 in every occupied position has structurally zero
// upper inputs and is skipped (Ntt::forward).
template <class Nt, class Lift>
__device__ __forceinline__ int load_source(uint32_t (&a)[32], uint32_t* sm, const Pack& s, int64_t p, int tid,
                                           Lift lift) {
  if (s.pos) {
    int* sup = reinterpret_cast<int*>(sm + Nt::TW_OFF);  // free until the NTT stages its twiddles
    if (tid == 0) *sup = 0;
    for (int j = tid; j < Nt::N; j += Nt::T) sm[Nt::pad(j)] = 0u;
    __syncthreads();
    int jor = 0;
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
        if (j[u] >= 0) sm[Nt::pad(j[u])] = lift(v[u]), jor |= j[u];
    }
    if (jor) atomicOr(sup, jor);
    __syncthreads();
    const int bits = *sup;
    Nt::ld1(sm, a, tid);
    __syncthreads();
    return bits;
  }
  const uint64_t* v = s.vals + p * Nt::N;
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = lift(__ldg(v + Nt::j1(tid, c)));
  return Nt::N - 1;
}

// Montgomery multiplication with R = 2^32: returns a*b*R^-1 mod q in [0, 2q)
// for a, b < q.  qn = -q^-1 mod 2^32.  Plaintext multipliers are stored in
// Montgomery form (pt*R mod q) so mont(ct, ptR) = ct*pt mod q and no Shoup
// companion row has to be streamed.
__device__ __forceinline__ uint32_t mont_lazy(uint32_t a, uint32_t b, uint32_t q, uint32_t qn) {
  const uint64_t t = (uint64_t)a * b;
  const uint32_t m = (uint32_t)t * qn;
  return (uint32_t)((t + (uint64_t)m * q) >> 32);
}

}  // namespace pbk
