// pb_tc.cu — the Z_{2^64} ring GEMMs of the conv / FC local terms
// (K:206-218 matmul_wrap, K:260-278 conv2d_wrap and the protocols' im2col
// lowerings) on the int8 TENSOR CORES, hand-written for sm_100a:
// tcgen05.mma kind::i8 with TMA-staged operands and TMEM accumulators.
//
// A u64 operand < 2^59 is written in balanced base-256 digits
// a = sum_{i<8} a_i 256^i, a_i in [-128, 127], so
//   a * b mod 2^64 = sum_{s<8} 256^s C_s,   C_s = sum_{i+j=s} a_i b_j
// (digit pairs with i + j >= 8 vanish mod 2^64): 36 int8 x int8 -> int32
// products per K step.  One CTA owns a 128 x 64 output tile and keeps ALL
// EIGHT C_s accumulators in tensor memory at once (8 x 64 columns = the
// whole 512-column TMEM), so the shift-and-add combine runs in the epilogue
// straight out of TMEM (tcgen05.ld) -- no int32 partial products in HBM.
// Exactness: |C_s| <= (s+1) K_cta 2^14 with balanced digits; C_0..C_3 must be
// exact (they are shifted by < 32 bits) which holds for K_cta <= 16384
// (|C_3| <= 2^30); C_4..C_7 are only needed mod 2^(64-8s) <= 2^32, so int32
// wrap-around is harmless.  Longer contractions are split over CTAs
// (gridDim.z) and summed with u64 atomics (exact mod 2^64).
//
// Pipeline per CTA (128 threads, one CTA per SM: 192 KB of shared memory):
//   warp 0 lane 0  TMA producer: per 64-byte K block one 3-D tensor copy of
//                  the 8 digit planes of the 128-row P tile and one of the
//                  64-row Q tile (SWIZZLE_64B), 2-stage full/empty mbarriers
//   warp 1 lane 0  MMA issuer: 2 x 36 tcgen05.mma (M=128, N=64, K=32) per
//                  block, tcgen05.commit releases the stage
//   warps 0-3      epilogue: tcgen05.ld 32x32b of the 8 accumulators,
//                  u64 combine, scatter through the operator's output map.
// The digit planes ([8][rows][Kp] int8, plane-major) are produced by
// k_tc_digits from the u64 operands with the conv pad / stride / dilation
// gathers applied on the fly (no im2col buffer of u64 values).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "pb_common.cuh"
#include "pb_gemm_maps.cuh"

void pb_keep_pool();

namespace {

constexpr int TC_BM = 128;              // P rows per tile (UMMA M)
constexpr int TC_BN = 64;               // Q rows per tile (UMMA N)
constexpr int TC_BK = 64;               // K bytes per pipeline stage (SWIZZLE_64B row)
constexpr int TC_STAGES = 2;
constexpr int TC_A_PLANE = TC_BM * TC_BK;        // 8 KB
constexpr int TC_B_PLANE = TC_BN * TC_BK;        // 4 KB
constexpr int TC_A_STAGE = 8 * TC_A_PLANE;       // 64 KB
constexpr int TC_B_STAGE = 8 * TC_B_PLANE;       // 32 KB
constexpr int TC_STAGE = TC_A_STAGE + TC_B_STAGE;
constexpr int TC_SMEM = TC_STAGES * TC_STAGE + 1024 + 128;
constexpr int TC_KMAX = 16384;          // contraction per CTA keeping C_0..C_3 exact in int32

// instruction descriptor: D s32, A/B signed int8, both K-major, M = 128, N = 64
constexpr uint32_t TC_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_BN >> 3) << 17) |
                              ((uint32_t)(TC_BM >> 4) << 24);

// shared-memory matrix descriptor, K-major SWIZZLE_64B: 8-row atoms of 64-byte
// rows (512 B, the stride-dimension byte offset), version 1 (sm_100)
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(TC_IDESC), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15},"
      " [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// Output-map of one launch: D[p][q] (P side rows x Q side rows) is element
// (row, col) = swap ? (q, p) : (p, q) of the operator's n x m output.
struct TcEpi {
  GemmMap d;
  int swap;
};

__global__ void __launch_bounds__(128, 1)
    k_tc_ring_gemm(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmQ, TcEpi e, int P,
                   int Q, int kb_per_split, int kb_total, uint64_t mask, int atomic, uint64_t* __restrict__ out) {
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC_STAGES * TC_STAGE);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* done = empty + TC_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = blockIdx.x * TC_BM, q0 = blockIdx.y * TC_BN;
  const int kb0 = blockIdx.z * kb_per_split;
  const int nkb = min(kb_total, kb0 + kb_per_split) - kb0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init_fence();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmP)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
  }
  if (warp == 0) {  // the whole TMEM: 8 accumulators x 64 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {  // ---- TMA producer
    for (int i = 0; i < nkb; ++i) {
      const int s = i % TC_STAGES;
      const uint32_t ph = (uint32_t)(i / TC_STAGES) & 1u;
      if (i >= TC_STAGES) mbar_wait(&empty[s], ph ^ 1u);
      uint8_t* st = smem + s * TC_STAGE;
      mbar_expect_tx(&full[s], TC_STAGE);
      const int kc = (kb0 + i) * TC_BK;
      tma_load_3d(st, &tmP, kc, p0, 0, &full[s]);
      tma_load_3d(st + TC_A_STAGE, &tmQ, kc, q0, 0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // ---- MMA issuer
    for (int i = 0; i < nkb; ++i) {
      const int s = i % TC_STAGES;
      const uint32_t ph = (uint32_t)(i / TC_STAGES) & 1u;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t a0 = smem_addr(smem + s * TC_STAGE), b0 = a0 + TC_A_STAGE;
#pragma unroll
      for (int kk = 0; kk < TC_BK / 32; ++kk) {
        // A digit d against B digits 0 .. 7-d: consecutive MMAs feed different
        // accumulators C_{d+e} (no read-after-write chain on one TMEM tile)
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          const uint64_t da = tc_desc(a0 + d * TC_A_PLANE + kk * 32);
#pragma unroll
          for (int e = 0; e < 8 - d; ++e) {
            const uint64_t db = tc_desc(b0 + e * TC_B_PLANE + kk * 32);
            tc_mma(tmem + (d + e) * TC_BN, da, db, (i > 0 || kk > 0 || d > 0) ? 1u : 0u);
          }
        }
      }
      tc_commit(&empty[s]);  // the stage is free once these MMAs have read it
    }
    tc_commit(done);
  }
  __syncwarp();
  // ---- epilogue: warp w reads TMEM lanes 32w..32w+31 = tile rows p0 + 32w + lane
  mbar_wait(done, 0);
  tc_fence_after();
  const int p = p0 + warp * 32 + lane;
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
  for (int c = 0; c < TC_BN / 16; ++c) {
    uint32_t v[8][16];
#pragma unroll
    for (int s = 0; s < 8; ++s) tmem_ld16(tl + s * TC_BN + c * 16, v[s]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (p < P) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int q = q0 + c * 16 + j;
        if (q >= Q) break;
        uint64_t acc = 0;
#pragma unroll
        for (int s = 0; s < 8; ++s) acc += (uint64_t)(int64_t)(int32_t)v[s][j] << (8 * s);
        const size_t o = e.swap ? gemm_out(e.d, q, p) : gemm_out(e.d, p, q);
        if (atomic) atomicAdd(reinterpret_cast<unsigned long long*>(out + o), (unsigned long long)acc);
        else out[o] = acc & mask;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// Balanced base-256 digit planes of one side, plane-major [8][rows][Kp]:
// side 0 = the output-row operand (gemm_a), side 1 = the output-column one
// (gemm_b); entries k >= kc (the chunk's tail up to Kp) are zero.
// Digits: v = sum_i d_i 256^i with d_i in [-128, 127] is unique and equals
// byte_i(v + C) - 128 for C = 0x80..80 (v < 2^59: no overflow), i.e. the int8
// bytes of (v + C) ^ C -- two 64-bit ops per value.  A thread owns 16
// consecutive contraction entries of one row (one 128-bit store per plane);
// the conv gathers are specialised on the kernel size S and walk the
// contraction index incrementally (no per-element divisions).
// 4 planes (bytes 4h .. 4h+3) of 16 values t[], word q of plane 4h + k =
// byte 4h + k of t[4q .. 4q+3]: a 4 x 4 byte transpose per group of four
// values in 8 byte permutes (two interleave levels).
__device__ __forceinline__ void byte_planes(const uint64_t (&t)[16], int h, uint32_t (&w)[4][4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t a = (uint32_t)(t[4 * q] >> (32 * h)), b = (uint32_t)(t[4 * q + 1] >> (32 * h));
    const uint32_t c = (uint32_t)(t[4 * q + 2] >> (32 * h)), d = (uint32_t)(t[4 * q + 3] >> (32 * h));
    const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);  // a0 b0 a1 b1 | a2 b2 a3 b3
    const uint32_t t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
    w[0][q] = __byte_perm(t0, t2, 0x5410);
    w[1][q] = __byte_perm(t0, t2, 0x7632);
    w[2][q] = __byte_perm(t1, t3, 0x5410);
    w[3][q] = __byte_perm(t1, t3, 0x7632);
  }
}

template <int KIND, int S, int SIDE>
__global__ void __launch_bounds__(256) k_tc_digits(GemmMap d, const uint64_t* __restrict__ src, int rows, int k0,
                                                   int kc, int Kp, uint64_t mask, int8_t* __restrict__ out) {
  const int q16 = Kp / 16;
  const int64_t total = (int64_t)rows * q16;
  const size_t plane = (size_t)rows * Kp;
  constexpr uint64_t C = 0x8080808080808080ull;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int row = total < (1ll << 32) ? (int)((uint32_t)e / (uint32_t)q16) : (int)(e / q16);
    const int kk = 16 * (int)(e - (int64_t)row * q16);
    uint64_t t[16];
    const int nk = kc - kk < 16 ? (kc - kk > 0 ? kc - kk : 0) : 16;
    if (KIND == 3) {  // matmul: strided or contiguous rows, no index arithmetic to save
#pragma unroll
      for (int u = 0; u < 16; ++u)
        t[u] = u < nk ? (SIDE == 0 ? gemm_a(d, src, row, k0 + kk + u) : gemm_b(d, src, k0 + kk + u, row)) : 0ull;
    } else {
      Gather<KIND, S, SIDE> g;
      g.init(d, src, row, k0 + kk);
      if (nk == 16) {  // whole chunks: no per-element tail predicate
#pragma unroll
        for (int u = 0; u < 16; ++u) t[u] = g.next(d);
      } else {
#pragma unroll
        for (int u = 0; u < 16; ++u) t[u] = u < nk ? g.next(d) : 0ull;
      }
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) t[u] = ((t[u] & mask) + C) ^ C;  // the eight int8 digits, little-endian
    uint4* o = reinterpret_cast<uint4*>(out + (size_t)row * Kp + kk);
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // planes 4h .. 4h+3: bytes 4h .. 4h+3 of each of the 16 values
      uint32_t w[4][4];
      byte_planes(t, h, w);
#pragma unroll
      for (int k = 0; k < 4; ++k) o[(4 * h + k) * (plane / 16)] = make_uint4(w[k][0], w[k][1], w[k][2], w[k][3]);
    }
  }
}

// ------------------------------------------------ fused implicit GEMM ---
// The conv operators without digit planes in HBM: eight producer warps gather
// each stage's u64 operand tiles straight from the activations / weights
// (the conv pad / stride / dilation index walks of Gather), turn them into
// balanced digits and store them, byte-transposed, into the SWIZZLE_64B
// K-major layout the UMMA descriptors read (16-byte chunk c of row r at
// r * 64 + ((c ^ ((r >> 1) & 3)) << 4) within each 512-byte atom); a
// generic -> async proxy fence precedes each stage's mbarrier arrival.  The
// MMA warp and the TMEM accumulators are the plane kernel's; eight of the
// producer warps share the epilogue (warp w: TMEM lanes 32 (w % 4), columns
// 32 (w / 4)).
constexpr int TCF_PROD_WARPS = 8;
constexpr int TCF_THREADS = (TCF_PROD_WARPS + 1) * 32;

// 16 gathered u64 -> the 16-byte chunk of each of the 8 digit planes
__device__ __forceinline__ void digit_chunk(uint64_t (&t)[16], uint4 (&o)[8]) {
  constexpr uint64_t C = 0x8080808080808080ull;
#pragma unroll
  for (int u = 0; u < 16; ++u) t[u] = (t[u] + C) ^ C;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t w[4][4];
    byte_planes(t, h, w);
#pragma unroll
    for (int k = 0; k < 4; ++k) o[4 * h + k] = make_uint4(w[k][0], w[k][1], w[k][2], w[k][3]);
  }
}

// Fill `nrow_tile` rows x 64 contraction entries of one side's stage tile
// (8 planes of nrow_tile x 64 bytes at `tile`), rows row0.. (< nrows valid),
// contraction k0.. (< K valid); producer thread pt of TCF_PROD_WARPS * 32.
template <int KIND, int S, int SIDE>
__device__ __forceinline__ void fill_tile(uint8_t* tile, int nrow_tile, const GemmMap& d, const uint64_t* src,
                                          int row0, int nrows, int64_t k0, int64_t K, uint64_t mask, int pt) {
  constexpr int NT = TCF_PROD_WARPS * 32;
  const int chunks = nrow_tile * 4;  // 16-value chunks per stage tile
  for (int c = pt; c < chunks; c += NT) {
    const int r = c % nrow_tile, c16 = c / nrow_tile;  // consecutive threads: consecutive rows (coalesced gathers)
    const int row = row0 + r;
    const int64_t k = k0 + 16 * c16;
    uint64_t t[16];
    const int nk = (row < nrows) ? (int)(K - k < 16 ? (K - k > 0 ? K - k : 0) : 16) : 0;
    if (nk > 0) {
      Gather<KIND, S, SIDE> g;
      g.init(d, src, row, (int)k);
#pragma unroll
      for (int u = 0; u < 16; ++u) t[u] = u < nk ? (g.next(d) & mask) : 0ull;
    } else {
#pragma unroll
      for (int u = 0; u < 16; ++u) t[u] = 0ull;
    }
    uint4 o[8];
    digit_chunk(t, o);
    const uint32_t off = (uint32_t)r * 64u + ((uint32_t)(c16 ^ ((r >> 1) & 3)) << 4);
#pragma unroll
    for (int p = 0; p < 8; ++p) *reinterpret_cast<uint4*>(tile + (size_t)p * nrow_tile * 64 + off) = o[p];
  }
}

template <int KIND, int S, int PSIDE>
__global__ void __launch_bounds__(TCF_THREADS, 1)
    k_tc_conv_fused(GemmMap d, const uint64_t* __restrict__ srcP, const uint64_t* __restrict__ srcQ, TcEpi e, int P,
                    int Q, int64_t K, int kb_per_split, int kb_total, uint64_t mask, int atomic,
                    uint64_t* __restrict__ out) {
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC_STAGES * TC_STAGE);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* done = empty + TC_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = blockIdx.x * TC_BM, q0 = blockIdx.y * TC_BN;
  const int kb0 = blockIdx.z * kb_per_split;
  const int nkb = min(kb_total, kb0 + kb_per_split) - kb0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], TCF_PROD_WARPS);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init_fence();
  }
  if (warp == TCF_PROD_WARPS) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr int QSIDE = 1 - PSIDE;
  if (warp < TCF_PROD_WARPS) {  // ---- producers
    const int pt = threadIdx.x;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % TC_STAGES;
      const uint32_t ph = (uint32_t)(i / TC_STAGES) & 1u;
      if (i >= TC_STAGES) mbar_wait(&empty[s], ph ^ 1u);
      uint8_t* st = smem + s * TC_STAGE;
      const int64_t k0 = (int64_t)(kb0 + i) * TC_BK;
      fill_tile<KIND, S, PSIDE>(st, TC_BM, d, srcP, p0, P, k0, K, mask, pt);
      fill_tile<KIND, S, QSIDE>(st + TC_A_STAGE, TC_BN, d, srcQ, q0, Q, k0, K, mask, pt);
      fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core's async proxy
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
    }
  } else if (lane == 0) {  // ---- MMA issuer
    for (int i = 0; i < nkb; ++i) {
      const int s = i % TC_STAGES;
      const uint32_t ph = (uint32_t)(i / TC_STAGES) & 1u;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t a0 = smem_addr(smem + s * TC_STAGE), b0 = a0 + TC_A_STAGE;
#pragma unroll
      for (int kk = 0; kk < TC_BK / 32; ++kk) {
#pragma unroll
        for (int dd = 0; dd < 8; ++dd) {
          const uint64_t da = tc_desc(a0 + dd * TC_A_PLANE + kk * 32);
#pragma unroll
          for (int ee = 0; ee < 8 - dd; ++ee) {
            const uint64_t db = tc_desc(b0 + ee * TC_B_PLANE + kk * 32);
            tc_mma(tmem + (dd + ee) * TC_BN, da, db, (i > 0 || kk > 0 || dd > 0) ? 1u : 0u);
          }
        }
      }
      tc_commit(&empty[s]);
    }
    tc_commit(done);
  }
  __syncwarp();
  // ---- epilogue: warps 0..7, TMEM lanes 32 (w % 4), column half w / 4
  if (warp < 8) {
    mbar_wait(done, 0);
    tc_fence_after();
    const int p = p0 + (warp & 3) * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      const int col = (warp >> 2) * 32 + c * 16;
      uint32_t v[8][16];
#pragma unroll
      for (int s = 0; s < 8; ++s) tmem_ld16(tl + s * TC_BN + col, v[s]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (p < P) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int q = q0 + col + j;
          if (q >= Q) break;
          uint64_t acc = 0;
#pragma unroll
          for (int s = 0; s < 8; ++s) acc += (uint64_t)(int64_t)(int32_t)v[s][j] << (8 * s);
          const size_t o = e.swap ? gemm_out(e.d, q, p) : gemm_out(e.d, p, q);
          if (atomic) atomicAdd(reinterpret_cast<unsigned long long*>(out + o), (unsigned long long)acc);
          else out[o] = acc & mask;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == TCF_PROD_WARPS)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

template <int SIDE>
void launch_digits(const GemmMap& d, const uint64_t* src, int rows, int k0, int kc, int Kp, uint64_t mask, int8_t* out,
                   cudaStream_t st) {
  const int grid = pb_grid_1d((int64_t)rows * (Kp / 16), 256);
#define PB_TCD(K, S) k_tc_digits<K, S, SIDE><<<grid, 256, 0, st>>>(d, src, rows, k0, kc, Kp, mask, out)
#define PB_TCD_S(K)          \
  switch (d.s) {             \
    case 1: PB_TCD(K, 1); return; \
    case 3: PB_TCD(K, 3); return; \
    case 5: PB_TCD(K, 5); return; \
    default: PB_TCD(3, 1); return; \
  }
  switch (d.kind) {  // the generic gathers (gemm_a / gemm_b) for matmuls and other kernel sizes
    case PB_CONV_FWD: PB_TCD_S(PB_CONV_FWD);
    case PB_CONV_BWDX: PB_TCD_S(PB_CONV_BWDX);
    case PB_CONV_GRADW: PB_TCD_S(PB_CONV_GRADW);
    default: PB_TCD(3, 1); return;
  }
#undef PB_TCD_S
#undef PB_TCD
}

__global__ void k_tc_mask(uint64_t* v, int64_t n, uint64_t m) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] &= m;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Tensor map over planes [8][rows][Kp] int8: box = 64 K bytes x box_rows x 8 planes, SWIZZLE_64B.
bool plane_map(CUtensorMap* tm, const int8_t* base, int rows, int Kp, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, 8};
  const cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)rows * (cuuint64_t)Kp};
  const cuuint32_t box[3] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows, 8};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// K blocks per CTA for `tiles` output tiles over `kb` K blocks: one CTA per SM
// (192 KB of shared memory), so the launch takes ceil(tiles * splits / 148)
// waves of about kps + 2 block-times each (2: the TMEM epilogue and its
// atomics).  Minimise that instead of doubling the splits until the grid
// covers the GPU, which left a 12-CTA second wave at 160 CTAs.
static int pick_kps(int tiles, int kb) {
  const int kmax = TC_KMAX / TC_BK;
  int best = kb < kmax ? kb : kmax;
  int64_t best_cost = INT64_MAX;
  for (int kps = best; kps >= 1; --kps) {
    const int64_t splits = (kb + kps - 1) / kps;
    const int64_t cost = (((int64_t)tiles * splits + 147) / 148) * (kps + 2);
    if (cost < best_cost) best_cost = cost, best = kps;  // ties keep the fewer splits
  }
  return best;
}

// out (n x m, through d's output map) = A (n x K) . B (K x m) mod 2^ell on the
// tensor cores.  Contractions are processed in chunks whose digit planes stay
// under ~512 MB; within a chunk the K blocks split over gridDim.z so that the
// grid covers the GPU, partial sums meeting in u64 atomics.
template <int KIND, int S, int PSIDE>
int launch_conv_fused(const GemmMap& d, const uint64_t* A, const uint64_t* Bm, int n, int64_t K, int m, uint64_t mask,
                      uint64_t* out, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_tc_conv_fused<KIND, S, PSIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM) !=
        cudaSuccess)
      return pb_set_error(PB_ERR_CUDA, "fused tcgen05 conv: shared-memory opt-in failed");
    attr = true;
  }
  const int swap = PSIDE;  // P = the output-column operand exactly when the sides are swapped
  const int P = swap ? m : n, Q = swap ? n : m;
  const int tiles = ((P + TC_BM - 1) / TC_BM) * ((Q + TC_BN - 1) / TC_BN);
  const int kb = (int)((K + TC_BK - 1) / TC_BK);
  const int kps = pick_kps(tiles, kb);
  const int splits = (kb + kps - 1) / kps;
  const int atomic = splits > 1;
  const TcEpi e{d, swap};
  if (atomic) cudaMemsetAsync(out, 0, (size_t)n * m * sizeof(uint64_t), st);
  dim3 grid((unsigned)((P + TC_BM - 1) / TC_BM), (unsigned)((Q + TC_BN - 1) / TC_BN), (unsigned)splits);
  k_tc_conv_fused<KIND, S, PSIDE><<<grid, TCF_THREADS, TC_SMEM, st>>>(d, PSIDE ? Bm : A, PSIDE ? A : Bm, e, P, Q, K,
                                                                      kps, kb, mask, atomic, out);
  if (atomic) {
    const int64_t no = (int64_t)n * m;
    k_tc_mask<<<pb_grid_1d(no, 256), 256, 0, st>>>(out, no, mask);
  }
  return cudaPeekAtLastError() == cudaSuccess ? PB_OK : pb_set_error(PB_ERR_CUDA, "fused tcgen05 conv launch failed");
}

template <int KIND>
int conv_fused(const GemmMap& d, const uint64_t* A, const uint64_t* Bm, int n, int64_t K, int m, uint64_t mask,
               uint64_t* out, cudaStream_t st) {
  const bool swap = n < m;
#define PB_TCF(S) return swap ? launch_conv_fused<KIND, S, 1>(d, A, Bm, n, K, m, mask, out, st) \
                              : launch_conv_fused<KIND, S, 0>(d, A, Bm, n, K, m, mask, out, st)
  switch (d.s) {
    case 1: PB_TCF(1);
    case 3: PB_TCF(3);
    default: PB_TCF(5);
  }
#undef PB_TCF
}

int pb_tc_ring_gemm(const GemmMap& d, const uint64_t* A, const uint64_t* Bm, int n, int64_t K, int m, int ell,
                    uint64_t* out, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_tc_ring_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM) != cudaSuccess)
      return pb_set_error(PB_ERR_CUDA, "tcgen05 GEMM: shared-memory opt-in failed");
    // the digit planes are stream-ordered allocations: keep them cached in the
    // device's default pool (re-mapping hundreds of MB per call costs milliseconds)
    pb_keep_pool();
    attr = true;
  }
  const uint64_t mask = ell >= 64 ? ~0ull : ((1ull << ell) - 1);
  // conv operators with the kernel sizes the models use, up to 2^29 MACs: the
  // fused implicit GEMM (digits built in shared memory by the producer warps,
  // no planes in HBM); above, the gathers of eight producer warps cannot keep
  // the tensor core fed and the plane kernels win (CIFAR conv2 0.18 vs 0.19 ms,
  // conv1 0.10 vs 0.08 ms; profiles/r02_ring_gemm_backends*.jsonl; re-measured
  // with pick_kps: conv2 fwd / dX / dW planes 0.15 / 0.15 / 0.19 ms, fused
  // 0.16 / 0.23 / 0.21, CIFAR step 8.2 vs 8.4 ms)
  if (d.kind <= PB_CONV_GRADW && (d.s == 1 || d.s == 3 || d.s == 5) && (double)n * m * (double)K < 536870912.0) {
    switch (d.kind) {
      case PB_CONV_FWD: return conv_fused<PB_CONV_FWD>(d, A, Bm, n, K, m, mask, out, st);
      case PB_CONV_BWDX: return conv_fused<PB_CONV_BWDX>(d, A, Bm, n, K, m, mask, out, st);
      default: return conv_fused<PB_CONV_GRADW>(d, A, Bm, n, K, m, mask, out, st);
    }
  }
  if (!encode_fn()) return pb_set_error(PB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int swap = n < m;  // the longer output side takes the 128-row UMMA M dimension
  const int P = swap ? m : n, Q = swap ? n : m;
  const int p_side = swap ? 1 : 0;
  // chunk the contraction: planes of one chunk (8 (P + Q) Kc bytes) <= 512 MB
  int64_t Kc = ((int64_t)512 << 20) / (8 * (int64_t)(P + Q));
  Kc = Kc / TC_BK * TC_BK;
  if (Kc < TC_BK) Kc = TC_BK;
  if (Kc > K) Kc = (K + TC_BK - 1) / TC_BK * TC_BK;
  const int nchunks = (int)((K + Kc - 1) / Kc);
  const int tiles = ((P + TC_BM - 1) / TC_BM) * ((Q + TC_BN - 1) / TC_BN);
  const int kb_chunk = (int)(Kc / TC_BK);
  const int kps = pick_kps(tiles, kb_chunk);  // K blocks per CTA
  const int splits = (kb_chunk + kps - 1) / kps;
  const int atomic = nchunks > 1 || splits > 1;
  int8_t *dp = nullptr, *dq = nullptr;
  if (cudaMallocAsync((void**)&dp, (size_t)8 * P * Kc, st) != cudaSuccess ||
      cudaMallocAsync((void**)&dq, (size_t)8 * Q * Kc, st) != cudaSuccess)
    return pb_set_error(PB_ERR_CUDA, "tcgen05 GEMM: digit-plane allocation failed");
  CUtensorMap tmP, tmQ;
  if (!plane_map(&tmP, dp, P, (int)Kc, TC_BM) || !plane_map(&tmQ, dq, Q, (int)Kc, TC_BN)) {
    cudaFreeAsync(dq, st);
    cudaFreeAsync(dp, st);
    return pb_set_error(PB_ERR_CUDA, "tcgen05 GEMM: tensor-map encoding failed");
  }
  const TcEpi e{d, swap};
  if (atomic) cudaMemsetAsync(out, 0, (size_t)n * m * sizeof(uint64_t), st);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int64_t k0 = (int64_t)ch * Kc;
    const int kc = (int)((K - k0) < Kc ? (K - k0) : Kc);
    const int kb = (kc + TC_BK - 1) / TC_BK;
    const int sp = (kb + kps - 1) / kps;
    if (p_side == 0) {
      launch_digits<0>(d, A, P, (int)k0, kc, (int)Kc, mask, dp, st);
      launch_digits<1>(d, Bm, Q, (int)k0, kc, (int)Kc, mask, dq, st);
    } else {
      launch_digits<1>(d, Bm, P, (int)k0, kc, (int)Kc, mask, dp, st);
      launch_digits<0>(d, A, Q, (int)k0, kc, (int)Kc, mask, dq, st);
    }
    dim3 grid((unsigned)((P + TC_BM - 1) / TC_BM), (unsigned)((Q + TC_BN - 1) / TC_BN), (unsigned)sp);
    k_tc_ring_gemm<<<grid, 128, TC_SMEM, st>>>(tmP, tmQ, e, P, Q, kps, kb, mask, atomic, out);
  }
  if (atomic) {
    const int64_t no = (int64_t)n * m;
    k_tc_mask<<<pb_grid_1d(no, 256), 256, 0, st>>>(out, no, mask);
  }
  cudaFreeAsync(dq, st);
  cudaFreeAsync(dp, st);
  return cudaPeekAtLastError() == cudaSuccess ? PB_OK : pb_set_error(PB_ERR_CUDA, "tcgen05 GEMM launch failed");
}

int pb_tc_conv(int kind, const uint64_t* a, const uint64_t* b, int B, int ci, int co, int H, int W, int s, int p,
               int st_, int oh, int ow, int ell, uint64_t* out, cudaStream_t st) {
  GemmMap d = {};
  d.kind = kind, d.B = B, d.ci = ci, d.co = co, d.H = H, d.W = W, d.s = s, d.p = p, d.st = st_, d.oh = oh, d.ow = ow;
  int n, m;
  int64_t K;
  const uint64_t *A, *Bm;
  if (kind == PB_CONV_FWD) { n = co; K = (int64_t)ci * s * s; m = B * oh * ow; A = b; Bm = a; }      // A = W, B = X
  else if (kind == PB_CONV_BWDX) { n = ci; K = (int64_t)co * s * s; m = B * H * W; A = b; Bm = a; }  // A = W, B = dY
  else { n = co; K = (int64_t)B * oh * ow; m = ci * s * s; A = b; Bm = a; }                          // A = dY, B = X
  return pb_tc_ring_gemm(d, A, Bm, n, K, m, ell, out, st);
}

int pb_tc_matmul(const uint64_t* a, const uint64_t* b, int n, int k, int m, int ta, int tb, int ell, uint64_t* out,
                 cudaStream_t st) {
  GemmMap d = {};
  d.kind = 3, d.n = n, d.k = k, d.m = m, d.ta = ta, d.tb = tb;
  return pb_tc_ring_gemm(d, a, b, n, k, m, ell, out, st);
}
