// Experimental NTT variants (scripts/exp_ntt.py drives them on the B200).
// Not part of the product library: variants that win get folded into
// csrc/pb_ntt.cuh / pb_poly.cu.
#include "../paper_2403_11166_b200/csrc/pb_ntt.cuh"

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int LOGN, int MINB>
__global__ void __launch_bounds__(1 << (LOGN - 5), MINB) k_v0(PbDev P, uint32_t* rows, int64_t n_rows) {
  using Nt = pb::Ntt<LOGN>;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    const int limb = (int)(r % P.L);
    const uint32_t q = P.q[limb];
    uint32_t* row = rows + r * Nt::N;
    uint32_t a[32];
    Nt::gld1(row, a, tid);
    Nt::forward(a, sm, P.tw_fwd + (size_t)limb * Nt::N, P.tw3_fwd + (size_t)limb * P.tw3_stride, tid, q);
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = pb::canon4(a[c], q);
    Nt::gst3(row, a, tid);
    __syncthreads();
  }
}

// v5: blocks visit rows limb-major (all concurrently running CTAs share a
// limb, so its twiddle tables stay hot in L1/L2).
template <int LOGN, int MINB>
__global__ void __launch_bounds__(1 << (LOGN - 5), MINB) k_v5(PbDev P, uint32_t* rows, int64_t n_rows) {
  using Nt = pb::Ntt<LOGN>;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  const int64_t per = n_rows / P.L;
  for (int64_t b = blockIdx.x; b < n_rows; b += gridDim.x) {
    const int limb = (int)(b / per);
    const int64_t r = (b % per) * P.L + limb;
    const uint32_t q = P.q[limb];
    uint32_t* row = rows + r * Nt::N;
    uint32_t a[32];
    Nt::gld1(row, a, tid);
    Nt::forward(a, sm, P.tw_fwd + (size_t)limb * Nt::N, P.tw3_fwd + (size_t)limb * P.tw3_stride, tid, q);
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = pb::canon4(a[c], q);
    Nt::gst3(row, a, tid);
    __syncthreads();
  }
}

// Persistent CTAs; the next row is prefetched into a shared-memory landing
// buffer with a bulk async copy (TMA engine) while the current row computes.
template <int LOGN, int MINB>
__global__ void __launch_bounds__(1 << (LOGN - 5), MINB) k_v3(PbDev P, uint32_t* rows, int64_t n_rows, int lm) {
  using Nt = pb::Ntt<LOGN>;
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* lb = sm + ((Nt::SMEM_WORDS + 3) & ~3);
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  int64_t r = blockIdx.x;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t per = n_rows / P.L;
  auto rowof = [&](int64_t b) { return lm ? (b % per) * P.L + b / per : b; };
  if (tid == 0 && r < n_rows) {
    mbar_expect_tx(&bar, Nt::N * 4);
    bulk_g2s(lb, rows + rowof(r) * Nt::N, Nt::N * 4, &bar);
  }
  uint32_t phase = 0;
  for (; r < n_rows; r += gridDim.x) {
    const int limb = (int)(rowof(r) % P.L);
    const uint32_t q = P.q[limb];
    uint32_t a[32];
    mbar_wait(&bar, phase);
    phase ^= 1;
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = lb[tid + Nt::T * c];
    __syncthreads();
    if (tid == 0 && r + gridDim.x < n_rows) {
      fence_proxy_async();
      mbar_expect_tx(&bar, Nt::N * 4);
      bulk_g2s(lb, rows + rowof(r + gridDim.x) * Nt::N, Nt::N * 4, &bar);
    }
    Nt::forward(a, sm, P.tw_fwd + (size_t)limb * Nt::N, P.tw3_fwd + (size_t)limb * P.tw3_stride, tid, q);
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = pb::canon4(a[c], q);
    Nt::gst3(rows + rowof(r) * Nt::N, a, tid);
    __syncthreads();
  }
}

template <int LOGN, int MINB>
int launch(int variant, const PbDev& P, uint32_t* rows, int64_t n, int ctas_per_sm, cudaStream_t st) {
  using Nt = pb::Ntt<LOGN>;
  if (variant == 0) {
    const size_t smem = Nt::SMEM_WORDS * 4;
    cudaFuncSetAttribute(k_v0<LOGN, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_v0<LOGN, MINB><<<(unsigned)n, Nt::T, smem, st>>>(P, rows, n);
  } else if (variant == 5 || variant == 6) {
    const size_t smem = Nt::SMEM_WORDS * 4;
    cudaFuncSetAttribute(k_v5<LOGN, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (variant == 6) cudaFuncSetAttribute(k_v5<LOGN, MINB>, cudaFuncAttributePreferredSharedMemoryCarveout, 50);
    k_v5<LOGN, MINB><<<(unsigned)n, Nt::T, smem, st>>>(P, rows, n);
  } else {
    const size_t smem = ((Nt::SMEM_WORDS + 3) & ~3) * 4 + Nt::N * 4;
    cudaFuncSetAttribute(k_v3<LOGN, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_v3<LOGN, MINB>, cudaFuncAttributePreferredSharedMemoryCarveout, ctas_per_sm >= 100 ? ctas_per_sm - 100 : 100);
    if (ctas_per_sm >= 100) ctas_per_sm = 0;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_v3<LOGN, MINB>, Nt::T, smem);
    if (ctas_per_sm > 0 && ctas_per_sm < occ) occ = ctas_per_sm;
    const int64_t g = (int64_t)sms * (occ > 0 ? occ : 1);
    k_v3<LOGN, MINB><<<(unsigned)(n < g ? n : g), Nt::T, smem, st>>>(P, rows, n, variant == 7 ? 1 : 0);
  }
  return (int)cudaGetLastError();
}

}  // namespace

extern "C" int exp_ntt_fwd(const pb_ctx* ctx, int variant, int minb, uint32_t* rows, int64_t n, int ctas_per_sm,
                           void* stream) {
  const PbDev& P = ctx->dev;
  cudaStream_t st = (cudaStream_t)stream;
  if (P.logN != 13) return -1;
  switch (minb) {
    case 3: return launch<13, 3>(variant, P, rows, n, ctas_per_sm, st);
    case 4: return launch<13, 4>(variant, P, rows, n, ctas_per_sm, st);
    default: return launch<13, 1>(variant, P, rows, n, ctas_per_sm, st);
  }
}

extern "C" int exp_occupancy(int variant, int minb) {
  using Nt = pb::Ntt<13>;
  int occ = 0;
  if (variant == 0) {
    const size_t smem = Nt::SMEM_WORDS * 4;
    if (minb == 3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_v0<13, 3>, Nt::T, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_v0<13, 1>, Nt::T, smem);
  } else {
    const size_t smem = ((Nt::SMEM_WORDS + 3) & ~3) * 4 + Nt::N * 4;
    if (minb == 3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_v3<13, 3>, Nt::T, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_v3<13, 1>, Nt::T, smem);
  }
  return occ;
}

// ---- wide NTT (pb_nttw.cuh) experiments ----
#include "../paper_2403_11166_b200/csrc/pb_nttw.cuh"
namespace {
template <int LOGN, int LOGV>
__global__ void __launch_bounds__(1 << (LOGN - LOGV)) k_wfwd(PbDev P, uint32_t* rows, int64_t n_rows) {
  using W = pb::NttW<LOGN, LOGV>;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    const int limb = (int)(r % P.L);
    const uint32_t q = P.q[limb];
    uint32_t a[W::V];
    W::gld1(rows + r * W::N, a, tid);
    W::forward(a, sm, P.tw_fwd + (size_t)limb * W::N, tid, q);
#pragma unroll
    for (int c = 0; c < W::V; ++c) a[c] = pb::canon4(a[c], q);
    W::gst_dev(rows + r * W::N, a, tid);
    __syncthreads();
  }
}
template <int LOGN, int LOGV>
__global__ void __launch_bounds__(1 << (LOGN - LOGV)) k_winv(PbDev P, uint32_t* rows, int64_t n_rows) {
  using W = pb::NttW<LOGN, LOGV>;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    const int limb = (int)(r % P.L);
    const uint32_t q = P.q[limb];
    uint32_t a[W::V];
    W::gld_dev(rows + r * W::N, a, tid);
    W::inverse(a, sm, P.tw_inv + (size_t)limb * W::N, tid, q);
    const uint32_t ni = P.ninv[limb], nis = P.ninv_sh[limb];
#pragma unroll
    for (int c = 0; c < W::V; ++c) a[c] = mul_shoup(a[c], ni, nis, q);
    W::gst1(rows + r * W::N, a, tid);
    __syncthreads();
  }
}
template <int LOGV>
int wlaunch(int inv, const PbDev& P, uint32_t* rows, int64_t n, cudaStream_t st) {
  using W = pb::NttW<13, LOGV>;
  const size_t smem = W::SMEM_WORDS * 4;
  if (inv) {
    cudaFuncSetAttribute(k_winv<13, LOGV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_winv<13, LOGV><<<(unsigned)n, W::T, smem, st>>>(P, rows, n);
  } else {
    cudaFuncSetAttribute(k_wfwd<13, LOGV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_wfwd<13, LOGV><<<(unsigned)n, W::T, smem, st>>>(P, rows, n);
  }
  return (int)cudaGetLastError();
}
}  // namespace
extern "C" int exp_wntt(const pb_ctx* ctx, int logv, int inv, uint32_t* rows, int64_t n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (ctx->dev.logN != 13) return -1;
  if (logv == 3) return wlaunch<3>(inv, ctx->dev, rows, n, st);
  if (logv == 4) return wlaunch<4>(inv, ctx->dev, rows, n, st);
  return -2;
}
