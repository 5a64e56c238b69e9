// pb_poly.cu — context, polynomial engine entry points (the sm_100a
// replacements of the reference kernel tier K:31-199) and error plumbing.
#include <cstdio>
#include <cstring>
#include <new>

#include "pb_ntt.cuh"

#include <cooperative_groups.h>

// ------------------------------------------------------------------ errors --
static thread_local char g_err[512] = "";

int pb_set_error(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}
int pb_set_cuda_error(cudaError_t e) {
  snprintf(g_err, sizeof(g_err), "CUDA error: %s", cudaGetErrorString(e));
  return PB_ERR_CUDA;
}

extern "C" const char* pb_last_error(void) { return g_err; }
extern "C" int pb_abi_version(void) { return PB_ABI_VERSION; }
extern "C" int pb_device_sm_count(int* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return pb_set_cuda_error(e);
  e = cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return pb_set_cuda_error(e);
  return PB_OK;
}

// --------------------------------------------------------- host mod arith --
static uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t q) {
  return (uint64_t)((unsigned __int128)a * b % q);
}
static uint64_t h_powmod(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = h_mulmod(r, a, q);
    a = h_mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
static uint32_t h_shoup(uint32_t w, uint32_t q) { return (uint32_t)(((uint64_t)w << 32) / q); }
static uint32_t h_bitrev(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

// ------------------------------------------------------------------ context --
// Stream-ordered scratch (encryption noise, digit planes) comes from the
// device's default memory pool: keep freed blocks cached there instead of
// unmapping them at every synchronisation.
void pb_keep_pool() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done = true;
}

extern "C" int pb_ctx_create(const pb_params* p, pb_ctx** out) {
  if (!p || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  pb_keep_pool();
  const int N = p->N, L = p->L;
  int logN = 0;
  while ((1 << logN) < N) ++logN;
  if (N < 4 || N > 32768 || (1 << logN) != N) return pb_set_error(PB_ERR_PARAMS, "N must be a power of two in [4, 32768]");
  if (L < 1 || L > PB_MAX_LIMBS) return pb_set_error(PB_ERR_PARAMS, "L must be in [1, 8]");
  if (p->ell < 2 || p->ell > 62) return pb_set_error(PB_ERR_PARAMS, "ell must be in [2, 62]");
  for (int i = 0; i < L; ++i) {
    const uint64_t q = p->q[i];
    if (q < 3 || q >= (1u << 30)) return pb_set_error(PB_ERR_PARAMS, "moduli must be < 2^30");
    if ((q - 1) % (2ull * N) != 0) return pb_set_error(PB_ERR_PARAMS, "moduli must be 1 mod 2N");
    if (h_powmod(p->psi[i], N, q) != q - 1) return pb_set_error(PB_ERR_PARAMS, "psi is not a primitive 2N-th root");
  }
  pb_ctx* c = new (std::nothrow) pb_ctx();
  if (!c) return pb_set_error(PB_ERR_ARG, "out of host memory");
  c->host = *p;
  PbDev& d = c->dev;
  memset(&d, 0, sizeof(d));
  d.N = N; d.logN = logN; d.L = L; d.ell = p->ell;
  d.t_mask = (p->ell >= 64) ? ~0ull : ((1ull << p->ell) - 1);
  const uint64_t t = 1ull << p->ell;
  for (int i = 0; i < L; ++i) {
    const uint32_t q = p->q[i];
    d.q[i] = q;
    d.ninv[i] = (uint32_t)h_powmod(N, q - 2, q);
    d.ninv_sh[i] = h_shoup(d.ninv[i], q);
    d.delta[i] = p->delta_mod_q[i] % q;
    d.delta_sh[i] = h_shoup(d.delta[i], q);
    d.mu[i] = (uint64_t)(((unsigned __int128)1 << 64) / q);
    d.inv_q32[i] = 4294967296.0 / (double)q;
    {
      uint32_t inv = 1;  // Newton iteration for q^-1 mod 2^32 (q odd)
      for (int it = 0; it < 5; ++it) inv *= 2u - q * inv;
      d.qn[i] = 0u - inv;
      d.r2[i] = (uint32_t)((1ull << 32) % q);
      d.r2_sh[i] = h_shoup(d.r2[i], q);
    }
    d.tmod[i] = (uint32_t)(t % q);
    d.pinv[i] = p->garner_prefix_inv[i] % q;
    d.pinv_sh[i] = h_shoup(d.pinv[i], q);
    uint64_t prod = 1;
    for (int k = 0; k < PB_MAX_LIMBS; ++k) {
      d.pmod[i][k] = (uint32_t)prod;
      d.pmod_sh[i][k] = h_shoup(d.pmod[i][k], q);
      if (k < L) prod = h_mulmod(prod, p->q[k] % q, q);
    }
    d.sc_int[i] = p->scale_int[i];
    d.sc_frac[i] = p->scale_frac[i];
  }
  // twiddle tables {w, shoup(w)}: psi^bitrev(i) and psi^-bitrev(i)  (K:22-29)
  const size_t n_tw = (size_t)L * N;
  uint2* h_f = (uint2*)malloc(n_tw * sizeof(uint2));
  uint2* h_i = (uint2*)malloc(n_tw * sizeof(uint2));
  uint64_t* pw = (uint64_t*)malloc((size_t)N * sizeof(uint64_t));
  uint64_t* ipw = (uint64_t*)malloc((size_t)N * sizeof(uint64_t));
  if (!h_f || !h_i || !pw || !ipw) {
    free(h_f); free(h_i); free(pw); free(ipw); delete c;
    return pb_set_error(PB_ERR_ARG, "out of host memory");
  }
  for (int l = 0; l < L; ++l) {
    const uint64_t q = p->q[l], psi = p->psi[l] % q, ipsi = h_powmod(psi, q - 2, q);
    uint64_t a = 1, b = 1;
    for (int k = 0; k < N; ++k) {
      pw[k] = a; ipw[k] = b;
      a = h_mulmod(a, psi, q);
      b = h_mulmod(b, ipsi, q);
    }
    for (int k = 0; k < N; ++k) {
      const uint32_t br = h_bitrev((uint32_t)k, logN);
      const uint32_t wf = (uint32_t)pw[br], wi = (uint32_t)ipw[br];
      h_f[(size_t)l * N + k] = make_uint2(wf, h_shoup(wf, (uint32_t)q));
      h_i[(size_t)l * N + k] = make_uint2(wi, h_shoup(wi, (uint32_t)q));
    }
    // N^-1 folded into the last inverse stage (pb_ntt.cuh inverse_scaled)
    d.w0n[l] = (uint32_t)h_mulmod(h_i[(size_t)l * N + 1].x, d.ninv[l], q);
    d.w0n_sh[l] = h_shoup(d.w0n[l], (uint32_t)q);
  }
  free(pw); free(ipw);
  // P3-stage tables (register NTT, N >= 2048): stage D (s = logN-5+D) at
  // uint2 offset (2^D-1)*T; for D >= 1 the pair (2v, 2v+1) of thread tid is
  // uint4 #(v*T + tid), so each warp load is contiguous (pb_ntt.cuh tw3).
  const int T = N / 32;
  const size_t n3 = (logN >= 11) ? (size_t)31 * T : 0;
  uint2* h3f = n3 ? (uint2*)malloc((size_t)L * n3 * sizeof(uint2)) : nullptr;
  uint2* h3i = n3 ? (uint2*)malloc((size_t)L * n3 * sizeof(uint2)) : nullptr;
  if (n3 && (!h3f || !h3i)) {
    free(h_f); free(h_i); free(h3f); free(h3i); delete c;
    return pb_set_error(PB_ERR_ARG, "out of host memory");
  }
  for (int l = 0; n3 && l < L; ++l) {
    for (int D = 0; D < 5; ++D) {
      const int s = logN - 5 + D;
      const size_t off = (size_t)l * n3 + (size_t)((1 << D) - 1) * T;
      for (int tid = 0; tid < T; ++tid) {
        for (int r = 0; r < (1 << D); ++r) {
          const size_t src = (size_t)l * N + (1u << s) + ((size_t)tid << D) + r;
          const size_t dst = (D == 0) ? off + tid : off + 2 * ((size_t)(r >> 1) * T + tid) + (r & 1);
          h3f[dst] = h_f[src];
          h3i[dst] = h_i[src];
        }
      }
    }
  }
  cudaError_t e = cudaMalloc(&c->d_tw_fwd, n_tw * sizeof(uint2));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_tw_inv, n_tw * sizeof(uint2));
  if (e == cudaSuccess) e = cudaMemcpy(c->d_tw_fwd, h_f, n_tw * sizeof(uint2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(c->d_tw_inv, h_i, n_tw * sizeof(uint2), cudaMemcpyHostToDevice);
  if (n3) {
    if (e == cudaSuccess) e = cudaMalloc(&c->d_tw3_fwd, (size_t)L * n3 * sizeof(uint2));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_tw3_inv, (size_t)L * n3 * sizeof(uint2));
    if (e == cudaSuccess) e = cudaMemcpy(c->d_tw3_fwd, h3f, (size_t)L * n3 * sizeof(uint2), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(c->d_tw3_inv, h3i, (size_t)L * n3 * sizeof(uint2), cudaMemcpyHostToDevice);
  }
  // N = 32768: tables of the two half transforms (pb_ntt k_ntt_*_c2).  Half b,
  // stage s' (m' = 2^s' groups) of the N/2-point transform is stage s' + 1 of
  // the full one restricted to groups b m' .. (b+1) m' - 1, twiddle index
  // 2 m' + b m' + g = I + (1 + b) m' for local index I = m' + g.
  if (e == cudaSuccess && logN == 15) {
    const int Nh = N / 2, Th = Nh / 32;
    const size_t n3s = (size_t)31 * Th;
    const size_t per_dir = (size_t)2 * L * (Nh + n3s);
    uint2* hs = (uint2*)calloc(2 * per_dir, sizeof(uint2));
    if (!hs) e = cudaErrorMemoryAllocation;
    for (int dir = 0; hs && dir < 2; ++dir) {
      uint2* tab = hs + dir * per_dir;                 // [2][L][Nh]
      uint2* t3 = tab + (size_t)2 * L * Nh;            // [2][L][n3s]
      uint2* full = dir ? h_i : h_f;
      for (int b = 0; b < 2; ++b)
        for (int l = 0; l < L; ++l) {
          uint2* sub = tab + ((size_t)b * L + l) * Nh;
          for (int I = 1; I < Nh; ++I) {
            int mp = 1;
            while (2 * mp <= I) mp *= 2;
            sub[I] = full[(size_t)l * N + I + (1 + b) * mp];
          }
          uint2* s3 = t3 + ((size_t)b * L + l) * n3s;
          for (int D = 0; D < 5; ++D) {
            const int s = 14 - 5 + D;
            const size_t off = (size_t)((1 << D) - 1) * Th;
            for (int tid = 0; tid < Th; ++tid)
              for (int r = 0; r < (1 << D); ++r) {
                const size_t src = (1u << s) + ((size_t)tid << D) + r;
                const size_t dst = (D == 0) ? off + tid : off + 2 * ((size_t)(r >> 1) * Th + tid) + (r & 1);
                s3[dst] = sub[src];
              }
          }
        }
    }
    if (hs) {
      e = cudaMalloc(&c->d_tws, 2 * per_dir * sizeof(uint2));
      if (e == cudaSuccess) e = cudaMemcpy(c->d_tws, hs, 2 * per_dir * sizeof(uint2), cudaMemcpyHostToDevice);
      free(hs);
      if (e == cudaSuccess) {
        d.tws_fwd = c->d_tws;
        d.tw3s_fwd = c->d_tws + (size_t)2 * L * Nh;
        d.tws_inv = c->d_tws + per_dir;
        d.tw3s_inv = d.tws_inv + (size_t)2 * L * Nh;
        d.tw3s_stride = (int)n3s;
      }
    }
  }
  free(h_f); free(h_i); free(h3f); free(h3i);
  if (e != cudaSuccess) {
    cudaFree(c->d_tw_fwd); cudaFree(c->d_tw_inv); cudaFree(c->d_tw3_fwd); cudaFree(c->d_tw3_inv);
    cudaFree(c->d_tws); delete c;
    return pb_set_cuda_error(e);
  }
  d.tw_fwd = c->d_tw_fwd;
  d.tw_inv = c->d_tw_inv;
  d.tw3_fwd = c->d_tw3_fwd;
  d.tw3_inv = c->d_tw3_inv;
  d.tw3_stride = (int)n3;
  *out = c;
  return PB_OK;
}

extern "C" int pb_ctx_destroy(pb_ctx* c) {
  if (!c) return PB_OK;
  cudaFree(c->d_tw_fwd);
  cudaFree(c->d_tw_inv);
  cudaFree(c->d_tw3_fwd);
  cudaFree(c->d_tw3_inv);
  cudaFree(c->d_tws);
  delete c;
  return PB_OK;
}

// ------------------------------------------------------------ NTT kernels --
__device__ __forceinline__ int row_limb_of(const PbDev& P, const int32_t* row_limb, int64_t r) {
  return row_limb ? row_limb[r] : (int)(r % P.L);
}

template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5), NTT_MINB(LOGN)) k_ntt_fwd(PbDev P, uint32_t* rows, int64_t n_rows,
                                                           const int32_t* row_limb) {
  using Nt = pb::Ntt<LOGN>;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  // implicit limbs (r % L): visit rows limb-major so co-resident CTAs share
  // one limb's twiddle tables (L1/L2-hot); measured +13% at N=8192
  const uint32_t per = (row_limb == nullptr && n_rows % P.L == 0 && n_rows < (1ll << 31)) ? (uint32_t)(n_rows / P.L) : 0;
  for (int64_t b = blockIdx.x; b < n_rows; b += gridDim.x) {
    const int64_t r = per ? (int64_t)((uint32_t)b % per) * P.L + (uint32_t)b / per : b;
    const int limb = row_limb_of(P, row_limb, r);
    const uint32_t q = P.q[limb];
    const uint2* tw = P.tw_fwd + (size_t)limb * Nt::N;
    const uint2* t3 = P.tw3_fwd + (size_t)limb * P.tw3_stride;
    uint32_t* row = rows + r * Nt::N;
    uint32_t a[32];
    Nt::gld1(row, a, tid);
    Nt::forward(a, sm, tw, t3, tid, q);
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = pb::canon4(a[c], q);
    Nt::gst3(row, a, tid);
    __syncthreads();
  }
}

template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5), NTT_MINB(LOGN)) k_ntt_inv(PbDev P, uint32_t* rows, int64_t n_rows,
                                                           const int32_t* row_limb) {
  using Nt = pb::Ntt<LOGN>;
  extern __shared__ uint32_t sm[];
  const int tid = threadIdx.x;
  // implicit limbs (r % L): visit rows limb-major so co-resident CTAs share
  // one limb's twiddle tables (L1/L2-hot); measured +13% at N=8192
  const uint32_t per = (row_limb == nullptr && n_rows % P.L == 0 && n_rows < (1ll << 31)) ? (uint32_t)(n_rows / P.L) : 0;
  for (int64_t b = blockIdx.x; b < n_rows; b += gridDim.x) {
    const int64_t r = per ? (int64_t)((uint32_t)b % per) * P.L + (uint32_t)b / per : b;
    const int limb = row_limb_of(P, row_limb, r);
    const uint32_t q = P.q[limb];
    const uint2* tw = P.tw_inv + (size_t)limb * Nt::N;
    const uint2* t3 = P.tw3_inv + (size_t)limb * P.tw3_stride;
    uint32_t* row = rows + r * Nt::N;
    uint32_t a[32];
    Nt::gld3(row, a, tid);
    Nt::inverse_scaled(a, sm, tw, t3, tid, q, P.ninv[limb], P.ninv_sh[limb], P.w0n[limb], P.w0n_sh[limb]);
    Nt::gst1(row, a, tid);
    __syncthreads();
  }
}

// N = 32768 as a CLUSTER of two 512-thread CTAs per row (one CTA of 1024
// threads at 64 registers leaves one CTA per SM whose every barrier stalls the
// whole SM).  The forward's first stage (distance N/2, twiddle psi^brv(1))
// pairs the two halves: each CTA stages its half in shared memory and reads
// the partner's through DSMEM (cluster barrier on both sides); after it the
// halves are independent N/2-point transforms (P.tws_* tables), run as the
// register NTT Ntt<14> by each CTA.  Same arithmetic as K:31-77 (Harvey lazy
// butterflies), bit-identical output in the device order of the full row:
// half b's P3 register v of thread t is uint4 #(v * 1024 + b * 512 + t).
namespace cg = cooperative_groups;

__device__ __forceinline__ int64_t limb_major_row(const PbDev& P, const int32_t* row_limb, int64_t n_rows,
                                                  int64_t b) {
  const uint32_t per = (row_limb == nullptr && n_rows % P.L == 0 && n_rows < (1ll << 31)) ? (uint32_t)(n_rows / P.L) : 0;
  return per ? (int64_t)((uint32_t)b % per) * P.L + (uint32_t)b / per : b;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 2)
    k_ntt_fwd_c2(PbDev P, uint32_t* rows, int64_t n_rows, const int32_t* row_limb) {
  using Nt = pb::Ntt<14>;
  extern __shared__ uint32_t sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int half = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const uint32_t* peer = cl.map_shared_rank(sm, half ^ 1);
  for (int64_t c = blockIdx.x >> 1; c < n_rows; c += gridDim.x >> 1) {
    const int64_t r = limb_major_row(P, row_limb, n_rows, c);
    const int limb = row_limb_of(P, row_limb, r);
    const uint32_t q = P.q[limb], q2 = 2 * q;
    uint32_t* row = rows + r * 32768;
    uint32_t a[32];
    Nt::gld1(row + half * 16384, a, tid);  // natural index half N/2 + tid + 512 c
#pragma unroll
    for (int k = 0; k < 32; ++k) sm[k * 512 + tid] = a[k];
    cl.sync();
    const uint2 w = __ldg(P.tw_fwd + (size_t)limb * 32768 + 1);
#pragma unroll
    for (int k = 0; k < 32; ++k) {  // stage 0: (x, y) -> (x + w y, x - w y), inputs < q
      const uint32_t o = peer[k * 512 + tid];
      const uint32_t tt = mul_shoup_lazy(half ? a[k] : o, w.x, w.y, q);  // [0, 2q)
      a[k] = half ? o - tt + q2 : a[k] + tt;                             // [0, 3q)
    }
    cl.sync();  // the partner has read this CTA's half: shared memory is free
    const size_t sub = (size_t)half * P.L + limb;
    Nt::forward(a, sm, P.tws_fwd + sub * 16384, P.tw3s_fwd + sub * P.tw3s_stride, tid, q);
    uint4* p = reinterpret_cast<uint4*>(row) + half * 512 + tid;
#pragma unroll
    for (int v = 0; v < 8; ++v)
      p[v * 1024] = make_uint4(pb::canon4(a[4 * v], q), pb::canon4(a[4 * v + 1], q), pb::canon4(a[4 * v + 2], q),
                               pb::canon4(a[4 * v + 3], q));
    __syncthreads();
  }
}

// The inverse in reverse: the two half transforms (GS, unscaled), then the
// cross-half stage with N^-1 folded in: x' = (x + y) N^-1, y' = (x - y) w N^-1.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 2)
    k_ntt_inv_c2(PbDev P, uint32_t* rows, int64_t n_rows, const int32_t* row_limb) {
  using Nt = pb::Ntt<14>;
  extern __shared__ uint32_t sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int half = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const uint32_t* peer = cl.map_shared_rank(sm, half ^ 1);
  for (int64_t c = blockIdx.x >> 1; c < n_rows; c += gridDim.x >> 1) {
    const int64_t r = limb_major_row(P, row_limb, n_rows, c);
    const int limb = row_limb_of(P, row_limb, r);
    const uint32_t q = P.q[limb], q2 = 2 * q;
    uint32_t* row = rows + r * 32768;
    uint32_t a[32];
    const uint4* p = reinterpret_cast<const uint4*>(row) + half * 512 + tid;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const uint4 x = __ldg(p + v * 1024);
      a[4 * v] = x.x; a[4 * v + 1] = x.y; a[4 * v + 2] = x.z; a[4 * v + 3] = x.w;
    }
    const size_t sub = (size_t)half * P.L + limb;
    Nt::inverse(a, sm, P.tws_inv + sub * 16384, P.tw3s_inv + sub * P.tw3s_stride, tid, q);  // [0, 2q), P1 layout
    __syncthreads();  // every thread is past the inverse's last shared-memory read
#pragma unroll
    for (int k = 0; k < 32; ++k) sm[k * 512 + tid] = a[k];
    cl.sync();
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const uint32_t o = peer[k * 512 + tid];
      a[k] = half ? mul_shoup(o - a[k] + q2, P.w0n[limb], P.w0n_sh[limb], q)
                  : mul_shoup(a[k] + o, P.ninv[limb], P.ninv_sh[limb], q);
    }
    cl.sync();
    Nt::gst1(row + half * 16384, a, tid);
  }
}

// Small-N path (N <= 1024): one CTA per row, one radix-2 stage per barrier,
// fully reduced arithmetic.  Used for tests / tiny parameter sets.
__global__ void k_ntt_small(PbDev P, uint32_t* rows, int64_t n_rows, const int32_t* row_limb, int inverse) {
  extern __shared__ uint32_t sm[];
  const int N = P.N, logN = P.logN;
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    const int limb = row_limb_of(P, row_limb, r);
    const uint32_t q = P.q[limb];
    const uint2* tw = (inverse ? P.tw_inv : P.tw_fwd) + (size_t)limb * N;
    uint32_t* row = rows + r * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) sm[j] = row[j];
    __syncthreads();
    for (int st = 0; st < logN; ++st) {
      const int s = inverse ? (logN - 1 - st) : st;
      const int t = N >> (s + 1);
      for (int b = threadIdx.x; b < N / 2; b += blockDim.x) {
        const int g = b / t, j = 2 * g * t + (b % t);
        const uint2 w = tw[(1 << s) + g];
        const uint32_t x = sm[j], y = sm[j + t];
        if (!inverse) {
          const uint32_t v = mul_shoup(y, w.x, w.y, q);
          sm[j] = addmod(x, v, q);
          sm[j + t] = submod(x, v, q);
        } else {
          sm[j] = addmod(x, y, q);
          sm[j + t] = mul_shoup(submod(x, y, q), w.x, w.y, q);
        }
      }
      __syncthreads();
    }
    for (int j = threadIdx.x; j < N; j += blockDim.x)
      row[j] = inverse ? mul_shoup(sm[j], P.ninv[limb], P.ninv_sh[limb], q) : sm[j];
    __syncthreads();
  }
}

template <int LOGN>
static void launch_ntt(const PbDev& P, uint32_t* rows, int64_t n_rows, const int32_t* row_limb,
                       cudaStream_t st, bool inverse) {
  if (LOGN == 15 && P.tws_fwd) {  // two-CTA cluster per row
    const size_t smem = pb::Ntt<14>::SMEM_WORDS * 4;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_ntt_fwd_c2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(k_ntt_inv_c2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    const int64_t clusters = n_rows < 148 * 64 ? n_rows : 148 * 64;
    if (inverse) k_ntt_inv_c2<<<(unsigned)(2 * clusters), 512, smem, st>>>(P, rows, n_rows, row_limb);
    else k_ntt_fwd_c2<<<(unsigned)(2 * clusters), 512, smem, st>>>(P, rows, n_rows, row_limb);
    return;
  }
  using Nt = pb::Ntt<LOGN>;
  const size_t smem = Nt::SMEM_WORDS * sizeof(uint32_t);
  const int grid = (int)(n_rows < (1 << 30) ? n_rows : (1 << 30));
  if (inverse) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_ntt_inv<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_ntt_inv<LOGN><<<grid, Nt::T, smem, st>>>(P, rows, n_rows, row_limb);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_ntt_fwd<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_ntt_fwd<LOGN><<<grid, Nt::T, smem, st>>>(P, rows, n_rows, row_limb);
  }
}

static int ntt_entry(const pb_ctx* ctx, uint32_t* rows, int64_t n_rows, const int32_t* row_limb,
                     void* stream, bool inverse) {
  if (!ctx || (!rows && n_rows)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (n_rows <= 0) return PB_OK;
  const PbDev& P = ctx->dev;
  cudaStream_t st = pb_stream_of(stream);
  if (P.logN >= 11) {
    PB_DISPATCH_LOGN(P.logN, launch_ntt, P, rows, n_rows, row_limb, st, inverse);
  } else {
    const int grid = (int)(n_rows < (1 << 30) ? n_rows : (1 << 30));
    const int thr = P.N / 2 < 32 ? 32 : (P.N / 2 > 512 ? 512 : P.N / 2);
    k_ntt_small<<<grid, thr, P.N * sizeof(uint32_t), st>>>(P, rows, n_rows, row_limb, inverse ? 1 : 0);
  }
  PB_CHECK_LAUNCH();
  return PB_OK;
}

extern "C" int pb_ntt_forward(const pb_ctx* ctx, uint32_t* rows, int64_t n_rows, const int32_t* row_limb,
                              void* stream) {
  return ntt_entry(ctx, rows, n_rows, row_limb, stream, false);
}
extern "C" int pb_ntt_inverse(const pb_ctx* ctx, uint32_t* rows, int64_t n_rows, const int32_t* row_limb,
                              void* stream) {
  return ntt_entry(ctx, rows, n_rows, row_limb, stream, true);
}

// ----------------------------------------------- NTT-domain order convert --
// Device order (pb_ntt.cuh dev_addr) <-> the reference's bit-reversed order.
__global__ void k_reorder(int N, int logN, uint32_t* rows, int64_t n_rows, int to_device) {
  extern __shared__ uint32_t sm[];
  const int T = N >> 5;
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x) {
    uint32_t* row = rows + r * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) sm[i] = row[i];
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      if (to_device) {  // address i holds K index j
        const int v = i / (4 * T), rem = i - v * 4 * T;
        row[i] = sm[(rem >> 2) * 32 + 4 * v + (rem & 3)];
      } else {  // K index i lives at device address dev_addr(i)
        row[i] = sm[((i & 31) >> 2) * 4 * T + (i >> 5) * 4 + (i & 3)];
      }
    }
    __syncthreads();
  }
}

extern "C" int pb_ntt_reorder(const pb_ctx* ctx, uint32_t* rows, int64_t n_rows, int to_device, void* stream) {
  if (!ctx || (!rows && n_rows)) return pb_set_error(PB_ERR_ARG, "null argument");
  if (n_rows <= 0 || ctx->dev.logN < 11) return PB_OK;  // small N: device order == reference order
  const int N = ctx->dev.N;
  const size_t smem = (size_t)N * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_reorder, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = (int)(n_rows < (1 << 30) ? n_rows : (1 << 30));
  k_reorder<<<grid, 512, smem, pb_stream_of(stream)>>>(N, ctx->dev.logN, rows, n_rows, to_device ? 1 : 0);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

// -------------------------------------------------------------- pointwise --
// Semantics follow K:80-113 exactly, including uint64 wraparound of
// (a + q - b) in pw_sub for non-canonical inputs.
__global__ void k_pw(PbDev P, int op, uint32_t* out, const uint32_t* a, const uint32_t* b, int64_t n_rows,
                     int64_t b_rows, const int32_t* row_limb) {
  const int N = P.N;
  const int64_t total = n_rows * (int64_t)N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / N;
    const int j = (int)(e - r * N);
    const int limb = row_limb_of(P, row_limb, r);
    const uint32_t q = P.q[limb];
    const uint64_t mu = P.mu[limb];
    const uint64_t av = a[e];
    const uint64_t bv = b[(r % b_rows) * N + j];
    uint32_t res;
    switch (op) {
      case PB_PW_MUL: res = reduce64(av * bv, q, mu); break;
      case PB_PW_MAC: {
        const uint64_t prod = reduce64(av * bv, q, mu);
        res = reduce64((uint64_t)out[e] + prod, q, mu);
        break;
      }
      case PB_PW_ADD: res = reduce64(av + bv, q, mu); break;
      default: res = reduce64(av + q - bv, q, mu); break;
    }
    out[e] = res;
  }
}

extern "C" int pb_pw(const pb_ctx* ctx, int op, uint32_t* out, const uint32_t* a, const uint32_t* b,
                     int64_t n_rows, int64_t b_rows, const int32_t* row_limb, void* stream) {
  if (!ctx || !out || !a || !b) return pb_set_error(PB_ERR_ARG, "null argument");
  if (op < 0 || op > 3) return pb_set_error(PB_ERR_ARG, "bad pointwise op");
  if (n_rows <= 0) return PB_OK;
  if (b_rows <= 0) return pb_set_error(PB_ERR_SHAPE, "b_rows must be positive");
  const int64_t total = n_rows * (int64_t)ctx->dev.N;
  k_pw<<<pb_grid_1d(total, 256), 256, 0, pb_stream_of(stream)>>>(ctx->dev, op, out, a, b, n_rows, b_rows, row_limb);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

// ----------------------------------------------------------------- decode --
// K:158-179 garner_digits for one coefficient: x[i] at stride `xs`.
__device__ __forceinline__ void garner(const PbDev& P, const uint32_t* x, int64_t xs, uint32_t (&d)[PB_MAXL]) {
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

// K:182-199 scale_round_digits for one coefficient (float64, same order, no FMA).
__device__ __forceinline__ uint64_t scale_round(const PbDev& P, const uint32_t (&d)[PB_MAXL]) {
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

__global__ void k_garner(PbDev P, const uint32_t* rows, int64_t n_polys, uint32_t* digits) {
  const int N = P.N, L = P.L;
  const int64_t total = n_polys * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / N;
    const int j = (int)(e - p * N);
    uint32_t d[PB_MAXL];
    garner(P, rows + p * L * N + j, N, d);
    for (int i = 0; i < L; ++i) digits[p * L * N + (int64_t)i * N + j] = d[i];
  }
}

__global__ void k_scale_round(PbDev P, const uint32_t* digits, int64_t n_polys, uint64_t* out) {
  const int N = P.N, L = P.L;
  const int64_t total = n_polys * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / N;
    const int j = (int)(e - p * N);
    uint32_t d[PB_MAXL];
#pragma unroll
    for (int i = 0; i < PB_MAXL; ++i) d[i] = (i < L) ? digits[p * L * N + (int64_t)i * N + j] : 0u;
    out[e] = scale_round(P, d);
  }
}

__global__ void k_decode(PbDev P, const uint32_t* rows, int64_t n_polys, uint64_t* out) {
  const int N = P.N, L = P.L;
  const int64_t total = n_polys * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / N;
    const int j = (int)(e - p * N);
    uint32_t d[PB_MAXL];
    garner(P, rows + p * L * N + j, N, d);
    out[e] = scale_round(P, d);
  }
}

extern "C" int pb_garner_digits(const pb_ctx* ctx, const uint32_t* rows, int64_t n_polys, uint32_t* digits,
                                void* stream) {
  if (!ctx || !rows || !digits) return pb_set_error(PB_ERR_ARG, "null argument");
  if (n_polys <= 0) return PB_OK;
  k_garner<<<pb_grid_1d(n_polys * ctx->dev.N, 256), 256, 0, pb_stream_of(stream)>>>(ctx->dev, rows, n_polys, digits);
  PB_CHECK_LAUNCH();
  return PB_OK;
}
extern "C" int pb_scale_round_digits(const pb_ctx* ctx, const uint32_t* digits, int64_t n_polys, uint64_t* out,
                                     void* stream) {
  if (!ctx || !digits || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (n_polys <= 0) return PB_OK;
  k_scale_round<<<pb_grid_1d(n_polys * ctx->dev.N, 256), 256, 0, pb_stream_of(stream)>>>(ctx->dev, digits, n_polys, out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}
extern "C" int pb_decode(const pb_ctx* ctx, const uint32_t* rows, int64_t n_polys, uint64_t* out, void* stream) {
  if (!ctx || !rows || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (n_polys <= 0) return PB_OK;
  k_decode<<<pb_grid_1d(n_polys * ctx->dev.N, 256), 256, 0, pb_stream_of(stream)>>>(ctx->dev, rows, n_polys, out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

// ------------------------------------------------ negacyclic mod 2^64 (K:135)
__global__ void k_negacyclic_wrap(const uint64_t* a, const uint64_t* b, int64_t n_pairs, int N, uint64_t* out) {
  const int64_t total = n_pairs * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / N;
    const int k = (int)(e - p * N);
    const uint64_t* ap = a + p * N;
    const uint64_t* bp = b + p * N;
    uint64_t acc = 0;
    for (int i = 0; i <= k; ++i) acc += ap[i] * bp[k - i];
    for (int i = k + 1; i < N; ++i) acc -= ap[i] * bp[k + N - i];
    out[e] = acc;
  }
}

extern "C" int pb_negacyclic_mul_wrap(const uint64_t* a, const uint64_t* b, int64_t n_pairs, int32_t N,
                                      uint64_t* out, void* stream) {
  if (!a || !b || !out) return pb_set_error(PB_ERR_ARG, "null argument");
  if (n_pairs <= 0 || N <= 0) return PB_OK;
  k_negacyclic_wrap<<<pb_grid_1d(n_pairs * N, 128), 128, 0, pb_stream_of(stream)>>>(a, b, n_pairs, N, out);
  PB_CHECK_LAUNCH();
  return PB_OK;
}

// ------------------------------------------------------------- launch cap ---
static thread_local int32_t g_launch_cap = 0;

int64_t pb_row_grid(int64_t rows) { return g_launch_cap > 0 && rows > g_launch_cap ? g_launch_cap : rows; }

extern "C" int pb_set_launch_cap(int32_t max_ctas) {
  if (max_ctas < 0) return pb_set_error(PB_ERR_ARG, "launch cap must be >= 0");
  g_launch_cap = max_ctas;
  return PB_OK;
}
