// pb_imma.cu — the Z_{2^64} ring GEMMs / conv operators (K:206-278 and the
// local terms of the conv protocols) on the int8 TENSOR CORES.
//
// A u64 operand < 2^59 is written in balanced base-256 digits
// a = sum_{i<8} a_i 256^i, a_i in [-128, 127], so
//   a * b mod 2^64 = sum_{s<8} 256^s * C_s,   C_s = sum_{i+j=s} a_i b_j
// (digit pairs with i+j >= 8 vanish mod 2^64).  Each C_s is ONE int8 x int8
// -> int32 GEMM over a concatenated contraction: with A's digit planes stored
// [row][a_0 .. a_7][K] and B's [col][b_7 .. b_0][K], the operands of C_s are
// the first (s+1)K entries of each A row and the last (s+1)K of each B row --
// strided views, no copies.  |C_s| <= 8 K 2^14 < 2^31 for K <= 8192, so
// longer contractions are split into chunks whose results are combined in
// u64.  The int8 GEMMs are plain library GEMMs (cuBLASLt IMMA on the
// tcgen05 tensor cores); the digit gathers (with the conv pad / stride /
// dilation index maps applied on the fly) and the shift-and-add combine are
// this file's kernels.
#include <cublasLt.h>

#include <map>
#include <mutex>
#include <tuple>

#include "pb_common.cuh"

namespace {

struct ImmaDims {  // generic GEMM out(n x m) = sum_k A(n,k) B(k,m) with conv / matmul gathers
  int kind;        // 0..2 PB_CONV_*, 3 matmul
  int B, ci, co, H, W, s, p, st, oh, ow;  // conv
  int n, k, m, ta, tb;                    // matmul
};

__device__ __forceinline__ uint64_t imma_a(const ImmaDims& d, const uint64_t* A, int row, int kk) {
  const int SS = d.s * d.s;
  switch (d.kind) {
    case PB_CONV_FWD: return __ldg(A + (size_t)row * (d.ci * SS) + kk);  // W[o][(c,i,j)]
    case PB_CONV_BWDX: {                                                 // W[o][c][i][j], row = c, kk = (o,i,j)
      const int o = kk / SS, r = kk - o * SS;
      return __ldg(A + (size_t)(o * d.ci + row) * SS + r);
    }
    case PB_CONV_GRADW: {  // dY[b][o][y][x], row = o, kk = (b,y,x)
      const unsigned hw = (unsigned)(d.oh * d.ow), b = (unsigned)kk / hw, r = (unsigned)kk - b * hw;
      return __ldg(A + (size_t)(b * d.co + row) * hw + r);
    }
    default: return __ldg(A + (d.ta ? (size_t)kk * d.n + row : (size_t)row * d.k + kk));
  }
}

__device__ __forceinline__ uint64_t imma_b(const ImmaDims& d, const uint64_t* Bm, int kk, int col) {
  const int SS = d.s * d.s;
  switch (d.kind) {
    case PB_CONV_FWD:
    case PB_CONV_GRADW: {
      const int kc = d.kind == PB_CONV_FWD ? kk : col;             // (c,i,j)
      const unsigned kp = (unsigned)(d.kind == PB_CONV_FWD ? col : kk);  // (b,y,x)
      const int c = kc / SS, r = kc - c * SS, i = r / d.s, j = r - i * d.s;
      const unsigned hw = (unsigned)(d.oh * d.ow), ow = (unsigned)d.ow;
      const unsigned b = kp / hw, q = kp - b * hw, y = q / ow, x = q - y * ow;
      const int yy = (int)y * d.st + i - d.p, xx = (int)x * d.st + j - d.p;
      if (yy < 0 || yy >= d.H || xx < 0 || xx >= d.W) return 0ull;
      return __ldg(Bm + ((size_t)(b * d.ci + c) * d.H + yy) * d.W + xx);
    }
    case PB_CONV_BWDX: {  // kk = (o,i,j), col = (b,y,x) of dX
      const int o = kk / SS, r = kk - o * SS, i = r / d.s, j = r - i * d.s;
      const unsigned hw = (unsigned)(d.H * d.W), Wd = (unsigned)d.W;
      const unsigned b = (unsigned)col / hw, q = (unsigned)col - b * hw, y = q / Wd, x = q - y * Wd;
      const int u = (int)y + d.p - i, v = (int)x + d.p - j;
      if (u < 0 || v < 0) return 0ull;
      const unsigned yy = (unsigned)u / (unsigned)d.st, xx = (unsigned)v / (unsigned)d.st;
      if (yy * d.st != (unsigned)u || xx * d.st != (unsigned)v || yy >= (unsigned)d.oh || xx >= (unsigned)d.ow)
        return 0ull;
      return __ldg(Bm + ((size_t)(b * d.co + o) * d.oh + yy) * d.ow + xx);
    }
    default: return __ldg(Bm + (d.tb ? (size_t)col * d.k + kk : (size_t)kk * d.m + col));
  }
}

__device__ __forceinline__ size_t imma_out(const ImmaDims& d, int row, int col) {
  switch (d.kind) {
    case PB_CONV_FWD: {
      const unsigned hw = (unsigned)(d.oh * d.ow), b = (unsigned)col / hw, q = (unsigned)col - b * hw;
      return (size_t)(b * d.co + row) * hw + q;
    }
    case PB_CONV_BWDX: {
      const unsigned hw = (unsigned)(d.H * d.W), b = (unsigned)col / hw, q = (unsigned)col - b * hw;
      return (size_t)(b * d.ci + row) * hw + q;
    }
    case PB_CONV_GRADW: return (size_t)row * (d.ci * d.s * d.s) + col;
    default: return (size_t)row * d.m + col;
  }
}

// balanced base-256 digits of v (< 2^59 after masking): v = sum d_i 256^i
__device__ __forceinline__ void digits8(uint64_t v, int8_t (&d)[8]) {
  int carry = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int x = (int)((v >> (8 * i)) & 0xFFu) + carry;
    carry = x >= 128;
    d[i] = (int8_t)(x - (carry << 8));
  }
}

// Digit planes, 4 consecutive contraction entries per thread (one 32-bit store
// per plane): A planes [n][8][Kp] with digit i at plane i; B planes,
// transposed, [m][8][Kp] with digit i at plane 7 - i.  Kp % 16 == 0.
template <bool IS_A>
__global__ void k_imma_digits(ImmaDims d, const uint64_t* src, int rows, int k0, int kc, int Kp, uint64_t mask,
                              int8_t* out) {
  const int q4 = Kp / 4;
  const int64_t total = (int64_t)rows * q4;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(e / q4), kk = 4 * (int)(e - (int64_t)row * q4);
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int k = kk + t;
      uint64_t v = 0;
      if (k < kc) v = (IS_A ? imma_a(d, src, row, k0 + k) : imma_b(d, src, k0 + k, row)) & mask;
      int8_t g[8];
      digits8(v, g);
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] |= (uint32_t)(uint8_t)g[i] << (8 * t);
    }
    uint32_t* o = reinterpret_cast<uint32_t*>(out + (size_t)row * 8 * Kp + kk);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[(size_t)(IS_A ? i : 7 - i) * (Kp / 4)] = w[i];
  }
}

// out[out_at(row, col)] (+)= sum_s 256^s C_s[row][col]  (C_s row-major n x m, int32)
__global__ void k_imma_combine(ImmaDims d, const int32_t* C, int n, int m, int accumulate, uint64_t mask,
                               uint64_t* out) {
  const int64_t nm = (int64_t)n * m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nm; e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t acc = 0;
#pragma unroll
    for (int s = 0; s < 8; ++s) acc += (uint64_t)(int64_t)C[(size_t)s * nm + e] << (8 * s);
    const int row = (int)(e / m), col = (int)(e - (int64_t)row * m);
    const size_t o = imma_out(d, row, col);
    out[o] = ((accumulate ? out[o] : 0ull) + acc) & mask;
  }
}

struct LtState {
  cublasLtHandle_t h = nullptr;
  size_t ws_bytes = 32u << 20;  // per-call, stream-ordered workspace (concurrent streams never share one)
  bool ok = false;
};

LtState& lt() {
  static LtState s;
  static std::once_flag once;
  std::call_once(once, [] {
    s.ok = cublasLtCreate(&s.h) == CUBLAS_STATUS_SUCCESS;
    // keep stream-ordered allocations (digit planes, partial products, workspace) cached
    // in the device's default pool instead of returning them to the driver at every sync
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  return s;
}

// C (cm x cn, column-major, int32) = A_op^T B_op: A_op = rows of `a` (K int8 each, stride lda),
// B_op = rows of `b` (K each, stride ldb).  Descriptors + the heuristic's algorithm are cached
// per shape (the heuristic query costs far more than a small GEMM).  Returns 0 on success.
constexpr int LT_CANDIDATES = 12;
struct LtPlan {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatmulAlgo_t algo;
  cublasLtMatmulAlgo_t cand[LT_CANDIDATES];
  int ncand = 0;
  bool ok = false, tuned = false;
};

LtPlan& lt_plan(int cm, int lda, int cn, int ldb, int K) {
  static std::map<std::tuple<int, int, int, int, int>, LtPlan> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  auto key = std::make_tuple(cm, lda, cn, ldb, K);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  LtPlan& P = cache[key];
  LtState& L = lt();
  const cublasOperation_t tA = CUBLAS_OP_T, tB = CUBLAS_OP_N;
  cublasLtMatmulPreference_t pref = nullptr;
  cublasLtMatmulHeuristicResult_t heur[LT_CANDIDATES] = {};
  int found = 0;
  if (cublasLtMatmulDescCreate(&P.op, CUBLAS_COMPUTE_32I, CUDA_R_32I) != CUBLAS_STATUS_SUCCESS) return P;
  cublasLtMatmulDescSetAttribute(P.op, CUBLASLT_MATMUL_DESC_TRANSA, &tA, sizeof(tA));
  cublasLtMatmulDescSetAttribute(P.op, CUBLASLT_MATMUL_DESC_TRANSB, &tB, sizeof(tB));
  if (cublasLtMatrixLayoutCreate(&P.la, CUDA_R_8I, K, cm, lda) != CUBLAS_STATUS_SUCCESS) return P;
  if (cublasLtMatrixLayoutCreate(&P.lb, CUDA_R_8I, K, cn, ldb) != CUBLAS_STATUS_SUCCESS) return P;
  if (cublasLtMatrixLayoutCreate(&P.lc, CUDA_R_32I, cm, cn, cm) != CUBLAS_STATUS_SUCCESS) return P;
  if (cublasLtMatmulPreferenceCreate(&pref) != CUBLAS_STATUS_SUCCESS) return P;
  cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &L.ws_bytes,
                                       sizeof(L.ws_bytes));
  if (cublasLtMatmulAlgoGetHeuristic(L.h, P.op, P.la, P.lb, P.lc, P.lc, pref, LT_CANDIDATES, heur, &found) ==
          CUBLAS_STATUS_SUCCESS &&
      found > 0) {
    P.algo = heur[0].algo;
    for (int i = 0; i < found; ++i)
      if (heur[i].state == CUBLAS_STATUS_SUCCESS) P.cand[P.ncand++] = heur[i].algo;
    P.ok = true;
  }
  cublasLtMatmulPreferenceDestroy(pref);
  return P;
}

int lt_gemm_tn(const int8_t* a, int cm, int lda, const int8_t* b, int cn, int ldb, int K, int32_t* c, void* ws,
               cudaStream_t st) {
  LtState& L = lt();
  if (!L.ok) return -1;
  LtPlan& P = lt_plan(cm, lda, cn, ldb, K);
  if (!P.ok) return -1;
  const int32_t alpha = 1, beta = 0;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (!P.tuned && P.ncand > 1 && cudaStreamIsCapturing(st, &cap) == cudaSuccess &&
      cap == cudaStreamCaptureStatusNone) {
    // first eager use of this shape: time the heuristic's candidates on the real
    // operands and keep the fastest (its first pick is often a 256x256-tile kernel
    // that leaves most of a 64-row GEMM idle); graph capture reuses the choice
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int i = 0; i < P.ncand; ++i) {
      float ms = 0.f, tot = 0.f;
      bool good = true;
      for (int r = 0; r < 3 && good; ++r) {
        cudaEventRecord(e0, st);
        good = cublasLtMatmul(L.h, P.op, &alpha, a, P.la, b, P.lb, &beta, c, P.lc, c, P.lc, &P.cand[i], ws, L.ws_bytes,
                              st) == CUBLAS_STATUS_SUCCESS;
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0) tot += ms;  // the first run warms up
      }
      if (good && tot < best) best = tot, P.algo = P.cand[i];
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    P.tuned = true;
  }
  return cublasLtMatmul(L.h, P.op, &alpha, a, P.la, b, P.lb, &beta, c, P.lc, c, P.lc, &P.algo, ws, L.ws_bytes, st) ==
                 CUBLAS_STATUS_SUCCESS
             ? 0
             : -1;
}

}  // namespace

// Ring GEMM out (n x m) of a conv / matmul operator on the int8 tensor cores.
// Returns PB_OK, or a nonzero status when the tensor-core path is unavailable
// (the caller then uses the CUDA-core kernel).
static int pb_imma_ring_gemm(const ImmaDims& d, const uint64_t* A, const uint64_t* Bm, int n, int K, int m, int ell,
                      uint64_t* out, cudaStream_t st) {
  if (!lt().ok) return PB_ERR_CUDA;
  const uint64_t mask = ell >= 64 ? ~0ull : ((1ull << ell) - 1);
  const int KC = 8192;  // contraction chunk: |C_s| <= 8 * KC * 2^14 = 2^30
  const int nchunks = (K + KC - 1) / KC;
  const int kc_max = K < KC ? K : KC;
  const int Kp = (kc_max + 15) / 16 * 16;
  int8_t *da = nullptr, *db = nullptr;
  int32_t* dc = nullptr;
  void* ws = nullptr;
  const size_t a_bytes = (size_t)n * 8 * Kp, b_bytes = (size_t)m * 8 * Kp, c_bytes = (size_t)8 * n * m * 4;
  if (cudaMallocAsync((void**)&da, a_bytes, st) != cudaSuccess) return PB_ERR_CUDA;
  if (cudaMallocAsync((void**)&db, b_bytes, st) != cudaSuccess) return PB_ERR_CUDA;
  if (cudaMallocAsync((void**)&dc, c_bytes, st) != cudaSuccess) return PB_ERR_CUDA;
  if (cudaMallocAsync(&ws, lt().ws_bytes, st) != cudaSuccess) return PB_ERR_CUDA;
  int rc = PB_OK;
  for (int ch = 0; ch < nchunks && rc == PB_OK; ++ch) {
    const int k0 = ch * KC, kc = (K - k0) < KC ? (K - k0) : KC;
    k_imma_digits<true><<<pb_grid_1d((int64_t)n * Kp / 4, 256), 256, 0, st>>>(d, A, n, k0, kc, Kp, mask, da);
    k_imma_digits<false><<<pb_grid_1d((int64_t)m * Kp / 4, 256), 256, 0, st>>>(d, Bm, m, k0, kc, Kp, mask, db);
    for (int s = 0; s < 8 && rc == PB_OK; ++s) {
      // C_s (m x n col-major == n x m row-major) = B_blk^T A_blk over (s+1) Kp
      const int8_t* bb = db + (size_t)(7 - s) * Kp;  // planes b_s .. b_0
      if (lt_gemm_tn(bb, m, 8 * Kp, da, n, 8 * Kp, (s + 1) * Kp, dc + (size_t)s * n * m, ws, st) != 0)
        rc = PB_ERR_CUDA;
    }
    if (rc == PB_OK)
      k_imma_combine<<<pb_grid_1d((int64_t)n * m, 256), 256, 0, st>>>(d, dc, n, m, ch > 0, mask, out);
  }
  cudaFreeAsync(ws, st);
  cudaFreeAsync(dc, st);
  cudaFreeAsync(db, st);
  cudaFreeAsync(da, st);
  return rc;
}

int pb_imma_conv(int kind, const uint64_t* a, const uint64_t* b, int B, int ci, int co, int H, int W, int s, int p,
                 int st_, int oh, int ow, int ell, uint64_t* out, cudaStream_t st) {
  ImmaDims d = {};
  d.kind = kind, d.B = B, d.ci = ci, d.co = co, d.H = H, d.W = W, d.s = s, d.p = p, d.st = st_, d.oh = oh, d.ow = ow;
  int n, K, m;
  const uint64_t *A, *Bm;
  if (kind == PB_CONV_FWD) { n = co; K = ci * s * s; m = B * oh * ow; A = b; Bm = a; }         // A = W, B = X
  else if (kind == PB_CONV_BWDX) { n = ci; K = co * s * s; m = B * H * W; A = b; Bm = a; }     // A = W, B = dY
  else { n = co; K = B * oh * ow; m = ci * s * s; A = b; Bm = a; }                             // A = dY, B = X
  return pb_imma_ring_gemm(d, A, Bm, n, K, m, ell, out, st);
}

int pb_imma_matmul(const uint64_t* a, const uint64_t* b, int n, int k, int m, int ta, int tb, int ell, uint64_t* out,
                   cudaStream_t st) {
  ImmaDims d = {};
  d.kind = 3, d.n = n, d.k = k, d.m = m, d.ta = ta, d.tb = tb;
  return pb_imma_ring_gemm(d, a, b, n, k, m, ell, out, st);
}
