/*
 * pencil_b200.h — C ABI of the B200-native Pencil HE linear-layer engine.
 *
 * Drop-in boundary for the hot path named in BASELINE.json.north_star:
 * encrypt -> ciphertext x plaintext multiply-accumulate in the NTT domain ->
 * masking -> decrypt-to-additive-share, plus share arithmetic mod 2^ell.
 *
 * Conventions
 *  - Every pointer argument is a DEVICE pointer (cudaMalloc'd or a torch CUDA
 *    tensor's data_ptr()) unless the name says `host`.  `stream` is a
 *    cudaStream_t (NULL = legacy default stream).  Calls are asynchronous on
 *    `stream`; no call synchronises except pb_ctx_create/destroy.
 *  - RNS residues are uint32 (moduli q_i < 2^30), polynomials are rows of N
 *    residues, a polynomial over all limbs is [L][N], a ciphertext [2][L][N]
 *    (c0 then c1), always in NTT form unless a function says "coefficient".
 *  - Z_{2^ell} elements (shares, plaintext coefficients) are uint64 holding a
 *    canonical value < 2^ell.
 *  - Every function returns an int status (PB_OK = 0); nothing throws across
 *    the ABI.  pb_last_error() returns a thread-local message.  Status codes
 *    map 1:1 to the reference exception taxonomy
 *    (/root/reference/pkg/src/pencil/errors.py:4-41).
 *
 * Each entry point cites the reference interface it replaces.  "K" is
 * /root/reference/pkg/src/pencil/_kernels.py, "R" is .../pencil/ring.py,
 * "SPEC" is /root/reference/SPEC.md (the SPEC-only modules the reference
 * specifies but does not ship).
 */
#ifndef PENCIL_B200_H_
#define PENCIL_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 2: round 2 -- pb_encrypt_sk takes the key's Shoup row, pb_host_softmax_post a
 * denominator; new pb_mask_mac, pb_nl_op / pb_nl_words, pb_scatter_u64,
 * pb_prep_scalars, pb_shoup_rows, pb_host_publish, pb_ring_chansum, pb_*_ex backends. */
#define PB_ABI_VERSION 2
#define PB_MAX_LIMBS 8

/* status codes -> errors.py classes (E:4-41) */
enum {
  PB_OK = 0,
  PB_ERR_PARAMS = 1,   /* ParamsError    E:8   */
  PB_ERR_RANGE = 2,    /* EncodeRangeError E:12 */
  PB_ERR_SCALE = 3,    /* ScaleError     E:16  */
  PB_ERR_SHAPE = 4,    /* ShapeError     E:20  */
  PB_ERR_FORM = 5,     /* FormError      E:24  */
  PB_ERR_GEOMETRY = 6, /* GeometryError  E:28  */
  PB_ERR_CUDA = 7,     /* PencilError (device failure) */
  PB_ERR_ARG = 8       /* PencilError (bad argument)   */
};

/* Parameter descriptor (SPEC:103-106 BfvParams).  All big-integer constants
 * are precomputed by the host (Python ints) and passed as words. */
typedef struct pb_params {
  int32_t N;   /* power of two, 16..32768 */
  int32_t L;   /* number of RNS limbs, 1..PB_MAX_LIMBS */
  int32_t ell; /* plaintext modulus t = 2^ell, 2..62 */
  int32_t reserved;
  uint32_t q[PB_MAX_LIMBS];                 /* primes, q = 1 mod 2N, q < 2^30 */
  uint32_t psi[PB_MAX_LIMBS];               /* primitive 2N-th roots of unity */
  uint32_t delta_mod_q[PB_MAX_LIMBS];       /* floor(Q/t) mod q_i            */
  uint32_t garner_prefix_inv[PB_MAX_LIMBS]; /* (q_0..q_{i-1})^-1 mod q_i  K:158 */
  uint64_t scale_int[PB_MAX_LIMBS];         /* floor(t*P_{i-1}/Q) mod 2^64 K:182 */
  double scale_frac[PB_MAX_LIMBS];          /* frac(t*P_{i-1}/Q)          K:182 */
} pb_params;

typedef struct pb_ctx pb_ctx; /* immutable, shareable across streams */

int pb_abi_version(void);
const char* pb_last_error(void);
int pb_device_sm_count(int* out_host);

/* Builds twiddle tables (Shoup form) on the device.  Replaces the host-side
 * table construction the K callers perform (K:22-29). */
int pb_ctx_create(const pb_params* params_host, pb_ctx** out_host);
int pb_ctx_destroy(pb_ctx* ctx);

/* ------------------------------------------------ polynomial engine (K) --- */
/* Row r of `rows` uses limb row_limb[r] (or r % L when row_limb == NULL). */

/* NTT-domain rows are kept in DEVICE ORDER: bit-reversed index j = 32*t + 4*v + k
 * (t < N/32, v < 8, k < 4) lives at address v*(N/8) + 4*t + k, which lets the
 * register-blocked NTT move whole rows with coalesced 128-bit accesses.  All
 * NTT-domain operands (ciphertexts, plaintexts, keys) share this order, so
 * pointwise products are unaffected.  N < 2048 uses the reference order. */

/* K:31-50 ntt_forward: in place, natural -> bit-reversed (device order). */
int pb_ntt_forward(const pb_ctx* ctx, uint32_t* rows, int64_t n_rows, const int32_t* row_limb,
                   void* stream);
/* K:53-77 ntt_inverse: in place, bit-reversed -> natural, includes x N^-1. */
int pb_ntt_inverse(const pb_ctx* ctx, uint32_t* rows, int64_t n_rows, const int32_t* row_limb,
                   void* stream);

/* Convert NTT-domain rows between device order (to_device=1 from reference
 * bit-reversed order, to_device=0 back).  K-compat callers use this to see
 * exactly K's output order. */
int pb_ntt_reorder(const pb_ctx* ctx, uint32_t* rows, int64_t n_rows, int to_device, void* stream);

/* K:80-113 pointwise ops.  op: 0 pw_mul, 1 pw_mul_acc (out += a*b), 2 pw_add,
 * 3 pw_sub.  Row r of b is b[r % b_rows] (b_rows == n_rows: plain). */
enum { PB_PW_MUL = 0, PB_PW_MAC = 1, PB_PW_ADD = 2, PB_PW_SUB = 3 };
int pb_pw(const pb_ctx* ctx, int op, uint32_t* out, const uint32_t* a, const uint32_t* b,
          int64_t n_rows, int64_t b_rows, const int32_t* row_limb, void* stream);

/* K:158-179 garner_digits over n_polys polynomials [L][N] (coefficient form). */
int pb_garner_digits(const pb_ctx* ctx, const uint32_t* rows, int64_t n_polys, uint32_t* digits,
                     void* stream);
/* K:182-199 scale_round_digits: digits [P][L][N] -> m [P][N] = round(t x/Q) mod t. */
int pb_scale_round_digits(const pb_ctx* ctx, const uint32_t* digits, int64_t n_polys,
                          uint64_t* out, void* stream);
/* Fused K:158-199 (garner + scale-round) for coefficient-form rows. */
int pb_decode(const pb_ctx* ctx, const uint32_t* rows, int64_t n_polys, uint64_t* out,
              void* stream);

/* K:135-147 negacyclic_mul_wrap (mod 2^64 schoolbook), batch of n pairs. */
int pb_negacyclic_mul_wrap(const uint64_t* a, const uint64_t* b, int64_t n_pairs, int32_t N,
                           uint64_t* out, void* stream);

/* ------------------------------------------------------- BFV (SPEC bfv) --- */
/* Plaintext sources: `vals` is a flat Z_t tensor.  A PACKED source gives,
 * for polynomial p and slot z < Z, coefficient pack_pos[p][z] =
 * vals[pack_src[p][z]] (pack_pos < 0: empty slot); all other coefficients
 * are zero.  This is the compact form of the packing maps pi_v / pi_W
 * (SPEC:231-266).  pack_pos == NULL means vals is a dense [P][N] array. */

/* Centered lift (fact 4) + forward NTT + Shoup companions:
 * plaintext multiplier for he_plain_mul.  pt/pt_shoup [P][L][N]. */
int pb_encode_plain(const pb_ctx* ctx, const uint64_t* vals, const int32_t* pack_pos,
                    const int32_t* pack_src, int32_t Z, int64_t P, uint32_t* pt, uint32_t* pt_shoup,
                    void* stream);

/* Lift of dense Z_t polys [P][N], coefficient form: out [P][L][N] = m mod q_i
 * (centered != 0 selects the centered lift v >= t/2 -> v - t). */
int pb_lift(const pb_ctx* ctx, const uint64_t* vals, int64_t P, int centered, uint32_t* out,
            void* stream);
/* Scatter a packed source into a zero-initialised dense [P][N] Z_t array. */
int pb_unpack(const uint64_t* vals, const int32_t* pack_pos, const int32_t* pack_src, int32_t Z,
              int32_t N, int64_t P, uint64_t* dense, void* stream);

/* SPEC:139-147 encrypt under the public key pk [2][L][N] (NTT form):
 * c0 = pk0*NTT(u) + NTT(e1 + Delta m), c1 = pk1*NTT(u) + NTT(e2).
 * u ternary, e1/e2 centred binomial (eta=20) drawn on the device from
 * Philox4x32(seed, nonce + poly index). ct [P][2][L][N]. */
int pb_encrypt_pk(const pb_ctx* ctx, const uint32_t* pk, const uint64_t* vals,
                  const int32_t* pack_pos, const int32_t* pack_src, int32_t Z, int64_t P,
                  uint64_t seed, const uint64_t* seed_dev, uint64_t nonce, uint32_t* ct, void* stream);
/* Same with caller-supplied noise (int8 [P][N] each): bit-exact with the
 * oracle's encrypt when fed the oracle's draws. */
int pb_encrypt_pk_noise(const pb_ctx* ctx, const uint32_t* pk, const uint64_t* vals,
                        const int32_t* pack_pos, const int32_t* pack_src, int32_t Z, int64_t P,
                        const int8_t* u, const int8_t* e1, const int8_t* e2, uint32_t* ct,
                        void* stream);
/* Symmetric-key encryption by the key owner: c1 = a (uniform, NTT domain),
 * c0 = NTT(e + Delta m) - a*s.  sk_ntt [L][N]; sk_shoup (nullable): its
 * Shoup companions (pb_shoup_rows), which make a*s three multiplies. */
int pb_encrypt_sk(const pb_ctx* ctx, const uint32_t* sk_ntt, const uint32_t* sk_shoup, const uint64_t* vals,
                  const int32_t* pack_pos, const int32_t* pack_src, int32_t Z, int64_t P,
                  uint64_t seed, const uint64_t* seed_dev, uint64_t nonce, uint32_t* ct, void* stream);
/* Shoup companions floor(x 2^32 / q_l) of n_rows NTT-domain rows (row r on limb r % L). */
int pb_shoup_rows(const pb_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n_rows, void* stream);
/* Caller-supplied a ([P][L][N], NTT domain, device order) and e (int8 [P][N]). */
int pb_encrypt_sk_noise(const pb_ctx* ctx, const uint32_t* sk_ntt, const uint64_t* vals,
                        const int32_t* pack_pos, const int32_t* pack_src, int32_t Z, int64_t P,
                        const uint32_t* a, const int8_t* e, uint32_t* ct, void* stream);

/* Split symmetric encryption: the ciphertexts of pb_encrypt_sk_noise, with
 * the message-independent work moved off the protocol's critical path.
 * pb_encrypt_sk_zero precomputes, elementwise (no NTT), ct = (-a*s, a) with
 * a the same uniform draw pb_encrypt_sk makes under (seed, nonce), and the
 * noise e int8 [P][N] (CBD(20), one draw per polynomial).  pb_encrypt_sk_add
 * then sets c0 += NTT(e + Delta m) in place: the result equals
 * pb_encrypt_sk_noise(m, a, e) bit for bit.  Replaces the same SPEC:139-147
 * encrypt as pb_encrypt_sk (mode "sk"). */
int pb_encrypt_sk_zero(const pb_ctx* ctx, const uint32_t* sk_ntt, int64_t P, uint64_t seed,
                       const uint64_t* seed_dev, uint64_t nonce, uint32_t* ct, int8_t* e, void* stream);
int pb_encrypt_sk_add(const pb_ctx* ctx, const uint64_t* vals, const int32_t* pack_pos,
                      const int32_t* pack_src, int32_t Z, int64_t P, const int8_t* e, uint32_t* ct,
                      void* stream);

/* x = INTT(c0 + c1*s) in coefficient form, x [P][L][N]. */
int pb_decrypt_coeffs(const pb_ctx* ctx, const uint32_t* sk_ntt, const uint32_t* ct, int64_t P,
                      uint32_t* x, void* stream);
/* SPEC:148-156 decrypt: m [P][N]; scratch [P][L][N] uint32. */
int pb_decrypt(const pb_ctx* ctx, const uint32_t* sk_ntt, const uint32_t* ct, int64_t P,
               uint64_t* m, uint32_t* scratch, void* stream);
/* Alg.1 step 4 / SPEC:240-266 decrypt + pi_y^-1 gather into a share tensor:
 * for each ct p and slot u < U: if out_pos[p][u] >= 0, share_out[out_dst[p][u]]
 * = decrypted coefficient out_pos[p][u].  scratch [P][L][U] uint32. */
int pb_decrypt_to_share(const pb_ctx* ctx, const uint32_t* sk_ntt, const uint32_t* ct, int64_t P,
                        const int32_t* out_pos, const int64_t* out_dst, int32_t U,
                        uint64_t* share_out, uint32_t* scratch, void* stream);

/* Alg.1 steps 2-3 / Alg.2 step 2, MO side, fused:
 *   ct_out[p] = sum_k ct_in[terms[p][k][0]] (*) pt[terms[p][k][1]]  -  Delta*mask_p
 * where mask_p has mask_vals[out_dst[p][u]] at coefficient out_pos[p][u] and,
 * when filler != 0, uniform Z_q filler (Philox4x32(filler_seed, p)) at every
 * other coefficient so the DO learns nothing beyond the useful slots.
 * Every RNG-consuming entry point takes `seed_dev` (nullable): when set, the
 * per-step seed is read from device memory so a CUDA graph can replay the
 * call with fresh randomness (see pb_common.cuh "seed indirection").
 * terms[p][k] with ct index < 0 is skipped.  ct_in [n][2][L][N],
 * pt/pt_shoup [n_pt][L][N], ct_out [P][2][L][N]. */
int pb_ctpt_mac_mask(const pb_ctx* ctx, const uint32_t* ct_in, const uint32_t* pt,
                     const uint32_t* pt_shoup, const int32_t* terms, int32_t K, int64_t P,
                     const int32_t* out_pos, const int64_t* out_dst, int32_t U,
                     const uint64_t* mask_vals, int filler, uint64_t filler_seed, const uint64_t* seed_dev,
                     uint32_t* ct_out, void* stream);

/* Tiled MO evaluation (the production path of Alg.1/Alg.2), in two steps:
 *  pb_mask_ntt:  ct_out[p].c0 = -Delta*NTT(mask_p)  (mask_p as in pb_ctpt_mac_mask:
 *                mask_vals at out_pos / filler elsewhere); c1 untouched.
 *  pb_ctpt_mac_tiled: for the nB x nO grid of outputs r = b*nO + o,
 *                ct_out[r].c0 += sum_k ctA[b*nI+k].c0 (*) ptA[o*nI+k] (+ ctB[o*nI+k].c0 (*) ptB[b*nI+k]),
 *                ct_out[r].c1  = the same sums over c1.
 *                Plaintexts in Montgomery form (pb_encode_plain_mont); either
 *                term may be absent (NULL ct). */
int pb_encode_plain_mont(const pb_ctx* ctx, const uint64_t* vals, const int32_t* pack_pos,
                         const int32_t* pack_src, int32_t Z, int64_t P, uint32_t* pt_mont, void* stream);
int pb_mask_ntt(const pb_ctx* ctx, int64_t P, const int32_t* out_pos, const int64_t* out_dst, int32_t U,
                const uint64_t* mask_vals, int filler, uint64_t filler_seed, const uint64_t* seed_dev,
                uint32_t* ct_out, void* stream);
int pb_ctpt_mac_tiled(const pb_ctx* ctx, const uint32_t* ctA, const uint32_t* ptA_mont, const uint32_t* ctB,
                      const uint32_t* ptB_mont, int32_t nB, int32_t nO, int32_t nI, uint32_t* ct_out,
                      void* stream);
/* Both steps in ONE pass for the streaming shapes (nI <= 2, e.g. FC-like
 * K = 1): per output row the -Delta*NTT(mask) row is built in registers and
 * the MAC terms added before the single store of c0 and c1 -- no -mask row
 * round trip through HBM.  Bit-identical to pb_mask_ntt + pb_ctpt_mac_tiled
 * with the same arguments. */
int pb_mask_mac(const pb_ctx* ctx, const uint32_t* ctA, const uint32_t* ptA_mont, const uint32_t* ctB,
                const uint32_t* ptB_mont, int32_t nB, int32_t nO, int32_t nI, const int32_t* out_pos,
                const int64_t* out_dst, int32_t U, const uint64_t* mask_vals, int filler, uint64_t filler_seed,
                const uint64_t* seed_dev, uint32_t* ct_out, void* stream);

/* ------------------------------------------- ring Z_{2^ell} (R:93-233) --- */
enum {
  PB_RING_ADD = 0, /* R:132-134 */
  PB_RING_SUB = 1, /* R:136-138 */
  PB_RING_MUL = 2, /* elementwise product (dealer / local terms) */
  PB_RING_NEG = 3, /* R:140-141 */
  PB_RING_SCALAR_MUL = 4, /* R:143-145, k = scalar */
  PB_RING_MASK = 5,       /* R:99-102 canonicalise */
  PB_RING_ARITH_SHIFT = 6 /* R:206-211, k = bits */
};
/* out = a (op) b elementwise mod 2^ell; b broadcast cyclically over b_n. */
int pb_ring_binary(int op, uint64_t* out, const uint64_t* a, const uint64_t* b, int64_t n,
                   int64_t b_n, int32_t ell, void* stream);
int pb_ring_unary(int op, uint64_t* out, const uint64_t* a, uint64_t k, int64_t n, int32_t ell,
                  void* stream);
/* out[i] = a[i] + b[(i / inner) % bn] mod 2^ell (bias add along an axis: FC (n_o, B) -> inner = B,
 * bn = n_o; conv (B, c_o, oh, ow) -> inner = oh*ow, bn = c_o). */
int pb_ring_add_bcast(uint64_t* out, const uint64_t* a, const uint64_t* b, int64_t n, int64_t inner, int64_t bn,
                      int32_t ell, void* stream);
/* R:174-182 encode_fixed; *range_flag (device int32) set to 1 on |x| >= limit. */
int pb_encode_fixed(const double* x, int64_t n, int32_t ell, int32_t scale, uint64_t* out,
                    int32_t* range_flag, void* stream);
/* R:185-191 decode_fixed. */
int pb_decode_fixed(const uint64_t* v, int64_t n, int32_t ell, int32_t scale, double* out,
                    void* stream);
/* R:60-61 SeededRng.uniform_ring: out[i] = raw(seed, stream_id, raw_offset+i) >> (64-ell),
 * bit-identical to numpy Generator(Philox(key=[seed, stream])).integers(0, 2^ell). */
int pb_uniform_ring(uint64_t* out, int64_t n, uint64_t seed, const uint64_t* seed_dev, uint64_t stream_id,
                    uint64_t raw_offset, int32_t ell, void* stream);
/* R:214-219 share_tensor fused: r = uniform_ring(...); mo = r; do = x - r. */
int pb_share(const uint64_t* x, int64_t n, uint64_t seed, const uint64_t* seed_dev, uint64_t stream_id,
             uint64_t raw_offset, int32_t ell, uint64_t* mo_out, uint64_t* do_out, void* stream);
/* K:206-218 matmul_wrap (+ mask to ell bits when ell < 64): (n,k)@(k,m).
 * trans_a / trans_b read a as (k,n) / b as (m,k) row-major. */
int pb_ring_matmul(const uint64_t* a, const uint64_t* b, int64_t n, int64_t k, int64_t m,
                   int trans_a, int trans_b, int32_t ell, uint64_t* out, void* stream);
/* out = c + sign * (a @ b) mod 2^ell (sign +1 / -1; c == NULL or sign == 0:
 * plain pb_ring_matmul) -- the protocols' "s - W <X>_0" and "msg + gY X^T"
 * local terms with the add fused into the GEMM epilogue. */
int pb_ring_matmul_add(const uint64_t* a, const uint64_t* b, int64_t n, int64_t k, int64_t m,
                       int trans_a, int trans_b, const uint64_t* c, int32_t sign, int32_t ell,
                       uint64_t* out, void* stream);
/* out[dst[i]] = src[i] for dst[i] >= 0: the multi-rank combine of sharded
 * block plans (all-gathered compact share tiles -> the output tensor). */
int pb_scatter_u64(uint64_t* out, const uint64_t* src, const int64_t* dst, int64_t n, void* stream);
/* Row reduction: out[i] = sum_j a[i][j] mod 2^ell  (reveal_grad_bias). */
int pb_ring_rowsum(const uint64_t* a, int64_t rows, int64_t cols, int32_t ell, uint64_t* out,
                   void* stream);
/* Channel reduction of an NCHW tensor a (B, C, HW): out[c] = sum_{b,i}
 * a[b][c][i] mod 2^ell (reveal_grad_bias for Conv2d). */
int pb_ring_chansum(const uint64_t* a, int32_t B, int32_t C, int64_t HW, int32_t ell, uint64_t* out,
                    void* stream);
/* K:221-238 im2col_wrap, K:241-257 col2im_wrap, K:260-278 conv2d_wrap. */
int pb_im2col(const uint64_t* x, int32_t B, int32_t C, int32_t H, int32_t W, int32_t s,
              int32_t stride, uint64_t* out, void* stream);
int pb_col2im(const uint64_t* cols, int32_t B, int32_t C, int32_t H, int32_t W, int32_t s,
              int32_t stride, uint64_t* out, void* stream);
int pb_conv2d(const uint64_t* x, const uint64_t* w, int32_t B, int32_t Ci, int32_t H, int32_t W,
              int32_t Co, int32_t s, int32_t ell, uint64_t* out, void* stream);

/* Conv-layer operators with padding / stride, computed directly (no padded
 * or dilated copies): the parties' local terms of the conv protocols.  They
 * equal the oracle's compositions of K:260-278 conv2d_wrap with the SPEC:284
 * pad / stride transforms (oracle/convops.py), mod 2^ell:
 *   PB_CONV_FWD   a = X  (B,c_i,H,W),   b = W (c_o,c_i,s,s), out = Y  (B,c_o,oh,ow)
 *   PB_CONV_BWDX  a = dY (B,c_o,oh,ow), b = W,               out = dX (B,c_i,H,W)
 *   PB_CONV_GRADW a = X,                b = dY,              out = dW (c_o,c_i,s,s)
 * with oh = (H + 2 pad - s) / stride + 1 (same for ow). */
enum { PB_CONV_FWD = 0, PB_CONV_BWDX = 1, PB_CONV_GRADW = 2 };
int pb_ring_conv(int kind, const uint64_t* a, const uint64_t* b, int32_t B, int32_t c_i, int32_t c_o, int32_t H,
                 int32_t W, int32_t s, int32_t pad, int32_t stride, int32_t ell, uint64_t* out, void* stream);
/* The ring GEMMs of pb_ring_matmul / pb_ring_conv with the kernel family
 * chosen explicitly: PB_BACKEND_AUTO (what the plain entry points do: a
 * function of the shape alone), PB_BACKEND_CUDA_CORE (u64 IMAD tiles),
 * PB_BACKEND_TENSOR (tcgen05 kind::i8 on balanced base-256 digit planes,
 * TMEM accumulators; pb_tc.cu).  Every backend is bit-exact mod 2^ell. */
enum { PB_BACKEND_AUTO = 0, PB_BACKEND_CUDA_CORE = 1, PB_BACKEND_TENSOR = 2 };
int pb_ring_conv_ex(int kind, const uint64_t* a, const uint64_t* b, int32_t B, int32_t c_i, int32_t c_o, int32_t H,
                    int32_t W, int32_t s, int32_t pad, int32_t stride, int32_t ell, uint64_t* out, int32_t backend,
                    void* stream);
int pb_ring_matmul_ex(const uint64_t* a, const uint64_t* b, int64_t n, int64_t k, int64_t m, int trans_a,
                      int trans_b, int32_t ell, uint64_t* out, int32_t backend, void* stream);
/* AvgPool2 local steps: PB_POOL_SUM in (bc,H,W) -> out (bc,H/2,W/2)
 * 2x2 window sums; PB_POOL_REPLICATE in (bc,H/2,W/2) -> out (bc,H,W). */
enum { PB_POOL_SUM = 0, PB_POOL_REPLICATE = 1 };
int pb_pool2(int op, const uint64_t* in, int64_t bc, int32_t H, int32_t W, int32_t ell, uint64_t* out,
             void* stream);

/* Pencil+ online phase (PAPER Alg. 3 steps 7-10): scalar-weighted
 * sums of mask tensors, out = base (+|-) sum_{i<ma,j<mb} a_i b_j T[i][j][:] mod
 * 2^ell; b == NULL means weights a_i alone (mb must be 1); base may be NULL. */
int pb_ring_lincomb(int subtract, uint64_t* out, const uint64_t* base, const uint64_t* a, int32_t ma,
                    const uint64_t* b, int32_t mb, const uint64_t* T, int64_t n, int32_t ell, void* stream);
/* The online scalars of one operator in one launch: k[i] (stream_k) and l[j]
 * (stream_l), i, j < m, = uniform_ring draws 0..m-1 of each numpy-identical
 * stream (R:60-61), 0 mapped to 1. */
int pb_prep_scalars(uint64_t* k_out, uint64_t* l_out, int32_t m, uint64_t seed, const uint64_t* seed_dev,
                    uint64_t stream_k, uint64_t stream_l, int32_t ell, void* stream);

/* ------------------------------- dealer-assisted non-linear --- */
/* The SPEC's dealer OT backend ("fast, insecure, default for benchmarks of
 * non-OT costs"): reconstruct x = mo + do, apply f, reshare with
 * r = uniform_ring(seed, stream_id, raw_offset + i).
 *   PB_DEALER_RELU     y = (x >= 0) ? x : 0, d_out[i] = (x >= 0)
 *   PB_DEALER_TRUNC    y = arith_shift(x, k)                       (faithful)
 *   PB_DEALER_SELECT   y = d_in[i] ? x : 0                         (ReLU backward, cached d)
 *   PB_DEALER_RESHARE  y = x
 *   PB_DEALER_RELU_TRUNC   y = arith_shift(relu(x), k), d_out as RELU  (forward ReLU + truncation;
 *                          the relu's own reshare is never observed, so the output shares equal
 *                          the two-step composition's when `stream_id` is the truncation's stream)
 *   PB_DEALER_TRUNC_SELECT y = d_in[i] ? arith_shift(x, k) : 0          (backward truncation + ReLU')
 * Outputs overwrite mo/do in place. */
enum {
  PB_DEALER_RELU = 0,
  PB_DEALER_TRUNC = 1,
  PB_DEALER_SELECT = 2,
  PB_DEALER_RESHARE = 3,
  PB_DEALER_RELU_TRUNC = 4,
  PB_DEALER_TRUNC_SELECT = 5
};
int pb_dealer_op(int op, uint64_t* mo, uint64_t* do_, int64_t n, int32_t k, const uint8_t* d_in,
                 uint8_t* d_out, uint64_t seed, const uint64_t* seed_dev, uint64_t stream_id,
                 uint64_t raw_offset, int32_t ell, void* stream);
/* The same with the input shares read from in_mo / in_do (out of place; the
 * inputs may alias the outputs). */
int pb_dealer_op_out(int op, const uint64_t* in_mo, const uint64_t* in_do, uint64_t* mo, uint64_t* do_,
                     int64_t n, int32_t k, const uint8_t* d_in, uint8_t* d_out, uint64_t seed,
                     const uint64_t* seed_dev, uint64_t stream_id, uint64_t raw_offset, int32_t ell,
                     void* stream);

/* OT-based non-linear protocols with the
 * SPEC:479 dealer OT backend, one thread per element (pb_nonlinear.cu):
 *   PB_NL_DRELU       XOR shares of 1{x >= 0} (millionaires' comparison in
 *                     4-bit blocks, 1-of-16 leaf OTs, Beaver-AND tree) -> d_out
 *                     (bit 0: P0 = MO share, bit 1: P1 = DO share)
 *   PB_NL_MUX         arithmetic shares of d * x (two 1-of-2 OTs), d from d_in
 *   PB_NL_TRUNC       faithful arith_shift(x, k) (wrap + low-carry comparisons, B2A)
 *   PB_NL_RELU_TRUNC  DReLU, MUX, TRUNC fused (d_out as DRELU)
 *   PB_NL_TRUNC_MUX   TRUNC then MUX with d_in (the backward ReLU')
 * x0 / x1: the MO's / DO's shares (n u64 < 2^ell); y0 / y1: output shares.
 * Randomness: raw draws raw_offset + i * pb_nl_words(op) + k of the
 * numpy-identical Philox stream (seed (+ *seed_dev), stream_id). */
enum { PB_NL_DRELU = 0, PB_NL_MUX = 1, PB_NL_TRUNC = 2, PB_NL_RELU_TRUNC = 3, PB_NL_TRUNC_MUX = 4 };
int pb_nl_words(int op);
int pb_nl_op(int op, const uint64_t* x0, const uint64_t* x1, int64_t n, int32_t ell, int32_t k, const uint8_t* d_in,
             uint8_t* d_out, uint64_t seed, const uint64_t* seed_dev, uint64_t stream_id, uint64_t raw_offset,
             uint64_t* y0, uint64_t* y1, void* stream);

/* SGD with momentum in float64 + re-quantisation:
 * v = mu*v + g; w = w - lr*v; w_ring = encode_fixed(w, scale).  skip
 * (nullable device word): nonzero -> no-op (an aborted step, see
 * pb_host_handoff). */
int pb_sgd_momentum(double* w, double* v, const uint64_t* grad_ring, int64_t n, int32_t grad_scale,
                    double lr, double momentum, int32_t ell, int32_t w_scale, uint64_t* w_ring,
                    int32_t* range_flag, const uint32_t* skip, void* stream);

/* The DO's host-side softmax cross-entropy around numpy's
 * exp / log: pb_host_softmax_pre writes z = logits/2^f2 (signed, ell bits)
 * minus the column max into z [C][B]; the caller sets z = exp(z) with numpy;
 * pb_host_softmax_post normalises, returns the label probabilities (for the
 * caller's numpy log / mean) and g = floor((p - onehot)/D * 2^f) mod 2^ell
 * with D = denom, or B when denom == 0 (data parallelism: D = the global
 * batch, so the ranks' revealed gradients sum to the global-batch gradient).
 * Host functions (no device work); bit-identical to oracle/protocols.py. */
int pb_host_softmax_pre(const uint64_t* logits, int32_t C, int32_t B, int32_t ell, int32_t f2, double* z);
int pb_host_softmax_post(double* ez, int32_t C, int32_t B, const int64_t* labels, int32_t ell, int32_t f,
                         int32_t denom, double* p_lab, uint64_t* g_out);

/* Cap the grid of the one-CTA-per-row kernels (encrypt, plaintext encoding)
 * launched afterwards from this host thread at max_ctas (0: no cap); the
 * kernels then loop over rows.  For background work (operands prepared off
 * the critical path) that must leave SM slots to concurrent kernels. */
int pb_set_launch_cap(int32_t max_ctas);

/* cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream). */
int pb_copy_async(void* dst, const void* src, int64_t bytes, void* stream);

/* Step prologue for a replayed graph: *dev_word = *host_word (pinned host
 * memory read by the kernel; host_word NULL: skipped) and a D2D copy of
 * `bytes` (multiple of 16, 16-byte aligned) from src to dst, one launch. */
int pb_step_prologue(const uint64_t* host_word, uint64_t* dev_word, const void* src, void* dst, int64_t bytes,
                     void* stream);

/* Device -> host publication at the end of a replayed graph: one CTA copies
 * n u64 from src (device) into pinned host memory dst_host with system-scope
 * stores, then increments *seq_dev and writes it to the pinned word
 * flag_host (system-scope release).  The host polls flag_host instead of a
 * D2H copy + event (the logits the DO's loss needs). */
int pb_host_publish(const uint64_t* src, uint64_t* dst_host, int64_t n, uint32_t* seq_dev, uint32_t* flag_host,
                    void* stream);

/* Host -> device handoff inside a CUDA graph launched ahead of the host:
 * one CTA waits until the pinned host word flag_host[0] equals *seq_dev + 1
 * (system-scope acquire), stores that into *seq_dev, acks it into
 * flag_host[1] and copies n u64 from pinned host memory src_host to dst.
 * The host releases the k-th replay by writing src then flag_host[0] = k.
 * After timeout_ns the kernel gives up, acks (and sets *seq_dev to)
 * UINT32_MAX and copies whatever src holds (the caller checks the ack).
 * *skip_dev (nullable) = 1 after a timeout or when the host set the abort
 * word flag_host[2] before releasing (its loss raised), else 0; every
 * pb_sgd_momentum of the step reads it and then leaves w, v, w_ring as
 * they were, so an aborted step never applies a stale gradient.
 * Replaces the loss-gradient H2D copy + graph launch between the DO's host
 * loss and the backward pass. */
int pb_host_handoff(uint32_t* flag_host, uint32_t* seq_dev, const uint64_t* src_host, uint64_t* dst,
                    int64_t n, int64_t timeout_ns, uint32_t* skip_dev, void* stream);

/* SPEC:196 response compaction (modulus switch, OFF by default): ct rows
 * [n_polys][L][N] (NTT form, device order) under Q = q_0..q_{L-1} ->
 * out [n_polys][L-1][N] under Q' = Q / q_{L-1}, c' = round(c Q'/Q), i.e.
 * c'_i = (c_i - [c]_{q_{L-1}}) q_{L-1}^-1 mod q_i with the centered
 * coefficient-form residue of the dropped limb.  ctx_low: the context of
 * q_0..q_{L-2}; ctx_last: the 1-limb context of q_{L-1}; scratch [n_polys][N].
 * Decrypt the result under ctx_low with the first L-1 key rows. */
int pb_mod_switch_drop(const pb_ctx* ctx_low, const pb_ctx* ctx_last, const uint32_t* ct, int64_t n_polys,
                       uint32_t* out, uint32_t* scratch, void* stream);

/* PBFV wire format (the serialize boundary of SPEC:194 and the
 * frame payload whose size the census counts).  One frame per
 * object: {magic "PBFV", version u16 = PB_WIRE_VERSION, N u32, L u8, form u8}
 * (12 bytes, packed little-endian) then n_polys (2: ciphertext c0, c1; 1:
 * plaintext) x L x N little-endian u64 residues.  form PB_WIRE_NTT rows are
 * in the reference's bit-reversed NTT order (K:ntt_forward), converted from
 * the device order inside the kernel; PB_WIRE_COEFF rows are written as
 * given (the caller passes coefficient-form rows).  `out` / `in` may be
 * device memory or pinned host memory (UVA: the kernel then does the
 * transfer itself); 4-byte aligned; polys 16-byte aligned.
 * pb_wire_deserialize zeroes *bad (device int32) and ORs PB_WIRE_BAD_* into
 * it; the caller reads it after the stream and raises (HandshakeError-class
 * header faults, ParamsError, FormError, EncodeRangeError). */
#define PB_WIRE_VERSION 1
enum { PB_WIRE_COEFF = 0, PB_WIRE_NTT = 1 };
enum { PB_WIRE_BAD_HEADER = 1, PB_WIRE_BAD_PARAMS = 2, PB_WIRE_BAD_FORM = 4, PB_WIRE_BAD_RESIDUE = 8 };
#define PB_WIRE_FRAME_SIZE(N, L, n_polys) (12 + (int64_t)(n_polys) * (L) * (N) * 8)
int pb_wire_frame_bytes(const pb_ctx* ctx, int32_t n_polys, int64_t* out_host);
int pb_wire_serialize(const pb_ctx* ctx, const uint32_t* polys, int64_t P, int32_t n_polys, int32_t form,
                      uint8_t* out, void* stream);
int pb_wire_deserialize(const pb_ctx* ctx, const uint8_t* in, int64_t P, int32_t n_polys, int32_t form,
                        uint32_t* polys, int32_t* bad, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PENCIL_B200_H_ */
