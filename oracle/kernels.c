/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C + OpenMP) of the reference's numeric kernel tier
 * `pencil._kernels` (/root/reference/pkg/src/pencil/_kernels.py, "K" below).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library; the product path
 * (paper_2403_11166_b200/) never does.
 *
 * Every function follows the K function named in its comment line-for-line
 * in *algorithm* (same loop order, same `%` reductions, same uint64
 * wraparound, same float64 accumulation order) so its outputs are
 * bit-identical to K on the same inputs.  Parity with K itself is pinned by
 * tests/golden/make_golden.py (run in the build container where the
 * reference is importable) and tests/test_oracle_golden.py.
 *
 * Build: see oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off).
 * -ffp-contract=off matters: K accumulates float(d)*frac in float64 without
 * FMA contraction (numba default, no fastmath), K:193-198.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;

/* K:18-19 set_threads */
#ifdef _OPENMP
#include <omp.h>
void orc_set_threads(int n) { omp_set_num_threads(n < 1 ? 1 : n); }
int orc_get_threads(void) { return omp_get_max_threads(); }
#else
void orc_set_threads(int n) { (void)n; }
int orc_get_threads(void) { return 1; }
#endif

/* K:31-50 ntt_forward: in-place negacyclic Cooley-Tukey, psi^bitrev tables,
 * bit-reversed output.  rows/psi_brv are (R, N) row-major; q is (R,). */
void orc_ntt_forward(u64 *rows, const u64 *psi_brv, const u64 *q, int64_t R, int64_t N) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    u64 *a = rows + r * N;
    const u64 *w = psi_brv + r * N;
    const u64 qq = q[r];
    int64_t t = N;
    for (int64_t m = 1; m < N; m *= 2) {
      t /= 2;
      for (int64_t i = 0; i < m; ++i) {
        const u64 wi = w[m + i];
        const int64_t j1 = 2 * i * t;
        for (int64_t j = j1; j < j1 + t; ++j) {
          const u64 u = a[j];
          const u64 v = (a[j + t] * wi) % qq;
          a[j] = (u + v) % qq;
          a[j + t] = (u + qq - v) % qq;
        }
      }
    }
  }
}

/* K:53-77 ntt_inverse: in-place Gentleman-Sande, then a separate x N^-1 pass. */
void orc_ntt_inverse(u64 *rows, const u64 *ipsi_brv, const u64 *n_inv, const u64 *q,
                     int64_t R, int64_t N) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    u64 *a = rows + r * N;
    const u64 *w = ipsi_brv + r * N;
    const u64 qq = q[r];
    int64_t t = 1;
    for (int64_t m = N; m > 1; m /= 2) {
      const int64_t h = m / 2;
      int64_t j1 = 0;
      for (int64_t i = 0; i < h; ++i) {
        const u64 wi = w[h + i];
        for (int64_t j = j1; j < j1 + t; ++j) {
          const u64 u = a[j];
          const u64 v = a[j + t];
          a[j] = (u + v) % qq;
          a[j + t] = ((u + qq - v) * wi) % qq;
        }
        j1 += 2 * t;
      }
      t *= 2;
    }
    const u64 ninv = n_inv[r];
    for (int64_t j = 0; j < N; ++j) a[j] = (a[j] * ninv) % qq;
  }
}

/* K:80-86 pw_mul */
void orc_pw_mul(u64 *out, const u64 *a, const u64 *b, const u64 *q, int64_t R, int64_t N) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    const u64 qq = q[r];
    for (int64_t j = 0; j < N; ++j) out[r * N + j] = (a[r * N + j] * b[r * N + j]) % qq;
  }
}

/* K:89-95 pw_mul_acc: out = (out + a*b % q) % q */
void orc_pw_mul_acc(u64 *out, const u64 *a, const u64 *b, const u64 *q, int64_t R, int64_t N) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    const u64 qq = q[r];
    for (int64_t j = 0; j < N; ++j)
      out[r * N + j] = (out[r * N + j] + (a[r * N + j] * b[r * N + j]) % qq) % qq;
  }
}

/* K:98-104 pw_add */
void orc_pw_add(u64 *out, const u64 *a, const u64 *b, const u64 *q, int64_t R, int64_t N) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    const u64 qq = q[r];
    for (int64_t j = 0; j < N; ++j) out[r * N + j] = (a[r * N + j] + b[r * N + j]) % qq;
  }
}

/* K:107-113 pw_sub */
void orc_pw_sub(u64 *out, const u64 *a, const u64 *b, const u64 *q, int64_t R, int64_t N) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    const u64 qq = q[r];
    for (int64_t j = 0; j < N; ++j) out[r * N + j] = (a[r * N + j] + qq - b[r * N + j]) % qq;
  }
}

/* K:116-132 negacyclic_mul_mod: schoolbook a*b mod (X^N+1, q). */
void orc_negacyclic_mul_mod(const u64 *a, const u64 *b, u64 q, int64_t N, u64 *out) {
  memset(out, 0, (size_t)N * sizeof(u64));
  for (int64_t i = 0; i < N; ++i) {
    const u64 ai = a[i] % q;
    if (ai == 0) continue;
    for (int64_t j = 0; j < N; ++j) {
      const int64_t k = i + j;
      const u64 v = (ai * (b[j] % q)) % q;
      if (k < N)
        out[k] = (out[k] + v) % q;
      else
        out[k - N] = (out[k - N] + q - v) % q;
    }
  }
}

/* K:135-147 negacyclic_mul_wrap: schoolbook negacyclic product mod 2^64. */
void orc_negacyclic_mul_wrap(const u64 *a, const u64 *b, int64_t N, u64 *out) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < N; ++k) {
    u64 acc = 0;
    for (int64_t i = 0; i <= k; ++i) acc += a[i] * b[k - i];
    for (int64_t i = k + 1; i < N; ++i) acc -= a[i] * b[k + N - i];
    out[k] = acc;
  }
}

/* K:158-179 garner_digits: mixed-radix digits, O(L^2) per coefficient. */
void orc_garner_digits(const u64 *rows, const u64 *q, const u64 *prefix_inv, int64_t L,
                       int64_t N, u64 *digits) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < N; ++j) {
    for (int64_t i = 0; i < L; ++i) {
      const u64 qi = q[i];
      u64 acc = 0, mul = 1;
      for (int64_t k = 0; k < i; ++k) {
        acc = (acc + digits[k * N + j] * mul) % qi;
        mul = (mul * (q[k] % qi)) % qi;
      }
      const u64 x = rows[i * N + j] % qi;
      const u64 diff = (x + qi - acc) % qi;
      digits[i * N + j] = (diff * prefix_inv[i]) % qi;
    }
  }
}

/* K:182-199 scale_round_digits: m = round(t*x/q) mod t from mixed-radix
 * digits; integer part in uint64 wraparound, fraction in float64. */
void orc_scale_round_digits(const u64 *digits, const u64 *int_part, const double *frac_part,
                            u64 t_mask, int64_t L, int64_t N, u64 *out) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < N; ++j) {
    u64 acc_i = 0;
    double acc_f = 0.0;
    for (int64_t i = 0; i < L; ++i) {
      const u64 d = digits[i * N + j];
      acc_i += d * int_part[i];
      acc_f += (double)d * frac_part[i];
    }
    out[j] = (acc_i + (u64)floor(acc_f + 0.5)) & t_mask;
  }
}

/* K:206-218 matmul_wrap: (n,k)@(k,m) with uint64 wraparound. */
void orc_matmul_wrap(const u64 *a, const u64 *b, int64_t n, int64_t k, int64_t m, u64 *out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < m; ++j) {
      u64 acc = 0;
      for (int64_t l = 0; l < k; ++l) acc += a[i * k + l] * b[l * m + j];
      out[i * m + j] = acc;
    }
  }
}

/* K:221-238 im2col_wrap: (B,C,H,W) -> (C*s*s, B*oh*ow). */
void orc_im2col_wrap(const u64 *x, int64_t B, int64_t C, int64_t H, int64_t W, int64_t s,
                     int64_t stride, u64 *out) {
  const int64_t oh = (H - s) / stride + 1, ow = (W - s) / stride + 1;
  const int64_t ncol = B * oh * ow;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t i = 0; i < oh; ++i)
      for (int64_t j = 0; j < ow; ++j) {
        const int64_t col = (b * oh + i) * ow + j;
        int64_t row = 0;
        for (int64_t c = 0; c < C; ++c)
          for (int64_t di = 0; di < s; ++di)
            for (int64_t dj = 0; dj < s; ++dj) {
              out[row * ncol + col] =
                  x[((b * C + c) * H + i * stride + di) * W + j * stride + dj];
              ++row;
            }
      }
}

/* K:241-257 col2im_wrap: adjoint scatter-add. */
void orc_col2im_wrap(const u64 *cols, int64_t B, int64_t C, int64_t H, int64_t W, int64_t s,
                     int64_t stride, u64 *out) {
  const int64_t oh = (H - s) / stride + 1, ow = (W - s) / stride + 1;
  const int64_t ncol = B * oh * ow;
  memset(out, 0, (size_t)(B * C * H * W) * sizeof(u64));
  for (int64_t b = 0; b < B; ++b)
    for (int64_t i = 0; i < oh; ++i)
      for (int64_t j = 0; j < ow; ++j) {
        const int64_t col = (b * oh + i) * ow + j;
        int64_t row = 0;
        for (int64_t c = 0; c < C; ++c)
          for (int64_t di = 0; di < s; ++di)
            for (int64_t dj = 0; dj < s; ++dj) {
              out[((b * C + c) * H + i * stride + di) * W + j * stride + dj] +=
                  cols[row * ncol + col];
              ++row;
            }
      }
}

/* K:260-278 conv2d_wrap: valid cross-correlation, stride 1, uint64 wrap. */
void orc_conv2d_wrap(const u64 *x, const u64 *w, int64_t B, int64_t Ci, int64_t H, int64_t W,
                     int64_t Co, int64_t s, u64 *out) {
  const int64_t oh = H - s + 1, ow = W - s + 1;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < B; ++b)
    for (int64_t co = 0; co < Co; ++co)
      for (int64_t i = 0; i < oh; ++i)
        for (int64_t j = 0; j < ow; ++j) {
          u64 acc = 0;
          for (int64_t ci = 0; ci < Ci; ++ci)
            for (int64_t di = 0; di < s; ++di)
              for (int64_t dj = 0; dj < s; ++dj)
                acc += x[((b * Ci + ci) * H + i + di) * W + j + dj] *
                       w[((co * Ci + ci) * s + di) * s + dj];
          out[((b * Co + co) * oh + i) * ow + j] = acc;
        }
}

/* ------------------------------------------------------------------------
 * Cyclic-limb variants used by the oracle's BFV glue.  Identical arithmetic
 * to the K functions above; the only difference is that row r uses the
 * table/modulus of limb (r % L) instead of a per-row copy of the table, so
 * a batch of P polynomials x L limbs does not replicate the twiddle tables
 * P times.  Bit-identical to calling the K functions on tiled tables
 * (tests/test_oracle_golden.py::test_cyclic_variants_match_k).
 * ------------------------------------------------------------------------ */
void orc_ntt_forward_cyc(u64 *rows, const u64 *psi_brv, const u64 *q, int64_t R, int64_t N,
                         int64_t L) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    const int64_t l = r % L;
    orc_ntt_forward(rows + r * N, psi_brv + l * N, q + l, 1, N);
  }
}

void orc_ntt_inverse_cyc(u64 *rows, const u64 *ipsi_brv, const u64 *n_inv, const u64 *q,
                         int64_t R, int64_t N, int64_t L) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    const int64_t l = r % L;
    orc_ntt_inverse(rows + r * N, ipsi_brv + l * N, n_inv + l, q + l, 1, N);
  }
}

/* op: 0 mul, 1 mul_acc, 2 add, 3 sub.  b_rows: number of rows of b; row r of
 * a/out pairs with row (r % b_rows) of b (broadcast of a [L,N] operand). */
void orc_pw_cyc(int op, u64 *out, const u64 *a, const u64 *b, const u64 *q, int64_t R,
                int64_t N, int64_t L, int64_t b_rows) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    const u64 qq = q[r % L];
    const u64 *br = b + (r % b_rows) * N;
    u64 *o = out + r * N;
    const u64 *ar = a + r * N;
    for (int64_t j = 0; j < N; ++j) {
      switch (op) {
        case 0: o[j] = (ar[j] * br[j]) % qq; break;
        case 1: o[j] = (o[j] + (ar[j] * br[j]) % qq) % qq; break;
        case 2: o[j] = (ar[j] + br[j]) % qq; break;
        default: o[j] = (ar[j] + qq - br[j]) % qq; break;
      }
    }
  }
}

/* Batched decode: garner_digits + scale_round_digits (K:158-199) applied to
 * P polynomials of L rows each; identical per-coefficient arithmetic. */
void orc_decode_batch(const u64 *rows, const u64 *q, const u64 *prefix_inv, const u64 *int_part,
                      const double *frac_part, u64 t_mask, int64_t P, int64_t L, int64_t N,
                      u64 *out) {
#pragma omp parallel for schedule(static)
  for (int64_t pj = 0; pj < P * N; ++pj) {
    const int64_t p = pj / N, j = pj % N;
    const u64 *x = rows + p * L * N;
    u64 dig[16];
    for (int64_t i = 0; i < L; ++i) {
      const u64 qi = q[i];
      u64 acc = 0, mul = 1;
      for (int64_t k = 0; k < i; ++k) {
        acc = (acc + dig[k] * mul) % qi;
        mul = (mul * (q[k] % qi)) % qi;
      }
      const u64 xv = x[i * N + j] % qi;
      const u64 diff = (xv + qi - acc) % qi;
      dig[i] = (diff * prefix_inv[i]) % qi;
    }
    u64 acc_i = 0;
    double acc_f = 0.0;
    for (int64_t i = 0; i < L; ++i) {
      acc_i += dig[i] * int_part[i];
      acc_f += (double)dig[i] * frac_part[i];
    }
    out[pj] = (acc_i + (u64)floor(acc_f + 0.5)) & t_mask;
  }
}
