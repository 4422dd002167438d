/* oracle/dfa_oracle.c -- CPU restatement of the reference's Dilated Flash
 * Attention forward path.  TEST INFRASTRUCTURE ONLY: it is the checker for
 * the CUDA path and the "port" CPU baseline; the product never links it.
 *
 * Every function restates the reference algorithm in plain C, in the same
 * floating-point operation order, so that built with the reference's flags
 * (-O3 -ffp-contract=off) it is BIT-IDENTICAL to the reference (pinned by
 * tests/test_oracle.py against oracle/_ref/libattnkit_ref.so, which is the
 * unmodified reference compiled from /root/reference).
 *
 * Reference = /root/reference/proj/include/attnkit/.
 *   oracle_validate            attention.hpp:44-65   AttentionConfig::validate
 *   oracle_segment_view        attention.hpp:84-98   make_segment_view
 *   oracle_dilated_attention_* attention.hpp:280-301 dilated_attention
 *       segment gather           attention.hpp:210-222, tensor.hpp:320-332
 *       naive kernel             attention.hpp:119-127, tensor.hpp:175-203,239-258
 *       tiled kernel             attention.hpp:147-207
 *       recompose/scatter        attention.hpp:246-274, tensor.hpp:334-352
 *   oracle_masked_dense_f64    oracles.hpp:67-107    masked_dense_dilated
 *   oracle_flop_count          attention.hpp:370-387 flop_count
 *   oracle_dilated_lse_f64     EXTENSION (no reference code): natural-log
 *                              log-sum-exp of the scaled scores per kept row
 *   oracle_multibranch_f64     EXTENSION (no reference code; SPEC.md:204
 *                              lists multi-(w,r) as a non-goal): LSE-weighted
 *                              combine of several (w, r, gamma) branches,
 *                              restated as one dense softmax over the multiset
 *                              of keys the covering branches select.  Parity
 *                              of this function is UNPINNED by the reference
 *                              except in the single-branch case, where it
 *                              must equal dilated_attention (tested).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_OK = 0, ORC_ERR_CONFIG = 1, ORC_ERR_DIMENSION = 2, ORC_ERR_OUT_OF_RANGE = 3, ORC_ERR_CONTRACT = 4 };

/* attention.hpp:44-65 */
int oracle_validate(int64_t n, int64_t w, int64_t r, int64_t h, int64_t d, const int64_t* offsets, int64_t n_offsets,
                    int32_t kernel_tiled, int64_t tile, int32_t full_coverage) {
  if (n < 1) return ORC_ERR_CONFIG;
  if (w < 1 || w > n) return ORC_ERR_CONFIG;
  if (r < 1 || r > w) return ORC_ERR_CONFIG;
  if (h < 1) return ORC_ERR_CONFIG;
  if (d < 1) return ORC_ERR_CONFIG;
  if (n_offsets != h) return ORC_ERR_CONFIG;
  for (int64_t j = 0; j < n_offsets; ++j)
    if (offsets[j] < 0 || offsets[j] >= r) return ORC_ERR_CONFIG;
  if (kernel_tiled && tile < 1) return ORC_ERR_CONFIG;
  if (full_coverage) {
    for (int64_t c = 0; c < r; ++c) {
      int hit = 0;
      for (int64_t j = 0; j < n_offsets; ++j) hit |= (offsets[j] % r) == c;
      if (!hit) return ORC_ERR_CONFIG;
    }
  }
  return ORC_OK;
}

/* attention.hpp:84-98: rows {i*w + g + t*r} clipped to [i*w, min((i+1)w, N)). */
int oracle_segment_view(int64_t n, int64_t w, int64_t r, int64_t i, int64_t g, int64_t* rows, int64_t cap,
                        int64_t* count) {
  const int64_t n_seg = (n + w - 1) / w;
  if (i < 0 || i >= n_seg) return ORC_ERR_OUT_OF_RANGE;
  if (g < 0 || g >= r) return ORC_ERR_OUT_OF_RANGE;
  const int64_t begin = i * w;
  const int64_t end = begin + w < n ? begin + w : n;
  int64_t c = 0;
  for (int64_t row = begin + g; row < end; row += r) {
    if (c < cap) rows[c] = row;
    ++c;
  }
  *count = c;
  return ORC_OK;
}

/* attention.hpp:370-387; multiplications only. */
int oracle_flop_count(int64_t n, int64_t w, int64_t r, int64_t h, int64_t d, const int64_t* offsets,
                      uint64_t* dense, uint64_t* dilated, double* ratio) {
  if (oracle_validate(n, w, r, h, d, offsets, h, 0, 1, 0) != ORC_OK) return ORC_ERR_CONFIG;
  *dense = (uint64_t)h * 2u * (uint64_t)n * (uint64_t)n * (uint64_t)d;
  *dilated = 0;
  const int64_t n_seg = (n + w - 1) / w;
  for (int64_t j = 0; j < h; ++j)
    for (int64_t i = 0; i < n_seg; ++i) {
      int64_t m = 0;
      oracle_segment_view(n, w, r, i, offsets[j], NULL, 0, &m);
      *dilated += 2u * (uint64_t)m * (uint64_t)m * (uint64_t)d;
    }
  *ratio = (double)*dense / (double)*dilated;
  return ORC_OK;
}

/* One type-generic body per scalar type.  S = scalar, SQRT/EXP = the libm
 * functions std::sqrt / std::exp resolve to for that type. */
#define DFA_ORACLE_BODY(S, SFX, SQRT, EXP)                                                                     \
  /* attention.hpp:119-127 naive_attention on gathered rows; tensor.hpp matmul (i,k,j order, zero-init),   \
   * scale after the dot product, softmax_rows (max, exp, sum, divide), matmul(P, v). */                    \
  static void naive_##SFX(const S* q, const S* k, const S* v, int64_t m, int64_t d, int64_t dv, int scale,    \
                          S* o) {                                                                            \
    S* s = (S*)calloc((size_t)(m * m), sizeof(S));                                                           \
    S* p = (S*)calloc((size_t)(m * m), sizeof(S));                                                           \
    for (int64_t i = 0; i < m; ++i)                                                                          \
      for (int64_t kk = 0; kk < d; ++kk) {                                                                   \
        const S a = q[i * d + kk];                                                                           \
        for (int64_t j = 0; j < m; ++j) s[i * m + j] += a * k[j * d + kk];                                   \
      }                                                                                                      \
    if (scale) {                                                                                             \
      const S sc = (S)1 / SQRT((S)d);                                                                        \
      for (int64_t e = 0; e < m * m; ++e) s[e] *= sc;                                                        \
    }                                                                                                        \
    for (int64_t i = 0; i < m; ++i) {                                                                        \
      const S* in = s + i * m;                                                                               \
      S* out = p + i * m;                                                                                    \
      S mx = in[0];                                                                                          \
      for (int64_t j = 1; j < m; ++j) mx = (mx < in[j]) ? in[j] : mx;                                        \
      S sum = 0;                                                                                             \
      for (int64_t j = 0; j < m; ++j) {                                                                      \
        out[j] = EXP(in[j] - mx);                                                                            \
        sum += out[j];                                                                                       \
      }                                                                                                      \
      for (int64_t j = 0; j < m; ++j) out[j] /= sum;                                                         \
    }                                                                                                        \
    memset(o, 0, sizeof(S) * (size_t)(m * dv));                                                              \
    for (int64_t i = 0; i < m; ++i)                                                                          \
      for (int64_t kk = 0; kk < m; ++kk) {                                                                   \
        const S a = p[i * m + kk];                                                                           \
        for (int64_t c = 0; c < dv; ++c) o[i * dv + c] += a * v[kk * dv + c];                                \
      }                                                                                                      \
    free(s);                                                                                                 \
    free(p);                                                                                                 \
  }                                                                                                          \
  /* attention.hpp:147-207 tiled_attention (online softmax over key tiles); tile >= m -> naive. */          \
  static void tiled_##SFX(const S* q, const S* k, const S* v, int64_t m, int64_t d, int64_t dv, int scale,    \
                          int64_t tile, S* o) {                                                              \
    if (tile >= m) {                                                                                         \
      naive_##SFX(q, k, v, m, d, dv, scale, o);                                                              \
      return;                                                                                                \
    }                                                                                                        \
    const S sc = scale ? (S)1 / SQRT((S)d) : (S)1;                                                           \
    S* rmax = (S*)malloc(sizeof(S) * (size_t)m);                                                             \
    S* rnorm = (S*)calloc((size_t)m, sizeof(S));                                                             \
    S* sco = (S*)calloc((size_t)(m * tile), sizeof(S));                                                      \
    for (int64_t i = 0; i < m; ++i) rmax[i] = -(S)INFINITY;                                                  \
    memset(o, 0, sizeof(S) * (size_t)(m * dv));                                                              \
    for (int64_t t0 = 0; t0 < m; t0 += tile) {                                                               \
      const int64_t tw = tile < m - t0 ? tile : m - t0;                                                      \
      for (int64_t i = 0; i < m; ++i)                                                                        \
        for (int64_t j = 0; j < tw; ++j) {                                                                   \
          S acc = 0;                                                                                         \
          for (int64_t c = 0; c < d; ++c) acc += q[i * d + c] * k[(t0 + j) * d + c];                         \
          sco[i * tile + j] = acc * sc;                                                                      \
        }                                                                                                    \
      for (int64_t i = 0; i < m; ++i) {                                                                      \
        S tmax = sco[i * tile];                                                                              \
        for (int64_t j = 1; j < tw; ++j) tmax = (tmax < sco[i * tile + j]) ? sco[i * tile + j] : tmax;       \
        const S nmax = (rmax[i] < tmax) ? tmax : rmax[i];                                                    \
        const S corr = EXP(rmax[i] - nmax);                                                                  \
        S* oi = o + i * dv;                                                                                  \
        for (int64_t c = 0; c < dv; ++c) oi[c] *= corr;                                                      \
        S tsum = 0;                                                                                          \
        for (int64_t j = 0; j < tw; ++j) {                                                                   \
          const S pj = EXP(sco[i * tile + j] - nmax);                                                        \
          tsum += pj;                                                                                        \
          for (int64_t c = 0; c < dv; ++c) oi[c] += pj * v[(t0 + j) * dv + c];                               \
        }                                                                                                    \
        rnorm[i] = rnorm[i] * corr + tsum;                                                                   \
        rmax[i] = nmax;                                                                                      \
      }                                                                                                      \
    }                                                                                                        \
    for (int64_t i = 0; i < m; ++i) {                                                                        \
      const S inv = (S)1 / rnorm[i];                                                                         \
      for (int64_t c = 0; c < dv; ++c) o[i * dv + c] *= inv;                                                 \
    }                                                                                                        \
    free(rmax);                                                                                              \
    free(rnorm);                                                                                             \
    free(sco);                                                                                               \
  }                                                                                                          \
  /* attention.hpp:280-301; q,k [n x d], v [n x dv] row-major; out [n x dv]. */                              \
  int oracle_dilated_attention_##SFX(const S* q, const S* k, const S* v, int64_t n, int64_t d, int64_t dv,    \
                                     int64_t w, int64_t r, int64_t gamma, int32_t scale, int32_t kernel_tiled, \
                                     int64_t tile, S* out) {                                                 \
    const int64_t off = gamma;                                                                               \
    if (oracle_validate(n, w, r, 1, d, &off, 1, kernel_tiled, tile, 0) != ORC_OK) return ORC_ERR_CONFIG;     \
    if (gamma < 0 || gamma >= r) return ORC_ERR_OUT_OF_RANGE;                                                \
    const int64_t n_seg = (n + w - 1) / w;                                                                   \
    const int64_t mmax = (w + r - 1) / r;                                                                    \
    S* qs = (S*)malloc(sizeof(S) * (size_t)(mmax * d));                                                      \
    S* ks = (S*)malloc(sizeof(S) * (size_t)(mmax * d));                                                      \
    S* vs = (S*)malloc(sizeof(S) * (size_t)(mmax * dv));                                                     \
    S* os = (S*)malloc(sizeof(S) * (size_t)(mmax * dv));                                                     \
    int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)mmax);                                        \
    memset(out, 0, sizeof(S) * (size_t)(n * dv));                                                            \
    for (int64_t i = 0; i < n_seg; ++i) {                                                                    \
      int64_t m = 0;                                                                                         \
      oracle_segment_view(n, w, r, i, gamma, rows, mmax, &m);                                                \
      if (m == 0) continue;                                                                                  \
      for (int64_t t = 0; t < m; ++t) {                                                                      \
        memcpy(qs + t * d, q + rows[t] * d, sizeof(S) * (size_t)d);                                          \
        memcpy(ks + t * d, k + rows[t] * d, sizeof(S) * (size_t)d);                                          \
        memcpy(vs + t * dv, v + rows[t] * dv, sizeof(S) * (size_t)dv);                                       \
      }                                                                                                      \
      if (kernel_tiled)                                                                                      \
        tiled_##SFX(qs, ks, vs, m, d, dv, scale, tile, os);                                                  \
      else                                                                                                   \
        naive_##SFX(qs, ks, vs, m, d, dv, scale, os);                                                        \
      /* scatter_rows: dest row += src row (0 + x), so -0.0 becomes +0.0. */                                 \
      for (int64_t t = 0; t < m; ++t)                                                                        \
        for (int64_t c = 0; c < dv; ++c) out[rows[t] * dv + c] += os[t * dv + c];                            \
    }                                                                                                        \
    free(qs);                                                                                                \
    free(ks);                                                                                                \
    free(vs);                                                                                                \
    free(os);                                                                                                \
    free(rows);                                                                                              \
    return ORC_OK;                                                                                           \
  }

DFA_ORACLE_BODY(float, f32, sqrtf, expf)
DFA_ORACLE_BODY(double, f64, sqrt, exp)

/* oracles.hpp:67-107: dense N x N attention, -inf outside each row's view,
 * rows kept by no view are 0. */
int oracle_masked_dense_f64(const double* q, const double* k, const double* v, int64_t n, int64_t d, int64_t dv,
                            int64_t w, int64_t r, int64_t gamma, int32_t scale, double* out) {
  const int64_t off = gamma;
  if (oracle_validate(n, w, r, 1, d, &off, 1, 0, 1, 0) != ORC_OK) return ORC_ERR_CONFIG;
  int64_t* group = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) group[i] = -1;
  const int64_t n_seg = (n + w - 1) / w;
  for (int64_t i = 0; i < n_seg; ++i)
    for (int64_t row = i * w + gamma; row < ((i + 1) * w < n ? (i + 1) * w : n); row += r) group[row] = i;
  const double sc = scale ? 1.0 / sqrt((double)d) : 1.0;
  double* s = (double*)malloc(sizeof(double) * (size_t)n);
  memset(out, 0, sizeof(double) * (size_t)(n * dv));
  for (int64_t i = 0; i < n; ++i) {
    if (group[i] < 0) continue;
    double m = -INFINITY;
    for (int64_t j = 0; j < n; ++j) {
      s[j] = -INFINITY;
      if (group[j] != group[i]) continue;
      double acc = 0;
      for (int64_t c = 0; c < d; ++c) acc += q[i * d + c] * k[j * d + c];
      s[j] = acc * sc;
      m = (m < s[j]) ? s[j] : m;
    }
    double z = 0;
    for (int64_t j = 0; j < n; ++j) {
      if (s[j] == -INFINITY) {
        s[j] = 0;
        continue;
      }
      s[j] = exp(s[j] - m);
      z += s[j];
    }
    for (int64_t c = 0; c < dv; ++c) {
      double acc = 0;
      for (int64_t j = 0; j < n; ++j) acc += s[j] * v[j * dv + c];
      out[i * dv + c] = acc / z;
    }
  }
  free(s);
  free(group);
  return ORC_OK;
}

/* EXTENSION (no reference code).  For one (w, r, gamma) branch: lse[row] =
 * ln(sum_j exp(s_j)) over the row's view, s = (q.k) * scale; rows kept by no
 * view get -inf.  Natural log, matching the kernel's optional LSE output. */
int oracle_dilated_lse_f64(const double* q, const double* k, int64_t n, int64_t d, int64_t w, int64_t r,
                           int64_t gamma, int32_t scale, double* lse) {
  const int64_t off = gamma;
  if (oracle_validate(n, w, r, 1, d, &off, 1, 0, 1, 0) != ORC_OK) return ORC_ERR_CONFIG;
  const double sc = scale ? 1.0 / sqrt((double)d) : 1.0;
  for (int64_t i = 0; i < n; ++i) lse[i] = -INFINITY;
  const int64_t n_seg = (n + w - 1) / w;
  for (int64_t i = 0; i < n_seg; ++i) {
    const int64_t end = (i + 1) * w < n ? (i + 1) * w : n;
    for (int64_t a = i * w + gamma; a < end; a += r) {
      double mx = -INFINITY;
      for (int64_t b = i * w + gamma; b < end; b += r) {
        double acc = 0;
        for (int64_t c = 0; c < d; ++c) acc += q[a * d + c] * k[b * d + c];
        mx = fmax(mx, acc * sc);
      }
      double z = 0;
      for (int64_t b = i * w + gamma; b < end; b += r) {
        double acc = 0;
        for (int64_t c = 0; c < d; ++c) acc += q[a * d + c] * k[b * d + c];
        z += exp(acc * sc - mx);
      }
      lse[a] = mx + log(z);
    }
  }
  return ORC_OK;
}

/* EXTENSION (no reference code).  nb branches (ws[b], rs[b], gs[b]).  For each
 * query row, gather the keys of every branch whose view contains the row (a
 * key selected by two branches counts twice), take one dense softmax over that
 * multiset, and weight v accordingly.  Algebraically this equals
 *   O = sum_b exp(lse_b) O_b / sum_b exp(lse_b)
 * over the covering branches (the kernel's LSE combine), so it checks the
 * combine without sharing its arithmetic.  Rows covered by no branch are 0;
 * lse_out (optional) receives ln(sum over the multiset). */
int oracle_multibranch_f64(const double* q, const double* k, const double* v, int64_t n, int64_t d, int64_t dv,
                           int64_t nb, const int64_t* ws, const int64_t* rs, const int64_t* gs, int32_t scale,
                           double* out, double* lse_out) {
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t off = gs[b];
    if (oracle_validate(n, ws[b], rs[b], 1, d, &off, 1, 0, 1, 0) != ORC_OK) return ORC_ERR_CONFIG;
  }
  const double sc = scale ? 1.0 / sqrt((double)d) : 1.0;
  int64_t cap = 0;
  for (int64_t b = 0; b < nb; ++b) cap += (ws[b] + rs[b] - 1) / rs[b];
  int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  double* s = (double*)malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
  memset(out, 0, sizeof(double) * (size_t)(n * dv));
  for (int64_t a = 0; a < n; ++a) {
    int64_t nk = 0;
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t i = a / ws[b];
      const int64_t begin = i * ws[b];
      const int64_t end = begin + ws[b] < n ? begin + ws[b] : n;
      if ((a - begin) % rs[b] != gs[b] % rs[b] || a - begin < gs[b]) continue;
      for (int64_t row = begin + gs[b]; row < end; row += rs[b]) keys[nk++] = row;
    }
    if (lse_out) lse_out[a] = -INFINITY;
    if (nk == 0) continue;
    double mx = -INFINITY;
    for (int64_t t = 0; t < nk; ++t) {
      double acc = 0;
      for (int64_t c = 0; c < d; ++c) acc += q[a * d + c] * k[keys[t] * d + c];
      s[t] = acc * sc;
      mx = fmax(mx, s[t]);
    }
    double z = 0;
    for (int64_t t = 0; t < nk; ++t) {
      s[t] = exp(s[t] - mx);
      z += s[t];
    }
    for (int64_t c = 0; c < dv; ++c) {
      double acc = 0;
      for (int64_t t = 0; t < nk; ++t) acc += s[t] * v[keys[t] * dv + c];
      out[a * dv + c] = acc / z;
    }
    if (lse_out) lse_out[a] = mx + log(z);
  }
  free(keys);
  free(s);
  return ORC_OK;
}

/* CPU "port" baseline timing: `units` forwards of oracle_dilated_attention_f32
 * (N, w, r, d; gamma = unit % r) on one thread over `distinct` input sets
 * supplied by the caller (q,k,v each distinct*n*d floats).  Returns seconds. */
#include <time.h>
double oracle_time_dilated_f32(const float* q, const float* k, const float* v, int64_t n, int64_t w, int64_t r,
                               int64_t d, int64_t units, int64_t distinct, float* scratch_out) {
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int64_t u = 0; u < units; ++u) {
    const int64_t s = u % distinct;
    oracle_dilated_attention_f32(q + s * n * d, k + s * n * d, v + s * n * d, n, d, d, w, r, u % r, 1, 0, 1,
                                 scratch_out);
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

/* Backward of the dilated core: gradients of
 * loss = sum(O * dO) w.r.t. q, k, v for one head at offset gamma, as the
 * reference's tape computes them for the dilated branch of
 * detail::attention_mix (encoder.hpp:204-219): per segment view,
 *   S = (Qs Ks^T) * sc            ag::scale(ag::matmul)    autodiff.hpp:99-137
 *   P = softmax_rows(S)           autodiff.hpp:166-179: dS = P o (dP - rowsum(dP o P))
 *   Os = P Vs                     matmul backward: dP = dO Vs^T, dVs = P^T dO
 * and slice_rows_strided / scatter_rows (:269-289) route the row gradients
 * back to the global rows; rows no view selects get 0.  f64 throughout.
 * sc = 1/sqrt(d) when `scale` (attention_mix always scales). */
int oracle_dilated_backward_f64(const double* q, const double* k, const double* v, const double* dout, int64_t n,
                                int64_t d, int64_t dv, int64_t w, int64_t r, int64_t gamma, int32_t scale,
                                double* dq, double* dk, double* dvo) {
  const int64_t off = gamma;
  if (oracle_validate(n, w, r, 1, d, &off, 1, 0, 1, 0) != ORC_OK) return ORC_ERR_CONFIG;
  if (gamma < 0 || gamma >= r) return ORC_ERR_OUT_OF_RANGE;
  const double sc = scale ? 1.0 / sqrt((double)d) : 1.0;
  const int64_t n_seg = (n + w - 1) / w, mmax = (w + r - 1) / r;
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)mmax);
  double* P = (double*)malloc(sizeof(double) * (size_t)(mmax * mmax));
  double* dP = (double*)malloc(sizeof(double) * (size_t)(mmax * mmax));
  memset(dq, 0, sizeof(double) * (size_t)(n * d));
  memset(dk, 0, sizeof(double) * (size_t)(n * d));
  memset(dvo, 0, sizeof(double) * (size_t)(n * dv));
  for (int64_t s = 0; s < n_seg; ++s) {
    int64_t m = 0;
    oracle_segment_view(n, w, r, s, gamma, rows, mmax, &m);
    if (m == 0) continue;
    for (int64_t i = 0; i < m; ++i) {
      const double* qi = q + rows[i] * d;
      double mx = -INFINITY;
      for (int64_t j = 0; j < m; ++j) {
        const double* kj = k + rows[j] * d;
        double acc = 0;
        for (int64_t c = 0; c < d; ++c) acc += qi[c] * kj[c];
        P[i * m + j] = acc * sc;
        mx = P[i * m + j] > mx ? P[i * m + j] : mx;
      }
      double sum = 0;
      for (int64_t j = 0; j < m; ++j) {
        P[i * m + j] = exp(P[i * m + j] - mx);
        sum += P[i * m + j];
      }
      for (int64_t j = 0; j < m; ++j) P[i * m + j] /= sum;
    }
    for (int64_t i = 0; i < m; ++i) {
      const double* gi = dout + rows[i] * dv;
      double dot = 0;
      for (int64_t j = 0; j < m; ++j) {
        const double* vj = v + rows[j] * dv;
        double acc = 0;
        for (int64_t c = 0; c < dv; ++c) acc += gi[c] * vj[c];
        dP[i * m + j] = acc;
        dot += acc * P[i * m + j];
      }
      for (int64_t j = 0; j < m; ++j) dP[i * m + j] = P[i * m + j] * (dP[i * m + j] - dot) * sc; /* dS * sc */
    }
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < m; ++j) {
        const double pij = P[i * m + j], sij = dP[i * m + j];
        for (int64_t c = 0; c < dv; ++c) dvo[rows[j] * dv + c] += pij * dout[rows[i] * dv + c];
        for (int64_t c = 0; c < d; ++c) {
          dq[rows[i] * d + c] += sij * k[rows[j] * d + c];
          dk[rows[j] * d + c] += sij * q[rows[i] * d + c];
        }
      }
  }
  free(rows);
  free(P);
  free(dP);
  return ORC_OK;
}

/* ------------------------------------------------------------------------
 * Batched, threaded drivers (test infrastructure): the multi-head layout
 * [B, N, h, d] of the device API, one (image, head) unit per task over a
 * pool of pthreads.  Each unit calls the single-head restatement above on
 * the head's column block, so the arithmetic is exactly the pinned port's
 * (attention.hpp:280-301 per head, the multi-head concat of :350-357). */
#include <pthread.h>
#include <stdatomic.h>

typedef struct {
  const double *q, *k, *v;
  int64_t B, n, h, d, dv, w, r, nb;
  const int64_t *offsets; /* [h] (single branch) or [nb * h] */
  const int64_t *ws, *rs; /* [nb] (multibranch) */
  double *out, *lse;
  atomic_long next;
  atomic_int status;
  int multibranch;
} orc_batch_t;

static void* orc_batch_worker(void* arg) {
  orc_batch_t* t = (orc_batch_t*)arg;
  const int64_t n = t->n, d = t->d, dv = t->dv, h = t->h;
  double* qs = (double*)malloc(sizeof(double) * (size_t)(n * d));
  double* ks = (double*)malloc(sizeof(double) * (size_t)(n * d));
  double* vs = (double*)malloc(sizeof(double) * (size_t)(n * dv));
  double* os = (double*)malloc(sizeof(double) * (size_t)(n * dv));
  double* ls = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t gs[64];
  for (;;) {
    const long u = atomic_fetch_add(&t->next, 1);
    if (u >= t->B * h) break;
    const int64_t b = u / h, j = u % h;
    for (int64_t a = 0; a < n; ++a) {
      memcpy(qs + a * d, t->q + ((b * n + a) * h + j) * d, sizeof(double) * (size_t)d);
      memcpy(ks + a * d, t->k + ((b * n + a) * h + j) * d, sizeof(double) * (size_t)d);
      memcpy(vs + a * dv, t->v + ((b * n + a) * h + j) * dv, sizeof(double) * (size_t)dv);
    }
    int st;
    if (t->multibranch) {
      for (int64_t e = 0; e < t->nb; ++e) gs[e] = t->offsets[e * h + j];
      st = oracle_multibranch_f64(qs, ks, vs, n, d, dv, t->nb, t->ws, t->rs, gs, 1, os, ls);
    } else {
      st = oracle_dilated_attention_f64(qs, ks, vs, n, d, dv, t->w, t->r, t->offsets[j], 1, 0, 1, os);
    }
    if (st != ORC_OK) {
      atomic_store(&t->status, st);
      break;
    }
    for (int64_t a = 0; a < n; ++a) {
      memcpy(t->out + ((b * n + a) * h + j) * dv, os + a * dv, sizeof(double) * (size_t)dv);
      if (t->multibranch && t->lse) t->lse[(b * h + j) * n + a] = ls[a];
    }
  }
  free(qs);
  free(ks);
  free(vs);
  free(os);
  free(ls);
  return NULL;
}

static int orc_batch_run(orc_batch_t* t, int32_t threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t pool[256];
  atomic_init(&t->next, 0);
  atomic_init(&t->status, ORC_OK);
  for (int32_t i = 0; i < threads; ++i) pthread_create(&pool[i], NULL, orc_batch_worker, t);
  for (int32_t i = 0; i < threads; ++i) pthread_join(pool[i], NULL);
  return atomic_load(&t->status);
}

/* dilated_attention (f64, naive kernel) for every (image, head) of [B, N, h, d]. */
int oracle_dilated_batched_f64(const double* q, const double* k, const double* v, int64_t B, int64_t n, int64_t h,
                               int64_t d, int64_t dv, int64_t w, int64_t r, const int64_t* offsets, int32_t threads,
                               double* out) {
  orc_batch_t t;
  memset(&t, 0, sizeof(t));
  t.q = q, t.k = k, t.v = v, t.B = B, t.n = n, t.h = h, t.d = d, t.dv = dv, t.w = w, t.r = r;
  t.offsets = offsets, t.out = out;
  return orc_batch_run(&t, threads);
}

/* oracle_multibranch_f64 for every (image, head); offsets [nb * h]
 * (branch-major), lse (optional) [B, h, N]. */
int oracle_multibranch_batched_f64(const double* q, const double* k, const double* v, int64_t B, int64_t n,
                                   int64_t h, int64_t d, int64_t dv, int64_t nb, const int64_t* ws, const int64_t* rs,
                                   const int64_t* offsets, int32_t threads, double* out, double* lse) {
  if (nb < 1 || nb > 64) return ORC_ERR_CONFIG;
  orc_batch_t t;
  memset(&t, 0, sizeof(t));
  t.q = q, t.k = k, t.v = v, t.B = B, t.n = n, t.h = h, t.d = d, t.dv = dv, t.nb = nb;
  t.ws = ws, t.rs = rs, t.offsets = offsets, t.out = out, t.lse = lse, t.multibranch = 1;
  return orc_batch_run(&t, threads);
}
