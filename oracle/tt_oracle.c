/* TEST INFRASTRUCTURE ONLY -- see tt_oracle.h.  Plain-C restatement of the
 * reference's serial TT-EmbeddingBag algorithm; every loop nest keeps the
 * reference's operation order (mul then add, no FMA -- compiled with
 * -ffp-contract=off) so results are bit-identical to the reference. */
#include "tt_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define MAXD 8

/* tt_table.hpp:71-78 decompose_row: q = flat / row_suffix[k]; flat -= q*row_suffix[k]. */
void tto_decompose_row(int64_t flat, int d, const int64_t* rf, int64_t* dig) {
  int64_t suffix[MAXD];
  suffix[d - 1] = 1;
  for (int k = d - 2; k >= 0; --k) suffix[k] = suffix[k + 1] * rf[k + 1];
  for (int k = 0; k < d; ++k) {
    const int64_t q = flat / suffix[k];
    dig[k] = q;
    flat -= q * suffix[k];
  }
}

/* index_batch.hpp:41-56 IndexBatch::validate (weights count is the caller's job). */
int tto_validate(int64_t num_rows, const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                 int64_t* bad) {
  if (off[0] != 0) return 2;
  for (int64_t b = 0; b < B; ++b)
    if (off[b] > off[b + 1]) return 2;
  if (off[B] != L) return 2;
  for (int64_t t = 0; t < L; ++t)
    if (idx[t] < 0 || idx[t] >= num_rows) {
      if (bad) *bad = t;
      return 3;
    }
  return 0;
}

static int64_t slice_size(int k, const int64_t* cf, const int64_t* rk) {
  return rk[k] * cf[k] * rk[k + 1];
}

static int64_t max_width(int d, const int64_t* cf, const int64_t* rk) {
  int64_t p = 1, mw = 0;
  for (int k = 0; k < d; ++k) {
    p *= cf[k];
    const int64_t w = p * rk[k + 1];
    if (w > mw) mw = w;
  }
  /* the backward D buffers also hold prefix[k-1]*R_k values (<= width[k-1]) */
  return mw;
}

#define DEFINE_ORACLE(T, SFX)                                                                   \
  /* embedding_ops.hpp:382-423 ref::forward_bags */                                             \
  int tto_forward_##SFX(int d, int64_t num_rows, int64_t emb, const int64_t* rf,                \
                        const int64_t* cf, const int64_t* rk, const T* const* cores,            \
                        const int64_t* idx, int64_t L, const int64_t* off, int64_t B,           \
                        const double* w, int pooling, T* out) {                                 \
    int64_t bad = 0;                                                                            \
    const int st = tto_validate(num_rows, idx, L, off, B, &bad);                                \
    if (st) return st;                                                                          \
    const int64_t mw = max_width(d, cf, rk);                                                    \
    T* cur = (T*)malloc(sizeof(T) * (mw + 1));                                                  \
    T* nxt = (T*)malloc(sizeof(T) * (mw + 1));                                                  \
    int64_t dig[MAXD];                                                                          \
    memset(out, 0, sizeof(T) * B * emb);                                                        \
    for (int64_t b = 0; b < B; ++b) {                                                           \
      T* orow = out + b * emb;                                                                  \
      for (int64_t t = off[b]; t < off[b + 1]; ++t) {                                           \
        tto_decompose_row(idx[t], d, rf, dig);                                                  \
        int64_t rows = cf[0];                                                                   \
        const int64_t s0 = slice_size(0, cf, rk);                                               \
        memcpy(cur, cores[0] + dig[0] * s0, sizeof(T) * s0);                                    \
        for (int k = 1; k < d; ++k) {                                                           \
          const int64_t r = rk[k], wk = cf[k] * rk[k + 1];                                      \
          const T* sl = cores[k] + dig[k] * slice_size(k, cf, rk);                              \
          for (int64_t e = 0; e < rows * wk; ++e) nxt[e] = (T)0;                                \
          for (int64_t i = 0; i < rows; ++i)                                                    \
            for (int64_t p = 0; p < r; ++p) {                                                   \
              const T a = cur[i * r + p];                                                       \
              const T* srow = sl + p * wk;                                                      \
              for (int64_t j = 0; j < wk; ++j) nxt[i * wk + j] += a * srow[j];                  \
            }                                                                                   \
          T* tmp = cur;                                                                         \
          cur = nxt;                                                                            \
          nxt = tmp;                                                                            \
          rows *= cf[k];                                                                        \
        }                                                                                       \
        const T alpha = (T)(w ? w[t] : 1.0);                                                    \
        for (int64_t j = 0; j < emb; ++j) orow[j] += alpha * cur[j];                            \
      }                                                                                         \
      if (pooling == 1) {                                                                       \
        const int64_t sz = off[b + 1] - off[b];                                                 \
        if (sz > 1) {                                                                           \
          const T inv = (T)(1.0 / (double)sz);                                                  \
          for (int64_t j = 0; j < emb; ++j) orow[j] *= inv;                                     \
        }                                                                                       \
      }                                                                                         \
    }                                                                                           \
    free(cur);                                                                                  \
    free(nxt);                                                                                  \
    return 0;                                                                                   \
  }                                                                                             \
                                                                                                \
  /* one lookup of embedding_ops.hpp:426-490 ref::backward_bags; u[k] scratch of mw each */     \
  static void bwd_lookup_##SFX(int d, int64_t emb, const int64_t* rf, const int64_t* cf,        \
                               const int64_t* rk, const T* const* cores, int64_t row,           \
                               double alpha, const T* grow, T* const* grads, T* u, T* dcur,     \
                               T* dnxt, int64_t mw) {                                           \
    int64_t dig[MAXD];                                                                          \
    int64_t prefix[MAXD];                                                                       \
    tto_decompose_row(row, d, rf, dig);                                                         \
    int64_t p = 1;                                                                              \
    for (int k = 0; k < d; ++k) {                                                               \
      p *= cf[k];                                                                               \
      prefix[k] = p;                                                                            \
    }                                                                                           \
    const int64_t s0 = slice_size(0, cf, rk);                                                   \
    memcpy(u, cores[0] + dig[0] * s0, sizeof(T) * s0);                                          \
    for (int k = 1; k < d; ++k) {                                                               \
      const int64_t pk = prefix[k - 1], r = rk[k], wk = cf[k] * rk[k + 1];                      \
      const T* sl = cores[k] + dig[k] * slice_size(k, cf, rk);                                  \
      T* uk = u + k * mw;                                                                       \
      const T* up = u + (k - 1) * mw;                                                           \
      for (int64_t e = 0; e < pk * wk; ++e) uk[e] = (T)0;                                       \
      for (int64_t i = 0; i < pk; ++i)                                                          \
        for (int64_t q = 0; q < r; ++q) {                                                       \
          const T a = up[i * r + q];                                                            \
          const T* srow = sl + q * wk;                                                          \
          for (int64_t j = 0; j < wk; ++j) uk[i * wk + j] += a * srow[j];                       \
        }                                                                                       \
    }                                                                                           \
    {                                                                                           \
      const T a = (T)alpha;                                                                     \
      for (int64_t j = 0; j < emb; ++j) dcur[j] = a * grow[j];                                  \
    }                                                                                           \
    for (int k = d - 1; k >= 1; --k) {                                                          \
      const int64_t pk = prefix[k - 1], r = rk[k], wk = cf[k] * rk[k + 1];                      \
      T* gs = grads[k] + dig[k] * slice_size(k, cf, rk);                                        \
      const T* up = u + (k - 1) * mw;                                                           \
      for (int64_t i = 0; i < pk; ++i)                                                          \
        for (int64_t q = 0; q < r; ++q) {                                                       \
          const T a = up[i * r + q];                                                            \
          for (int64_t j = 0; j < wk; ++j) gs[q * wk + j] += a * dcur[i * wk + j];              \
        }                                                                                       \
      const T* sl = cores[k] + dig[k] * slice_size(k, cf, rk);                                  \
      for (int64_t i = 0; i < pk; ++i)                                                          \
        for (int64_t q = 0; q < r; ++q) {                                                       \
          T acc = (T)0;                                                                         \
          for (int64_t j = 0; j < wk; ++j) acc += dcur[i * wk + j] * sl[q * wk + j];            \
          dnxt[i * r + q] = acc;                                                                \
        }                                                                                       \
      T* tmp = dcur;                                                                            \
      dcur = dnxt;                                                                              \
      dnxt = tmp;                                                                               \
    }                                                                                           \
    T* g0 = grads[0] + dig[0] * s0;                                                             \
    for (int64_t j = 0; j < s0; ++j) g0[j] += dcur[j];                                          \
  }                                                                                             \
                                                                                                \
  int tto_backward_##SFX(int d, int64_t num_rows, int64_t emb, const int64_t* rf,               \
                         const int64_t* cf, const int64_t* rk, const T* const* cores,           \
                         const int64_t* idx, int64_t L, const int64_t* off, int64_t B,          \
                         const double* w, int pooling, const T* grad_out, T* const* grads) {    \
    int64_t bad = 0;                                                                            \
    const int st = tto_validate(num_rows, idx, L, off, B, &bad);                                \
    if (st) return st;                                                                          \
    for (int k = 0; k < d; ++k)                                                                 \
      memset(grads[k], 0, sizeof(T) * rf[k] * slice_size(k, cf, rk));                           \
    const int64_t mw = max_width(d, cf, rk) + 1;                                                \
    T* u = (T*)malloc(sizeof(T) * mw * d);                                                      \
    T* dcur = (T*)malloc(sizeof(T) * mw);                                                       \
    T* dnxt = (T*)malloc(sizeof(T) * mw);                                                       \
    for (int64_t b = 0; b < B; ++b)                                                             \
      for (int64_t t = off[b]; t < off[b + 1]; ++t) {                                           \
        double alpha = w ? w[t] : 1.0;                                                          \
        if (pooling == 1) alpha /= (double)(off[b + 1] - off[b]);                               \
        bwd_lookup_##SFX(d, emb, rf, cf, rk, cores, idx[t], alpha, grad_out + b * emb, grads,   \
                         u, dcur, dnxt, mw);                                                    \
      }                                                                                         \
    free(u);                                                                                    \
    free(dcur);                                                                                 \
    free(dnxt);                                                                                 \
    return 0;                                                                                   \
  }                                                                                             \
                                                                                                \
  /* embedding_ops.hpp:361-376 sgd_step: c -= T(lr) * g */                                      \
  void tto_sgd_##SFX(int d, const int64_t* rf, const int64_t* cf, const int64_t* rk,            \
                     T* const* cores, const T* const* grads, double lr) {                       \
    const T step = (T)lr;                                                                       \
    for (int k = 0; k < d; ++k) {                                                               \
      const int64_t n = rf[k] * slice_size(k, cf, rk);                                          \
      for (int64_t i = 0; i < n; ++i) cores[k][i] -= step * grads[k][i];                        \
    }                                                                                           \
  }                                                                                             \
                                                                                                \
  /* embedding_ops.hpp:120-152 lookup_row (matmul zero-fill then i,p,j) */                      \
  int tto_lookup_row_##SFX(int d, int64_t num_rows, int64_t emb, const int64_t* rf,             \
                           const int64_t* cf, const int64_t* rk, const T* const* cores,         \
                           int64_t row, T* out) {                                               \
    if (row < 0 || row >= num_rows) return 3;                                                   \
    int64_t off[2] = {0, 1};                                                                    \
    return tto_forward_##SFX(d, num_rows, emb, rf, cf, rk, cores, &row, 1, off, 1, 0, 0, out);  \
  }

DEFINE_ORACLE(float, f32)
DEFINE_ORACLE(double, f64)

/* Parallel CPU step (forward over bag ranges, backward with per-worker dense
 * gradients merged in worker order, then SGD) -- the reference's OpenMP
 * structure (embedding_ops.hpp:187-191, 280-287, 355-357, 372). */
double tto_time_step_f32(int d, int64_t num_rows, int64_t emb, const int64_t* rf,
                         const int64_t* cf, const int64_t* rk, float* const* cores,
                         const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                         const float* grad_out, double lr, int threads) {
  if (threads > 0) omp_set_num_threads(threads);
  const int W = omp_get_max_threads();
  int64_t csz[MAXD], total = 0;
  for (int k = 0; k < d; ++k) {
    csz[k] = rf[k] * slice_size(k, cf, rk);
    total += csz[k];
  }
  float* out = (float*)malloc(sizeof(float) * (B * emb + 1));
  float* gbuf = (float*)calloc((size_t)W * total + 1, sizeof(float));
  const int64_t mw = max_width(d, cf, rk) + 1;
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
#pragma omp parallel num_threads(W)
  {
    const int wid = omp_get_thread_num();
    const int64_t lo = B * wid / W, hi = B * (wid + 1) / W;
    float* u = (float*)malloc(sizeof(float) * mw * d);
    float* dc = (float*)malloc(sizeof(float) * mw);
    float* dn = (float*)malloc(sizeof(float) * mw);
    float* g[MAXD];
    float* base = gbuf + (size_t)wid * total;
    memset(base, 0, sizeof(float) * total);
    for (int k = 0, o = 0; k < d; o += (int)csz[k], ++k) g[k] = base + o;
    const float* cc[MAXD];
    for (int k = 0; k < d; ++k) cc[k] = cores[k];
    for (int64_t b = lo; b < hi; ++b) {
      int64_t o2[2] = {0, off[b + 1] - off[b]};
      tto_forward_f32(d, num_rows, emb, rf, cf, rk, cc, idx + off[b], o2[1], o2, 1, 0, 0,
                      out + b * emb);
    }
    for (int64_t b = lo; b < hi; ++b)
      for (int64_t t = off[b]; t < off[b + 1]; ++t)
        bwd_lookup_f32(d, emb, rf, cf, rk, cc, idx[t], 1.0, grad_out + b * emb, g, u, dc, dn,
                       mw);
    free(u);
    free(dc);
    free(dn);
  }
  for (int wk = 1; wk < W; ++wk)
    for (int64_t i = 0; i < total; ++i) gbuf[i] += gbuf[(size_t)wk * total + i];
  {
    const float step = (float)lr;
    int64_t o = 0;
    for (int k = 0; k < d; ++k) {
      for (int64_t i = 0; i < csz[k]; ++i) cores[k][i] -= step * gbuf[o + i];
      o += csz[k];
    }
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  free(out);
  free(gbuf);
  return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}
