/*
 * gm_oracle.c — plain-C restatement of the reference hot path.
 * TEST INFRASTRUCTURE ONLY (see gm_oracle.h). Each function cites the
 * reference lines it restates (paths relative to /root/reference/proj).
 */
#include "gm_oracle.h"

#include <stdlib.h>
#include <string.h>
#include <math.h>

/* edge_index.cpp:45-62 */
void or_build_compressed(const int64_t* keys, const int64_t* values, int64_t e, int64_t num_rows,
                         int64_t* rowptr, int64_t* col, int64_t* perm) {
  memset(rowptr, 0, sizeof(int64_t) * (size_t)(num_rows + 1));
  for (int64_t i = 0; i < e; ++i) ++rowptr[keys[i] + 1];
  for (int64_t r = 0; r < num_rows; ++r) rowptr[r + 1] += rowptr[r];
  int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)(num_rows > 0 ? num_rows : 1));
  memcpy(cursor, rowptr, sizeof(int64_t) * (size_t)num_rows);
  for (int64_t i = 0; i < e; ++i) {
    const int64_t pos = cursor[keys[i]]++;
    col[pos] = values[i];
    perm[pos] = i;
  }
  free(cursor);
}

/* message_passing.hpp:62-84 — per destination row, ascending CSC position,
 * `o[j] += w * xi[j]` (weighted) or `o[j] += xi[j]`, then `*= S(1)/S(deg)`. */
#define DEFINE_SPMM(SUF, S)                                                                   \
  void or_spmm_##SUF(const int64_t* rowptr, const int64_t* col, const int64_t* perm,          \
                     int64_t n_rows, const S* x, int64_t f, const S* w, int mean,             \
                     const int64_t* rows, int64_t n_list, S* out) {                           \
    const int64_t count = rows ? n_list : n_rows;                                             \
    for (int64_t i = 0; i < count; ++i) {                                                     \
      const int64_t v = rows ? rows[i] : i;                                                   \
      S* o = out + i * f;                                                                     \
      for (int64_t j = 0; j < f; ++j) o[j] = (S)0;                                            \
      for (int64_t k = rowptr[v]; k < rowptr[v + 1]; ++k) {                                   \
        const S* xi = x + col[k] * f;                                                         \
        if (w) {                                                                              \
          const S wk = w[perm[k]];                                                            \
          for (int64_t j = 0; j < f; ++j) o[j] += wk * xi[j];                                 \
        } else {                                                                              \
          for (int64_t j = 0; j < f; ++j) o[j] += xi[j];                                      \
        }                                                                                     \
      }                                                                                       \
      const int64_t deg = rowptr[v + 1] - rowptr[v];                                          \
      if (mean && deg > 0) {                                                                  \
        const S inv = (S)1 / (S)deg;                                                          \
        for (int64_t j = 0; j < f; ++j) o[j] *= inv;                                          \
      }                                                                                       \
    }                                                                                         \
  }
DEFINE_SPMM(f32, float)
DEFINE_SPMM(f64, double)

/* message_passing.hpp:51-59 (+ mean 76-84): COO sweep for undirected+weights. */
#define DEFINE_SPMM_COO(SUF, S)                                                               \
  void or_spmm_coo_##SUF(const int64_t* src, const int64_t* dst, int64_t e, int64_t n_dst,    \
                         const S* x, int64_t f, const S* w, int mean, S* out) {               \
    memset(out, 0, sizeof(S) * (size_t)(n_dst * f));                                          \
    for (int64_t i = 0; i < e; ++i) {                                                         \
      S* o = out + dst[i] * f;                                                                \
      const S* xi = x + src[i] * f;                                                           \
      const S wi = w[i];                                                                      \
      for (int64_t j = 0; j < f; ++j) o[j] += wi * xi[j];                                     \
    }                                                                                         \
    if (mean) {                                                                               \
      int64_t* deg = (int64_t*)calloc((size_t)(n_dst > 0 ? n_dst : 1), sizeof(int64_t));      \
      for (int64_t i = 0; i < e; ++i) ++deg[dst[i]];                                          \
      for (int64_t v = 0; v < n_dst; ++v)                                                     \
        if (deg[v] > 0) {                                                                     \
          const S inv = (S)1 / (S)deg[v];                                                     \
          for (int64_t j = 0; j < f; ++j) out[v * f + j] *= inv;                              \
        }                                                                                     \
      free(deg);                                                                              \
    }                                                                                         \
  }
DEFINE_SPMM_COO(f32, float)
DEFINE_SPMM_COO(f64, double)

/* aggregate.hpp:197-215 over the grouped order of message_passing.hpp:190-214:
 * `better = ap < 0 || v > cur` (v < cur for min); argpos mapped through perm. */
#define DEFINE_MAX(SUF, S)                                                                    \
  void or_spmm_max_##SUF(const int64_t* rowptr, const int64_t* col, const int64_t* perm,      \
                         int64_t n_rows, const S* x, int64_t f, const S* w, int is_min,       \
                         const int64_t* rows, int64_t n_list, S* out, int64_t* arg) {         \
    const int64_t count = rows ? n_list : n_rows;                                             \
    for (int64_t i = 0; i < count; ++i) {                                                     \
      const int64_t v = rows ? rows[i] : i;                                                   \
      S* o = out + i * f;                                                                     \
      int64_t* a = arg + i * f;                                                               \
      for (int64_t j = 0; j < f; ++j) {                                                       \
        o[j] = (S)0;                                                                          \
        a[j] = -1;                                                                            \
      }                                                                                       \
      for (int64_t k = rowptr[v]; k < rowptr[v + 1]; ++k) {                                   \
        const S* xi = x + col[k] * f;                                                         \
        const S wk = w ? w[perm[k]] : (S)1;                                                   \
        for (int64_t j = 0; j < f; ++j) {                                                     \
          const S val = w ? xi[j] * wk : xi[j];                                               \
          const int better = a[j] < 0 || (is_min ? val < o[j] : val > o[j]);                  \
          if (better) {                                                                       \
            o[j] = val;                                                                       \
            a[j] = perm[k];                                                                   \
          }                                                                                   \
        }                                                                                     \
      }                                                                                       \
    }                                                                                         \
  }
DEFINE_MAX(f32, float)
DEFINE_MAX(f64, double)

/* Backward of the max/min path (aggregate.hpp:295-308 then the gather_rows
 * adjoint tensor.hpp:510-524): the gradient of output (v, j) lands on the
 * grouped position whose COO edge id is arg[v][j], and gather_rows' adjoint
 * adds every grouped position's row into dx[src] in ascending grouped (CSC)
 * order, starting from +0. Positions that did not win add exact zeros, which
 * never change a sum that starts at +0 under round-to-nearest, so only the
 * winners are added here. rowptr/col/perm: the CSC (destination grouping). */
#define DEFINE_MAX_BWD(SUF, S)                                                                 \
  void or_spmm_max_backward_##SUF(const int64_t* rowptr, const int64_t* col, const int64_t* perm,   \
                                  int64_t n_rows, const int64_t* arg, const S* g, int64_t f,        \
                                  int64_t n_src, S* dx) {                                           \
    for (int64_t i = 0; i < n_src * f; ++i) dx[i] = (S)0;                                        \
    for (int64_t v = 0; v < n_rows; ++v)                                                         \
      for (int64_t k = rowptr[v]; k < rowptr[v + 1]; ++k) {                                      \
        S* d = dx + col[k] * f;                                                                  \
        for (int64_t j = 0; j < f; ++j)                                                          \
          if (arg[v * f + j] == perm[k]) d[j] = d[j] + g[v * f + j];                             \
      }                                                                                          \
  }
DEFINE_MAX_BWD(f32, float)
DEFINE_MAX_BWD(f64, double)

/* message_passing.hpp:437-463 */
#define DEFINE_GCN_NORM(SUF, S, SQRT)                                                         \
  void or_gcn_norm_##SUF(const int64_t* base_src, const int64_t* base_dst, int64_t base_len,  \
                         int64_t n_src, int64_t n_dst, const int64_t* g_src,                  \
                         const int64_t* g_dst, int64_t g_len, int square, S* norm) {          \
    int64_t* din = (int64_t*)calloc((size_t)(n_dst > 0 ? n_dst : 1), sizeof(int64_t));       \
    for (int64_t i = 0; i < base_len; ++i)                                                    \
      if (base_dst[i] < n_dst) ++din[base_dst[i]];                                            \
    if (square) {                                                                             \
      for (int64_t v = 0; v < n_dst; ++v) din[v] += 1;                                        \
      for (int64_t i = 0; i < g_len; ++i)                                                     \
        norm[i] = (S)1 / SQRT((S)din[g_src[i]] * (S)din[g_dst[i]]);                           \
    } else {                                                                                  \
      int64_t* dout = (int64_t*)calloc((size_t)(n_src > 0 ? n_src : 1), sizeof(int64_t));    \
      for (int64_t i = 0; i < base_len; ++i)                                                  \
        if (base_src[i] < n_src) ++dout[base_src[i]];                                         \
      for (int64_t i = 0; i < g_len; ++i) {                                                   \
        const int64_t da = dout[g_src[i]] > 1 ? dout[g_src[i]] : 1;                           \
        const int64_t db = din[g_dst[i]] > 1 ? din[g_dst[i]] : 1;                             \
        const S a = (S)da;                                                                    \
        const S b = (S)db;                                                                    \
        norm[i] = (S)1 / SQRT(a * b);                                                         \
      }                                                                                       \
      free(dout);                                                                             \
    }                                                                                         \
    free(din);                                                                                \
  }
DEFINE_GCN_NORM(f32, float, sqrtf)
DEFINE_GCN_NORM(f64, double, sqrt)

/* message_passing.hpp:76-78 / 441-443 */
void or_degree(const int64_t* ids, int64_t len, int64_t n, int64_t* deg) {
  memset(deg, 0, sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < len; ++i)
    if (ids[i] >= 0 && ids[i] < n) ++deg[ids[i]];
}

/* hetero.hpp:134-157 (per group matmul, tensor.hpp:445-460) */
#define DEFINE_SEGMM(SUF, S)                                                                  \
  void or_segment_matmul_##SUF(const S* x, const int64_t* ptr, int64_t groups, int64_t k,     \
                               int64_t n, const S* w, S* out) {                               \
    for (int64_t g = 0; g < groups; ++g) {                                                    \
      const S* wg = w + g * k * n;                                                            \
      for (int64_t i = ptr[g]; i < ptr[g + 1]; ++i)                                           \
        for (int64_t j = 0; j < n; ++j) {                                                     \
          S acc = (S)0;                                                                       \
          for (int64_t q = 0; q < k; ++q) acc += x[i * k + q] * wg[q * n + j];                \
          out[i * n + j] = acc;                                                               \
        }                                                                                     \
    }                                                                                         \
  }
DEFINE_SEGMM(f64, double)
DEFINE_SEGMM(f32, float)

/* message_passing.hpp:119-166 (the spmm backward closure) */
#define DEFINE_SPMM_BWD(SUF, S)                                                               \
  void or_spmm_backward_##SUF(const int64_t* rp, const int64_t* col, const int64_t* perm,     \
                              int64_t n_src, const int64_t* src, const int64_t* dst,          \
                              int64_t e, const S* g, const S* x, int64_t f, const S* w,       \
                              const int64_t* deg, S* dx, S* dw) {                             \
    /* scaled_g(v, j) = mean ? g / S(max(deg[v], 1)) : g  (:128-132) */                       \
    for (int64_t u = 0; u < n_src; ++u) {                                                     \
      S* o = dx + u * f;                                                                      \
      for (int64_t j = 0; j < f; ++j) o[j] = (S)0;                                            \
      for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {                                           \
        const int64_t v = col[k];                                                             \
        const S coeff = w ? w[perm[k]] : (S)1;                                                \
        for (int64_t j = 0; j < f; ++j) {                                                     \
          const S gv = g[v * f + j];                                                          \
          const S sg = deg ? gv / (S)(deg[v] > 1 ? deg[v] : 1) : gv;                          \
          o[j] += coeff * sg;                                                                 \
        }                                                                                     \
      }                                                                                       \
    }                                                                                         \
    if (w && dw)                                                                              \
      for (int64_t i = 0; i < e; ++i) {                                                       \
        S acc = (S)0;                                                                         \
        for (int64_t j = 0; j < f; ++j) {                                                     \
          const S gv = g[dst[i] * f + j];                                                     \
          const S sg = deg ? gv / (S)(deg[dst[i]] > 1 ? deg[dst[i]] : 1) : gv;                \
          acc += sg * x[src[i] * f + j];                                                      \
        }                                                                                     \
        dw[i] = acc;                                                                          \
      }                                                                                       \
  }
DEFINE_SPMM_BWD(f32, float)
DEFINE_SPMM_BWD(f64, double)
