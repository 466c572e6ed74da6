/*
 * oracle.c — CPU restatement of the reference lseforge loss path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Parity: pinned against the
 * reference compiled in place (oracle/_ref) and the reference's golden
 * vectors; see tests/test_oracle.py.
 *
 * Every floating-point expression below reproduces the reference's operand
 * order (double accumulation, k ascending, column order for the online LSE),
 * so results are bitwise identical to the reference built with the same
 * flags (-O3, no FP contraction; x86-64 baseline has no FMA).  Parallelism is
 * OpenMP over outputs that have exactly one owner (rows for pos/lse/dE,
 * columns for dC), so it never changes an operation order.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_RB 64   /* rows per cache block (order-neutral) */
#define ORC_CB 256  /* columns per cache block (order-neutral in the forward) */

/* ------------------------------------------------------------------------ */
/* SplitMix64 — proj/include/lseforge/rng.hpp:13-60                          */
/* ------------------------------------------------------------------------ */
uint64_t orc_mix64(uint64_t z) { /* rng.hpp:51-55 */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void orc_rng_init(orc_rng* r, uint64_t seed) { r->seed = seed; r->state = seed; }

uint64_t orc_rng_next(orc_rng* r) { /* rng.hpp:17-20 */
  r->state += 0x9E3779B97F4A7C15ULL;
  return orc_mix64(r->state);
}

uint64_t orc_rng_bounded(orc_rng* r, uint64_t bound) { /* rng.hpp:23-38 */
  uint64_t mask = bound - 1;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  mask |= mask >> 32;
  for (;;) {
    const uint64_t v = orc_rng_next(r) & mask;
    if (v < bound) return v;
  }
}

double orc_rng_uniform(orc_rng* r) { /* rng.hpp:41 */
  return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
}

void orc_rng_derived(const orc_rng* r, uint64_t index, orc_rng* out) { /* rng.hpp:45-47 */
  orc_rng_init(out, orc_mix64(r->seed + 0x9E3779B97F4A7C15ULL * (index + 1)));
}

/* ------------------------------------------------------------------------ */
/* Fixtures — proj/tests/support.hpp:22-56                                   */
/* ------------------------------------------------------------------------ */
static float symmetric_uniform(orc_rng* r, double half_width) { /* support.hpp:22-24 */
  return (float)((2.0 * orc_rng_uniform(r) - 1.0) * half_width);
}

void orc_make_instance(orc_rng* r, size_t n, size_t d, size_t v, double half_width, float* E,
                       float* C, int64_t* targets) { /* support.hpp:27-37 */
  for (size_t i = 0; i < n * d; ++i) E[i] = symmetric_uniform(r, half_width);
  for (size_t i = 0; i < d * v; ++i) C[i] = symmetric_uniform(r, half_width);
  for (size_t i = 0; i < n; ++i) targets[i] = (int64_t)orc_rng_bounded(r, v);
}

void orc_make_candidates(orc_rng* r, const int64_t* targets, size_t n, size_t ns, size_t v,
                         int64_t* inds) { /* support.hpp:41-56 */
  const size_t w = 1 + ns;
  for (size_t row = 0; row < n; ++row) {
    inds[row * w] = targets[row];
    for (size_t s = 1; s <= ns; ++s) {
      int64_t draw;
      do {
        draw = (int64_t)orc_rng_bounded(r, v);
      } while (draw == targets[row]);
      inds[row * w + s] = draw;
    }
  }
}

int orc_sample_uniform(const int64_t* positives, size_t n, size_t ns, size_t catalog,
                       uint64_t rng_seed, int retry_cap, int64_t* inds) { /* sampler.cpp:44-75 */
  const size_t w = 1 + ns;
  orc_rng base;
  orc_rng_init(&base, rng_seed);
  int failed = 0;
#pragma omp parallel for schedule(static) reduction(| : failed)
  for (size_t i = 0; i < n; ++i) {
    orc_rng row;
    orc_rng_derived(&base, i, &row);
    inds[i * w] = positives[i];
    for (size_t s = 1; s <= ns; ++s) {
      int placed = 0;
      for (int attempt = 0; attempt < retry_cap; ++attempt) {
        const int64_t v = (int64_t)orc_rng_bounded(&row, catalog);
        if (v != positives[i]) {
          inds[i * w + s] = v;
          placed = 1;
          break;
        }
      }
      if (!placed) failed = 1;
    }
  }
  return failed ? -1 : 0;
}

int orc_sample_popularity(const int64_t* positives, size_t n, size_t ns, const int64_t* counts,
                          size_t catalog, double exponent, uint64_t rng_seed, int retry_cap,
                          int64_t* inds) { /* sampler.cpp:77-127 */
  double* cum = (double*)malloc(sizeof(double) * (catalog ? catalog : 1));
  double running = 0.0;
  for (size_t v = 0; v < catalog; ++v) { /* sampler.cpp:93-99 */
    const double c = (double)counts[v];
    running += exponent == 1.0 ? c : pow(c, exponent);
    cum[v] = running;
  }
  if (!(running > 0.0)) {
    free(cum);
    return -2;
  }
  const size_t w = 1 + ns;
  orc_rng base;
  orc_rng_init(&base, rng_seed);
  int failed = 0;
#pragma omp parallel for schedule(static) reduction(| : failed)
  for (size_t i = 0; i < n; ++i) {
    orc_rng row;
    orc_rng_derived(&base, i, &row);
    inds[i * w] = positives[i];
    for (size_t s = 1; s <= ns; ++s) {
      int placed = 0;
      for (int attempt = 0; attempt < retry_cap; ++attempt) {
        const double u = orc_rng_uniform(&row) * running;
        size_t lo = 0, hi = catalog; /* upper_bound: first cum[v] > u */
        while (lo < hi) {
          const size_t mid = lo + (hi - lo) / 2;
          if (!(u < cum[mid])) lo = mid + 1; else hi = mid;
        }
        if (lo == catalog) continue; /* u rounded up to the total: redraw */
        if ((int64_t)lo != positives[i]) {
          inds[i * w + s] = (int64_t)lo;
          placed = 1;
          break;
        }
      }
      if (!placed) failed = 1;
    }
  }
  free(cum);
  return failed ? -1 : 0;
}

/* ------------------------------------------------------------------------ */
/* Logit tile — cce.cpp:40-55: tile[i][j] = sum_k E[i][k]*C[k][j], double,   */
/* k ascending, starting from 0.0.                                           */
/* ------------------------------------------------------------------------ */
static void logit_tile(const float* E, const float* C, size_t d, size_t v, size_t r0, size_t nb,
                       size_t c0, size_t cbn, double* tile) {
  memset(tile, 0, sizeof(double) * nb * cbn);
  for (size_t i = 0; i < nb; ++i) {
    const float* erow = E + (r0 + i) * d;
    double* trow = tile + i * cbn;
    for (size_t k = 0; k < d; ++k) {
      const double e = erow[k];
      const float* crow = C + k * v + c0;
      for (size_t j = 0; j < cbn; ++j) trow[j] += e * (double)crow[j];
    }
  }
}

/* OnlineLse::update — numeric.hpp:19-27 (same branch structure as cce.cpp:116-124) */
static inline void lse_update(double* m, double* dsum, double o) {
  if (o <= *m) {
    *dsum += exp(o - *m);
  } else {
    *dsum = *dsum * exp(*m - o) + 1.0;
    *m = o;
  }
}

/* ------------------------------------------------------------------------ */
/* cce_forward — cce.cpp:65-145                                               */
/* ------------------------------------------------------------------------ */
static void cce_partial_rows(const float* E, const float* C, const int64_t* x, size_t n, size_t d,
                             size_t v, size_t v0, size_t v1, double* m_out, double* s_out,
                             double* t_out, int32_t* has_t) {
  const size_t nrb = (n + ORC_RB - 1) / ORC_RB;
#pragma omp parallel
  {
    double* tile = (double*)malloc(sizeof(double) * ORC_RB * ORC_CB);
    double m[ORC_RB], ds[ORC_RB];
#pragma omp for schedule(dynamic, 1)
    for (size_t b = 0; b < nrb; ++b) {
      const size_t r0 = b * ORC_RB;
      const size_t nb = (n - r0) < ORC_RB ? (n - r0) : ORC_RB;
      for (size_t i = 0; i < nb; ++i) {
        m[i] = -INFINITY;
        ds[i] = 0.0;
        t_out[r0 + i] = 0.0;
        has_t[r0 + i] = 0;
      }
      for (size_t c0 = v0; c0 < v1; c0 += ORC_CB) {
        const size_t cbn = (v1 - c0) < ORC_CB ? (v1 - c0) : ORC_CB;
        logit_tile(E, C, d, v, r0, nb, c0, cbn, tile);
        for (size_t i = 0; i < nb; ++i) {
          const double* trow = tile + i * cbn;
          for (size_t j = 0; j < cbn; ++j) lse_update(&m[i], &ds[i], trow[j]);
          const size_t xi = (size_t)x[r0 + i];
          if (xi >= c0 && xi < c0 + cbn) { /* cce.cpp:128-131 */
            t_out[r0 + i] = trow[xi - c0];
            has_t[r0 + i] = 1;
          }
        }
      }
      for (size_t i = 0; i < nb; ++i) {
        m_out[r0 + i] = m[i];
        s_out[r0 + i] = ds[i];
      }
    }
    free(tile);
  }
}

void orc_cce_forward_partial(const float* E, const float* C, const int64_t* x, size_t n,
                             size_t d, size_t v, size_t v0, size_t v1, double* m, double* s,
                             double* t, int32_t* has_t) {
  cce_partial_rows(E, C, x, n, d, v, v0, v1, m, s, t, has_t);
}

double orc_cce_forward(const float* E, const float* C, const int64_t* x, size_t n, size_t d,
                       size_t v, double* pos, double* lse) {
  double* s = (double*)malloc(sizeof(double) * n);
  int32_t* has_t = (int32_t*)malloc(sizeof(int32_t) * n);
  cce_partial_rows(E, C, x, n, d, v, 0, v, lse, s, pos, has_t);
  for (size_t i = 0; i < n; ++i) lse[i] += log(s[i]); /* cce.cpp:134-136 */
  double total = 0.0;                                   /* cce.cpp:139-141 */
  for (size_t i = 0; i < n; ++i) total += lse[i] - pos[i];
  free(s);
  free(has_t);
  return total / (double)n;
}

/* ------------------------------------------------------------------------ */
/* cce_backward — cce.cpp:147-272                                            */
/* ------------------------------------------------------------------------ */
/* coefficients lambda — cce.cpp:189-204 */
static inline uint64_t coefficients(double* trow, double row_lse, int64_t xi, size_t c0,
                                    size_t cbn, double eps, double scale) {
  uint64_t skips = 0;
  for (size_t j = 0; j < cbn; ++j) {
    const double s = exp(trow[j] - row_lse);
    if ((int64_t)(c0 + j) == xi) {
      trow[j] = (s - 1.0) * scale;
    } else if (eps > 0.0 && s < eps) {
      trow[j] = 0.0;
      ++skips;
    } else {
      trow[j] = s * scale;
    }
  }
  return skips;
}

double orc_cce_backward(const float* E, const float* C, const int64_t* x, const double* lse,
                        double upstream, double filter_eps, size_t col_block, size_t n, size_t d,
                        size_t v, double* dE, double* dC, uint64_t* skipped_out) {
  const double scale = upstream / (double)n; /* cce.cpp:174 */
  const size_t cb = col_block < v ? col_block : v;
  const size_t ncb = (v + cb - 1) / cb;
  const size_t nrb = (n + ORC_RB - 1) / ORC_RB;
  memset(dE, 0, sizeof(double) * n * d);
  memset(dC, 0, sizeof(double) * d * v);
  uint64_t skipped = 0;

  /* Pass 1 — dE, row-owned; per column block a partial `acc` folded into
   * derow[k] (cce.cpp:210-233). */
#pragma omp parallel reduction(+ : skipped)
  {
    double* tile = (double*)malloc(sizeof(double) * ORC_RB * cb);
#pragma omp for schedule(dynamic, 1)
    for (size_t b = 0; b < nrb; ++b) {
      const size_t r0 = b * ORC_RB;
      const size_t nb = (n - r0) < ORC_RB ? (n - r0) : ORC_RB;
      for (size_t cI = 0; cI < ncb; ++cI) {
        const size_t c0 = cI * cb;
        const size_t cbn = (v - c0) < cb ? (v - c0) : cb;
        logit_tile(E, C, d, v, r0, nb, c0, cbn, tile);
        for (size_t i = 0; i < nb; ++i)
          skipped += coefficients(tile + i * cbn, lse[r0 + i], x[r0 + i], c0, cbn, filter_eps,
                                  scale);
        for (size_t i = 0; i < nb; ++i) {
          const double* trow = tile + i * cbn;
          double* derow = dE + (r0 + i) * d;
          for (size_t k = 0; k < d; ++k) {
            const float* crow = C + k * v + c0;
            double acc = 0.0;
            for (size_t j = 0; j < cbn; ++j) acc += trow[j] * (double)crow[j];
            derow[k] += acc;
          }
        }
      }
    }
    free(tile);
  }

  /* Pass 2 — dC, column-owned; rows ascending (cce.cpp:240-262). */
#pragma omp parallel
  {
    double* tile = (double*)malloc(sizeof(double) * ORC_RB * cb);
#pragma omp for schedule(dynamic, 1)
    for (size_t cI = 0; cI < ncb; ++cI) {
      const size_t c0 = cI * cb;
      const size_t cbn = (v - c0) < cb ? (v - c0) : cb;
      for (size_t b = 0; b < nrb; ++b) {
        const size_t r0 = b * ORC_RB;
        const size_t nb = (n - r0) < ORC_RB ? (n - r0) : ORC_RB;
        logit_tile(E, C, d, v, r0, nb, c0, cbn, tile);
        for (size_t i = 0; i < nb; ++i)
          (void)coefficients(tile + i * cbn, lse[r0 + i], x[r0 + i], c0, cbn, filter_eps, scale);
        for (size_t i = 0; i < nb; ++i) {
          const double* trow = tile + i * cbn;
          const float* erow = E + (r0 + i) * d;
          for (size_t k = 0; k < d; ++k) {
            double* dcrow = dC + k * v + c0;
            const double e = erow[k];
            for (size_t j = 0; j < cbn; ++j) dcrow[j] += e * trow[j];
          }
        }
      }
    }
    free(tile);
  }

  if (skipped_out) *skipped_out = skipped;
  const uint64_t off_target = (uint64_t)n * (v - 1); /* cce.cpp:264-268 */
  return off_target == 0 ? 0.0 : (double)skipped / (double)off_target;
}

/* ------------------------------------------------------------------------ */
/* CCE- — ccem.cpp:48-205                                                    */
/* ------------------------------------------------------------------------ */
/* gather_column + dot_row — ccem.cpp:34-44 */
static inline double dot_col(const float* erow, const float* C, size_t d, size_t v, size_t col) {
  double acc = 0.0;
  for (size_t k = 0; k < d; ++k) acc += (double)erow[k] * (double)C[k * v + col];
  return acc;
}

double orc_ccem_forward(const float* E, const float* C, const int64_t* inds, size_t n, size_t d,
                        size_t v, size_t w, double* pos, double* lse) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) { /* ccem.cpp:80-97 */
    const float* erow = E + i * d;
    double m = -INFINITY, dsum = 0.0;
    for (size_t s = 0; s < w; ++s) {
      const double o = dot_col(erow, C, d, v, (size_t)inds[i * w + s]);
      if (s == 0) pos[i] = o;
      lse_update(&m, &dsum, o);
    }
    lse[i] = m + log(dsum);
  }
  double total = 0.0; /* ccem.cpp:99-101 */
  for (size_t i = 0; i < n; ++i) total += lse[i] - pos[i];
  return total / (double)n;
}

void orc_ccem_backward_rows(const float* E, const float* C, const int64_t* inds,
                            const double* lse, const double* row_upstream, size_t n, size_t d,
                            size_t v, size_t w, double* dE, double* dC) {
  double* coeff = (double*)malloc(sizeof(double) * n * w); /* ccem.cpp:144 */
  memset(dE, 0, sizeof(double) * n * d);
  memset(dC, 0, sizeof(double) * d * v);
  /* Pass 1 — rows (ccem.cpp:146-164). */
#pragma omp parallel
  {
    float* col = (float*)malloc(sizeof(float) * (d ? d : 1));
#pragma omp for schedule(static)
    for (size_t i = 0; i < n; ++i) {
      const float* erow = E + i * d;
      double* derow = dE + i * d;
      const double row_lse = lse[i];
      const double u = row_upstream[i];
      for (size_t s = 0; s < w; ++s) {
        const size_t c = (size_t)inds[i * w + s];
        for (size_t k = 0; k < d; ++k) col[k] = C[k * v + c];
        double o = 0.0;
        for (size_t k = 0; k < d; ++k) o += (double)erow[k] * (double)col[k];
        const double soft = exp(o - row_lse);
        const double g = (s == 0 ? soft - 1.0 : soft) * u;
        coeff[i * w + s] = g;
        for (size_t k = 0; k < d; ++k) derow[k] += g * (double)col[k];
      }
    }
    free(col);
  }
  /* Pass 2 — columns, (row, slot) ascending per owned column (ccem.cpp:170-187).
   * Each thread owns a contiguous column range and scans the whole matrix. */
#pragma omp parallel
  {
#ifdef _OPENMP
    extern int omp_get_thread_num(void);
    extern int omp_get_num_threads(void);
    const size_t tid = (size_t)omp_get_thread_num();
    const size_t nt = (size_t)omp_get_num_threads();
#else
    const size_t tid = 0, nt = 1;
#endif
    const int64_t lo = (int64_t)(v * tid / nt);
    const int64_t hi = (int64_t)(v * (tid + 1) / nt);
    for (size_t i = 0; i < n; ++i) {
      const float* erow = E + i * d;
      for (size_t s = 0; s < w; ++s) {
        const int64_t t = inds[i * w + s];
        if (t < lo || t >= hi) continue;
        const double g = coeff[i * w + s];
        for (size_t k = 0; k < d; ++k) dC[k * v + (size_t)t] += g * (double)erow[k];
      }
    }
  }
  free(coeff);
}

/* ------------------------------------------------------------------------ */
/* Validation — losses.cpp:48-69, neg_index.cpp:8-28                          */
/* ------------------------------------------------------------------------ */
int64_t orc_validate_targets(const int64_t* x, size_t n, size_t v) {
  for (size_t i = 0; i < n; ++i)
    if (x[i] < 0 || x[i] >= (int64_t)v) return (int64_t)i + 1;
  return 0;
}

int64_t orc_validate_inds(const int64_t* inds, size_t n, size_t w, size_t v) {
  for (size_t r = 0; r < n; ++r) {
    const int64_t pos = inds[r * w];
    for (size_t s = 0; s < w; ++s) {
      const int64_t x = inds[r * w + s];
      if (x < 0 || x >= (int64_t)v) return (int64_t)r + 1;
      if (s > 0 && x == pos) return (int64_t)r + 1;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* estimate_flops — ccem.cpp:207-235                                         */
/* ------------------------------------------------------------------------ */
void orc_estimate_flops(size_t n, size_t d, size_t v, size_t ns, int backend, uint64_t* fwd,
                        uint64_t* bwd) {
  uint64_t scored = 0, factor = 2;
  switch (backend) {
    case 0: scored = v; break;
    case 1: scored = 1 + ns; break;
    case 2: scored = v; factor = 3; break;
    case 3: scored = 1 + ns; factor = 3; break;
    case 4: scored = 2; break;
    default: scored = 0;
  }
  *fwd = (uint64_t)n * d * scored;
  *bwd = factor * *fwd;
}

/* ---- full-catalog evaluation (metrics.cpp:13-103) ------------------------- */
static void eval_scores(const double* h, const float* C, size_t d, size_t v, double* scores) {
  for (size_t j = 0; j < v; ++j) scores[j] = 0.0;
  for (size_t kk = 0; kk < d; ++kk) { /* metrics.cpp:49-54 */
    const double hk = h[kk];
    const float* crow = C + kk * v;
    for (size_t j = 0; j < v; ++j) scores[j] += hk * (double)crow[j];
  }
}

void orc_eval_rank_topk(const double* H, const float* C, const int64_t* targets, size_t n,
                        size_t d, size_t v, size_t v0, size_t v1, size_t k, int64_t* ahead,
                        int64_t* top_idx, double* top_score) {
#pragma omp parallel
  {
    double* scores = (double*)malloc(sizeof(double) * (v ? v : 1));
#pragma omp for schedule(dynamic)
    for (size_t i = 0; i < n; ++i) {
      eval_scores(H + i * d, C, d, v, scores);
      const size_t t = (size_t)targets[i];
      const double st = scores[t];
      int64_t a = 0;
      for (size_t j = v0; j < v1; ++j) /* metrics.cpp:57-60 */
        if (scores[j] > st || (scores[j] == st && j < t)) ++a;
      ahead[i] = a;
      /* top-k by (score desc, index asc): insertion into a sorted list */
      int64_t* ti = top_idx + i * k;
      double* tv = top_score + i * k;
      size_t filled = 0;
      for (size_t j = v0; j < v1; ++j) {
        const double s = scores[j];
        if (filled == k && !(s > tv[k - 1])) continue; /* ascending j: ties never displace */
        size_t pos = filled < k ? filled : k - 1;
        while (pos > 0 && s > tv[pos - 1]) {
          if (pos < k) { tv[pos] = tv[pos - 1]; ti[pos] = ti[pos - 1]; }
          --pos;
        }
        tv[pos] = s;
        ti[pos] = (int64_t)j;
        if (filled < k) ++filled;
      }
      for (size_t e = filled; e < k; ++e) { ti[e] = -1; tv[e] = -INFINITY; }
    }
    free(scores);
  }
}

int orc_eval_summary(const int64_t* rank, const int64_t* top_idx, size_t n, size_t k,
                     const int64_t* counts, size_t v, double* out3) {
  double total = 0.0;
  for (size_t j = 0; j < v; ++j) { /* metrics.cpp:26-33 */
    if (counts[j] < 0) return 1;
    total += (double)counts[j];
  }
  if (total < 2.0) return 2;
  const double log2_total = log2(total);
  double ndcg_sum = 0.0, surp_sum = 0.0;
  size_t distinct = 0;
  char* seen = (char*)calloc(v ? v : 1, 1);
  for (size_t i = 0; i < n; ++i) {
    const int64_t r = rank[i]; /* metrics.cpp:61 */
    ndcg_sum += r <= (int64_t)k ? 1.0 / log2((double)r + 1.0) : 0.0;
    double acc = 0.0; /* metrics.cpp:74-80 */
    for (size_t e = 0; e < k; ++e) {
      const int64_t item = top_idx[i * k + e];
      const double c = (double)(counts[item] > 1 ? counts[item] : 1);
      acc += -log2(c / total) / log2_total;
      if (!seen[item]) { seen[item] = 1; ++distinct; } /* metrics.cpp:90-97 */
    }
    surp_sum += acc / (double)k;
  }
  free(seen);
  out3[0] = ndcg_sum / (double)n;
  out3[1] = (double)distinct / (double)v;
  out3[2] = surp_sum / (double)n;
  return 0;
}

/* ---- optimizer (adam.cpp:22-36) ------------------------------------------- */
void orc_adam_apply(float* param, const double* grad, double* m, double* v, size_t n, double lr,
                    double b1, double b2, double eps, uint64_t t) {
  const double corr1 = 1.0 - pow(b1, (double)t); /* adam.cpp:46-47 */
  const double corr2 = 1.0 - pow(b2, (double)t);
  for (size_t i = 0; i < n; ++i) { /* adam.cpp:27-35 */
    const double g = grad[i];
    m[i] = b1 * m[i] + (1.0 - b1) * g;
    v[i] = b2 * v[i] + (1.0 - b2) * g * g;
    const double mhat = m[i] / corr1;
    const double vhat = v[i] / corr2;
    const double p = (double)param[i] - lr * mhat / (sqrt(vhat) + eps);
    param[i] = (float)p;
  }
}

/* ---- encoder (encoder.cpp:64-173) ----------------------------------------- */
void orc_encode_batch(const int64_t* items, const int64_t* win_off, size_t n_windows,
                      const float* emb, const float* W, const float* b, size_t d, double* a,
                      double* h, float* e, int64_t* targets, int64_t* row_pos) {
  double* sum = (double*)malloc(sizeof(double) * d);
  size_t r = 0;
  for (size_t wi = 0; wi < n_windows; ++wi) { /* encoder.cpp:88-112 */
    const int64_t* win = items + win_off[wi];
    const size_t len = (size_t)(win_off[wi + 1] - win_off[wi]);
    for (size_t k = 0; k < d; ++k) sum[k] = 0.0;
    for (size_t t = 1; t < len; ++t, ++r) {
      const float* erow = emb + (size_t)win[t - 1] * d;
      for (size_t k = 0; k < d; ++k) sum[k] += (double)erow[k];
      const double inv = 1.0 / (double)t;
      double* arow = a + r * d;
      for (size_t j = 0; j < d; ++j) arow[j] = sum[j] * inv;
      for (size_t j = 0; j < d; ++j) {
        double z = (double)b[j];
        const float* wrow = W + j * d;
        for (size_t k = 0; k < d; ++k) z += (double)wrow[k] * arow[k];
        h[r * d + j] = tanh(z);
        e[r * d + j] = (float)h[r * d + j];
      }
      targets[r] = win[t];
      row_pos[r] = (int64_t)t;
    }
  }
  free(sum);
}

void orc_encoder_backward(const int64_t* items, const int64_t* win_off, size_t n_windows,
                          const float* W, size_t catalog, size_t d, const double* a, const double* h,
                          const int64_t* row_pos, size_t rows, const double* dh, double* d_emb,
                          double* d_W, double* d_b) {
  memset(d_emb, 0, sizeof(double) * catalog * d);
  memset(d_W, 0, sizeof(double) * d * d);
  memset(d_b, 0, sizeof(double) * d);
  double* g = (double*)malloc(sizeof(double) * d);
  double* u = (double*)malloc(sizeof(double) * d);
  double* suffix = (double*)malloc(sizeof(double) * d);
  /* row offsets of each window */
  size_t r_end = rows;
  for (size_t wi = n_windows; wi-- > 0;) { /* encoder.cpp:137-170, windows last to first */
    const int64_t* win = items + win_off[wi];
    const size_t len = (size_t)(win_off[wi + 1] - win_off[wi]);
    const size_t r_begin = r_end - (len - 1);
    for (size_t k = 0; k < d; ++k) suffix[k] = 0.0;
    for (size_t r = r_end; r-- > r_begin;) {
      const size_t t = (size_t)row_pos[r];
      const double* hrow = h + r * d;
      const double* dhr = dh + r * d;
      for (size_t j = 0; j < d; ++j) g[j] = (1.0 - hrow[j] * hrow[j]) * dhr[j];
      const double* arow = a + r * d;
      for (size_t j = 0; j < d; ++j) {
        double* dwrow = d_W + j * d;
        for (size_t k = 0; k < d; ++k) dwrow[k] += g[j] * arow[k];
        d_b[j] += g[j];
      }
      const double inv = 1.0 / (double)t;
      for (size_t k = 0; k < d; ++k) {
        double acc = 0.0;
        for (size_t j = 0; j < d; ++j) acc += (double)W[j * d + k] * g[j];
        u[k] = acc * inv;
      }
      for (size_t k = 0; k < d; ++k) suffix[k] += u[k];
      double* derow = d_emb + (size_t)win[t - 1] * d;
      for (size_t k = 0; k < d; ++k) derow[k] += suffix[k];
    }
    r_end = r_begin;
  }
  (void)catalog;
  free(g);
  free(u);
  free(suffix);
}
