/*
 * oracle.h — CPU restatement of the reference lseforge loss path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2509_09682_b200/ links, loads or
 * calls this code; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it, and only as the checker.
 *
 * Parity status: PINNED.  Every function below is checked bit-for-bit against
 * the reference itself compiled in place (oracle/_ref/liblseforge_ref.so, see
 * oracle/Makefile and tests/test_oracle.py) and against golden vectors from the
 * reference's own tests (SplitMix64 streams, test_core.cpp:21-52; known answers
 * in test_cce.cpp / test_ccem.cpp / test_oracles.cpp).
 *
 * Layout conventions follow the REFERENCE (not the B200 library):
 *   E    : n x d  float, row-major   (reference "E", hidden states; B200 "X")
 *   C    : d x v  float, row-major   (reference "C", classifier;  B200 "E"^T)
 *   dE   : n x d  double             (GradPair::d_embeddings)
 *   dC   : d x v  double             (GradPair::d_classifier)
 *   inds : n x w  int64, slot 0 = positive (NegIndexMatrix)
 * All accumulation is double, k ascending, exactly as the reference orders it.
 */
#ifndef LSEFORGE_ORACLE_H
#define LSEFORGE_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- SplitMix64 (proj/include/lseforge/rng.hpp:13-60) -------------------- */
typedef struct {
  uint64_t seed;
  uint64_t state;
} orc_rng;

void orc_rng_init(orc_rng* r, uint64_t seed);              /* rng.hpp:15 */
uint64_t orc_rng_next(orc_rng* r);                         /* rng.hpp:17-20 */
uint64_t orc_rng_bounded(orc_rng* r, uint64_t bound);      /* rng.hpp:23-38 */
double orc_rng_uniform(orc_rng* r);                        /* rng.hpp:41 */
void orc_rng_derived(const orc_rng* r, uint64_t index, orc_rng* out); /* rng.hpp:45-47 */
uint64_t orc_mix64(uint64_t z);                            /* rng.hpp:51-55 */

/* ---- test fixtures (proj/tests/support.hpp:27-56) ------------------------- */
/* Fills E (n*d), C (d*v), targets (n) in the reference draw order. */
void orc_make_instance(orc_rng* r, size_t n, size_t d, size_t v, double half_width,
                       float* E, float* C, int64_t* targets);
/* make_candidates: slot 0 = target, negatives uniform with rejection. */
void orc_make_candidates(orc_rng* r, const int64_t* targets, size_t n, size_t ns, size_t v,
                         int64_t* inds);
/* sample_uniform (proj/src/sampler.cpp:44-75): per-row derived(i) streams.
 * Returns 0 on success, -1 if a row exhausts retry_cap. */
int orc_sample_uniform(const int64_t* positives, size_t n, size_t ns, size_t catalog,
                       uint64_t rng_seed, int retry_cap, int64_t* inds);

/* ---- CCE (proj/src/cce.cpp) ----------------------------------------------- */
/* cce_forward (cce.cpp:65-145).  pos, lse: n doubles.  Returns the mean loss.
 * Tiling does not change any per-row operation order in the forward, so no
 * block parameters are needed for bitwise parity. */
double orc_cce_forward(const float* E, const float* C, const int64_t* x, size_t n, size_t d,
                       size_t v, double* pos, double* lse);

/* cce_backward (cce.cpp:147-272).  dE (n*d) and dC (d*v) are OVERWRITTEN.
 * col_block reproduces the reference's per-column-block partial sums for dE
 * (cce.cpp:222-231), which is what makes dE bitwise comparable.
 * Returns skipped_fraction (cce.cpp:264-268); *skipped gets the raw count. */
double orc_cce_backward(const float* E, const float* C, const int64_t* x, const double* lse,
                        double upstream, double filter_eps, size_t col_block, size_t n, size_t d,
                        size_t v, double* dE, double* dC, uint64_t* skipped);

/* Per-shard forward partials for catalog sharding: over columns [v0, v1)
 * of C only.  m = running max, s = rescaled sum (OnlineLse, numeric.hpp:15-30),
 * t = target logit if x[i] in [v0,v1) else 0, has_t = 1/0. */
void orc_cce_forward_partial(const float* E, const float* C, const int64_t* x, size_t n,
                             size_t d, size_t v, size_t v0, size_t v1, double* m, double* s,
                             double* t, int32_t* has_t);

/* ---- CCE- (proj/src/ccem.cpp) --------------------------------------------- */
/* ccem_forward (ccem.cpp:48-105).  inds: n*w.  Returns the mean loss. */
double orc_ccem_forward(const float* E, const float* C, const int64_t* inds, size_t n, size_t d,
                        size_t v, size_t w, double* pos, double* lse);

/* ccem_backward_rows (ccem.cpp:107-194).  dE, dC overwritten. */
void orc_ccem_backward_rows(const float* E, const float* C, const int64_t* inds,
                            const double* lse, const double* row_upstream, size_t n, size_t d,
                            size_t v, size_t w, double* dE, double* dC);

/* ---- validation (losses.cpp:48-69, neg_index.cpp:8-28) --------------------
 * Return 0 if valid, else the first offending row index + 1 (message text is
 * produced by the host library; the oracle only locates the row). */
int64_t orc_validate_targets(const int64_t* x, size_t n, size_t v);
int64_t orc_validate_inds(const int64_t* inds, size_t n, size_t w, size_t v);

/* ---- closed forms (ccem.cpp:207-235, memory_model.cpp:26-74) -------------- */
/* backend: 0 ce, 1 cem, 2 cce, 3 ccem, 4 bce (backend.hpp:10-16) */
void orc_estimate_flops(size_t n, size_t d, size_t v, size_t ns, int backend, uint64_t* fwd,
                        uint64_t* bwd);

/* sample_popularity (sampler.cpp:77-127): inverse CDF over the running sum of
 * count^exponent (exponent 1: the counts), per-row rng.derived(i), one
 * uniform() per attempt; returns 0, -1 (retry cap), -2 (all weights zero). */
int orc_sample_popularity(const int64_t* positives, size_t n, size_t ns, const int64_t* counts,
                          size_t catalog, double exponent, uint64_t rng_seed, int retry_cap,
                          int64_t* inds);

/* ---- full-catalog evaluation (metrics.cpp:13-103, minus the encoder) ------
 * H : n x d double (encode() output, metrics.cpp:46); C : d x v float.
 * Scores s_j = sum_k H[k] * (double)C[k][j], k ascending (metrics.cpp:49-54).
 * Over the item range [v0, v1): ahead[i] = #{j : s_j > s_t, or == and j < t}
 * (metrics.cpp:56-60; rank = 1 + ahead over the whole catalog), top_idx /
 * top_score = the first k items by (score desc, index asc) (metrics.cpp:63-72),
 * -1 / -inf past the range size.  The target score comes from the full C. */
void orc_eval_rank_topk(const double* H, const float* C, const int64_t* targets, size_t n,
                        size_t d, size_t v, size_t v0, size_t v1, size_t k, int64_t* ahead,
                        int64_t* top_idx, double* top_score);
/* metrics.cpp:26-33, 62, 74-103: out3 = {ndcg, coverage, surprisal} from
 * 1-based ranks and top-k lists (k = k_eff).  Returns 0, or 1 for a negative
 * count, 2 for fewer than 2 training events (the reference's invalid_argument). */
int orc_eval_summary(const int64_t* rank, const int64_t* top_idx, size_t n, size_t k,
                     const int64_t* counts, size_t v, double* out3);

/* ---- encoder (encoder.cpp:64-173) -----------------------------------------
 * Windows as a CSR (items, win_off[n_windows + 1]); emb [catalog x d],
 * W [d x d], b [d] float.  encode: rows = sum(len - 1) outputs a, h (double),
 * e (float), targets, row_pos.  backward: from d_h (double) to d_emb, d_W,
 * d_b (double, overwritten). */
void orc_encode_batch(const int64_t* items, const int64_t* win_off, size_t n_windows,
                      const float* emb, const float* W, const float* b, size_t d, double* a,
                      double* h, float* e, int64_t* targets, int64_t* row_pos);
void orc_encoder_backward(const int64_t* items, const int64_t* win_off, size_t n_windows,
                          const float* W, size_t catalog, size_t d, const double* a, const double* h,
                          const int64_t* row_pos, size_t rows, const double* dh, double* d_emb,
                          double* d_W, double* d_b);

/* ---- optimizer (adam.cpp:22-36, 38-55) ------------------------------------
 * One AdamState::apply over n float params with double grads and moments;
 * corr1/2 = 1 - beta^t computed as the reference does (adam.cpp:46-47). */
void orc_adam_apply(float* param, const double* grad, double* m, double* v, size_t n, double lr,
                    double b1, double b2, double eps, uint64_t t);

#ifdef __cplusplus
}
#endif

#endif
