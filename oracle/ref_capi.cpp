// ref_capi.cpp — flat C entry points over the UNMODIFIED reference lseforge
// sources, compiled in place from /root/reference/proj/src by oracle/Makefile
// into oracle/_ref/liblseforge_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the C restatement
// (oracle/oracle.c) and by bench.py's `--impl reference` arm as the
// reference CPU timing.  The product library never links this.
//
// Layouts are the reference's own: E n×d float, C d×v float, outputs double.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "lseforge/accountant.hpp"
#include "lseforge/adam.hpp"
#include "lseforge/backend.hpp"
#include "lseforge/cce.hpp"
#include "lseforge/ccem.hpp"
#include "lseforge/losses.hpp"
#include "lseforge/encoder.hpp"
#include "lseforge/memory_model.hpp"
#include "lseforge/metrics.hpp"
#include "lseforge/neg_index.hpp"
#include "lseforge/rng.hpp"
#include "lseforge/sampler.hpp"
#include "support.hpp"

using namespace lseforge;

namespace {

thread_local std::string g_err;

DenseMatrix to_matrix(const float* p, std::size_t r, std::size_t c) {
  DenseMatrix m(r, c);
  if (r * c) std::memcpy(m.data().data(), p, sizeof(float) * r * c);
  return m;
}

NegIndexMatrix to_inds(const int64_t* p, std::size_t n, std::size_t w) {
  NegIndexMatrix m(n, w);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t s = 0; s < w; ++s) m(i, s) = p[i * w + s];
  return m;
}

CceConfig make_cfg(std::size_t rb, std::size_t cb, double eps, int workers) {
  CceConfig cfg;
  cfg.row_block = rb;
  cfg.col_block = cb;
  cfg.filter_eps = eps;
  cfg.workers = workers;
  return cfg;
}

void copy_out(const DenseMatrixD& m, double* dst) {
  if (dst && m.size()) std::memcpy(dst, m.data().data(), sizeof(double) * m.size());
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- rng.hpp / support.hpp -------------------------------------------------
void ref_rng_stream(uint64_t seed, uint64_t* out, int count) {
  SplitMix64 r(seed);
  for (int i = 0; i < count; ++i) out[i] = r.next();
}

void ref_make_instance(uint64_t seed, std::size_t n, std::size_t d, std::size_t v,
                       double half_width, float* E, float* C, int64_t* targets) {
  SplitMix64 rng(seed);
  testsupport::Instance inst = testsupport::make_instance(rng, n, d, v, half_width);
  std::memcpy(E, inst.E.data().data(), sizeof(float) * n * d);
  std::memcpy(C, inst.C.data().data(), sizeof(float) * d * v);
  std::memcpy(targets, inst.targets.data(), sizeof(int64_t) * n);
}

// make_instance followed by make_candidates on the same generator.
void ref_make_instance_candidates(uint64_t seed, std::size_t n, std::size_t d, std::size_t v,
                                  std::size_t ns, float* E, float* C, int64_t* targets,
                                  int64_t* inds) {
  SplitMix64 rng(seed);
  testsupport::Instance inst = testsupport::make_instance(rng, n, d, v);
  NegIndexMatrix m = testsupport::make_candidates(rng, inst.targets, ns, v);
  std::memcpy(E, inst.E.data().data(), sizeof(float) * n * d);
  std::memcpy(C, inst.C.data().data(), sizeof(float) * d * v);
  std::memcpy(targets, inst.targets.data(), sizeof(int64_t) * n);
  std::memcpy(inds, m.data().data(), sizeof(int64_t) * n * (1 + ns));
}

int ref_sample_uniform(const int64_t* positives, std::size_t n, std::size_t ns,
                       std::size_t catalog, uint64_t seed, int64_t* inds) {
  return guard([&] {
    NegIndexMatrix m =
        sample_uniform(std::span<const int64_t>(positives, n), ns, catalog, SplitMix64(seed));
    std::memcpy(inds, m.data().data(), sizeof(int64_t) * n * (1 + ns));
  });
}

int ref_sample_popularity(const int64_t* positives, std::size_t n, std::size_t ns,
                          const int64_t* counts, std::size_t catalog, double exponent,
                          uint64_t seed, int64_t* inds) {
  return guard([&] {
    PopularityTable pop = PopularityTable::FromCounts(std::vector<int64_t>(counts, counts + catalog));
    SamplerConfig cfg;
    cfg.popularity_exponent = exponent;
    NegIndexMatrix m = sample_popularity(std::span<const int64_t>(positives, n), ns, pop,
                                         SplitMix64(seed), cfg);
    std::memcpy(inds, m.data().data(), sizeof(int64_t) * n * (1 + ns));
  });
}

// ---- cce.cpp ---------------------------------------------------------------
int ref_cce_forward(const float* E, const float* C, const int64_t* x, std::size_t n,
                    std::size_t d, std::size_t v, std::size_t rb, std::size_t cb, int workers,
                    double* pos, double* lse, double* loss) {
  return guard([&] {
    const DenseMatrix Em = to_matrix(E, n, d), Cm = to_matrix(C, d, v);
    LossOutput o = cce_forward(Em, Cm, std::span<const int64_t>(x, n),
                               make_cfg(rb, cb, 0.0, workers));
    std::memcpy(pos, o.pos_logits.data(), sizeof(double) * n);
    std::memcpy(lse, o.lse.data(), sizeof(double) * n);
    *loss = o.loss;
  });
}

int ref_cce_backward(const float* E, const float* C, const int64_t* x, const double* lse,
                     double upstream, double eps, std::size_t n, std::size_t d, std::size_t v,
                     std::size_t rb, std::size_t cb, int workers, double* dE, double* dC,
                     double* skipped_fraction) {
  return guard([&] {
    const DenseMatrix Em = to_matrix(E, n, d), Cm = to_matrix(C, d, v);
    CceBackwardResult r =
        cce_backward(Em, Cm, std::span<const int64_t>(x, n), std::span<const double>(lse, n),
                     upstream, make_cfg(rb, cb, eps, workers));
    copy_out(r.grads.d_embeddings, dE);
    copy_out(r.grads.d_classifier, dC);
    *skipped_fraction = r.skipped_fraction;
  });
}

// ---- ccem.cpp --------------------------------------------------------------
int ref_ccem_forward(const float* E, const float* C, const int64_t* inds, std::size_t n,
                     std::size_t d, std::size_t v, std::size_t w, std::size_t rb, int workers,
                     double* pos, double* lse, double* loss) {
  return guard([&] {
    const DenseMatrix Em = to_matrix(E, n, d), Cm = to_matrix(C, d, v);
    LossOutput o = ccem_forward(Em, Cm, to_inds(inds, n, w), make_cfg(rb, 256, 0.0, workers));
    std::memcpy(pos, o.pos_logits.data(), sizeof(double) * n);
    std::memcpy(lse, o.lse.data(), sizeof(double) * n);
    *loss = o.loss;
  });
}

int ref_ccem_backward_rows(const float* E, const float* C, const int64_t* inds,
                           const double* lse, const double* row_upstream, std::size_t n,
                           std::size_t d, std::size_t v, std::size_t w, std::size_t rb,
                           int workers, double* dE, double* dC) {
  return guard([&] {
    const DenseMatrix Em = to_matrix(E, n, d), Cm = to_matrix(C, d, v);
    GradPair g = ccem_backward_rows(Em, Cm, to_inds(inds, n, w), std::span<const double>(lse, n),
                                    std::span<const double>(row_upstream, n),
                                    make_cfg(rb, 256, 0.0, workers));
    copy_out(g.d_embeddings, dE);
    copy_out(g.d_classifier, dC);
  });
}

// ---- losses.cpp (materializing oracles) -----------------------------------
int ref_ce_full(const float* E, const float* C, const int64_t* x, std::size_t n, std::size_t d,
                std::size_t v, double upstream, double* pos, double* lse, double* loss,
                double* dE, double* dC) {
  return guard([&] {
    const DenseMatrix Em = to_matrix(E, n, d), Cm = to_matrix(C, d, v);
    const std::span<const int64_t> xs(x, n);
    LossOutput o = ce_full_forward(Em, Cm, xs);
    std::memcpy(pos, o.pos_logits.data(), sizeof(double) * n);
    std::memcpy(lse, o.lse.data(), sizeof(double) * n);
    *loss = o.loss;
    if (dE || dC) {
      GradPair g = ce_full_backward(Em, Cm, xs, upstream);
      copy_out(g.d_embeddings, dE);
      copy_out(g.d_classifier, dC);
    }
  });
}

int ref_ce_sampled(const float* E, const float* C, const int64_t* inds, std::size_t n,
                   std::size_t d, std::size_t v, std::size_t w, double upstream, double* pos,
                   double* lse, double* loss, double* dE, double* dC) {
  return guard([&] {
    const DenseMatrix Em = to_matrix(E, n, d), Cm = to_matrix(C, d, v);
    const NegIndexMatrix im = to_inds(inds, n, w);
    LossOutput o = ce_sampled_forward(Em, Cm, im);
    std::memcpy(pos, o.pos_logits.data(), sizeof(double) * n);
    std::memcpy(lse, o.lse.data(), sizeof(double) * n);
    *loss = o.loss;
    if (dE || dC) {
      GradPair g = ce_sampled_backward(Em, Cm, im, upstream);
      copy_out(g.d_embeddings, dE);
      copy_out(g.d_classifier, dC);
    }
  });
}

// ---- validation / closed forms ----------------------------------------------
int ref_validate_targets(std::size_t n_rows_E, std::size_t d, std::size_t v, const int64_t* x,
                         std::size_t nx) {
  return guard([&] {
    DenseMatrix Em(n_rows_E, d), Cm(d, v);
    validate_loss_inputs(Em, Cm, std::span<const int64_t>(x, nx));
  });
}

int ref_validate_inds(const int64_t* inds, std::size_t n, std::size_t w, std::size_t v) {
  return guard([&] { to_inds(inds, n, w).validate(v); });
}

void ref_estimate_flops(std::size_t n, std::size_t d, std::size_t v, std::size_t ns, int backend,
                        uint64_t* fwd, uint64_t* bwd) {
  FlopEstimate f = estimate_flops(n, d, v, ns, static_cast<Backend>(backend));
  *fwd = f.forward;
  *bwd = f.backward;
}

// ---- metrics.cpp -----------------------------------------------------------
// One evaluation instance through the reference's own evaluate(): params =
// ToyEncoderParams::Init(catalog, hidden, SplitMix64(seed)), pairs with
// prefixes [n x L] and targets.  Returns the summary (out3 = ndcg, coverage,
// surprisal), the encoded rows H [n x hidden] (encode(), what evaluate()
// scores with), the classifier C [hidden x catalog], and per-row ranks
// recovered from single-pair evaluate() calls at k = catalog
// (ndcg = 1 / log2(rank + 1)).
int ref_eval_instance(std::size_t catalog, std::size_t hidden, uint64_t seed, std::size_t n,
                      std::size_t L, const int64_t* prefixes, const int64_t* targets, std::size_t k,
                      const int64_t* counts, int workers, double* out3, double* H, float* C,
                      int64_t* ranks) {
  return guard([&] {
    const ToyEncoderParams p = ToyEncoderParams::Init(catalog, hidden, SplitMix64(seed));
    std::vector<EvalPair> pairs(n);
    for (std::size_t i = 0; i < n; ++i) {
      pairs[i].user = static_cast<int64_t>(i);
      pairs[i].prefix.assign(prefixes + i * L, prefixes + (i + 1) * L);
      pairs[i].target = targets[i];
    }
    const std::vector<int64_t> cnt(counts, counts + catalog);
    const EvalSummary sum = evaluate(p, pairs, k, cnt, workers);
    out3[0] = sum.ndcg;
    out3[1] = sum.coverage;
    out3[2] = sum.surprisal;
    if (C) std::memcpy(C, p.c.data().data(), sizeof(float) * hidden * catalog);
    for (std::size_t i = 0; i < n; ++i) {
      if (H) {
        const std::vector<double> h = encode(p, pairs[i].prefix);
        std::memcpy(H + i * hidden, h.data(), sizeof(double) * hidden);
      }
      if (ranks) {
        const EvalSummary one = evaluate(p, std::span<const EvalPair>(&pairs[i], 1), catalog, cnt, 1);
        ranks[i] = static_cast<int64_t>(std::llround(std::exp2(1.0 / one.ndcg) - 1.0));
      }
    }
  });
}

// ---- adam.cpp -------------------------------------------------------------
// `steps` AdamState::step calls on ToyEncoderParams::Init(catalog, hidden,
// SplitMix64(seed)) with the caller's gradients (grads: steps blocks of
// [d_emb (catalog*hidden) | d_w (hidden^2) | d_b (hidden) | d_classifier
// (hidden*catalog)] doubles); writes the final parameters in the same
// concatenated order (floats).
int ref_adam_steps(std::size_t catalog, std::size_t hidden, uint64_t seed, double lr, double b1,
                   double b2, double eps, int steps, const double* grads, float* params_out) {
  return guard([&] {
    ToyEncoderParams p = ToyEncoderParams::Init(catalog, hidden, SplitMix64(seed));
    AdamConfig cfg;
    cfg.lr = lr;
    cfg.beta1 = b1;
    cfg.beta2 = b2;
    cfg.eps = eps;
    AdamState adam(catalog, hidden, cfg);
    const std::size_t ne = catalog * hidden, nw = hidden * hidden, nb = hidden, nc = hidden * catalog;
    const std::size_t block = ne + nw + nb + nc;
    for (int s = 0; s < steps; ++s) {
      EncoderGrads g(catalog, hidden);
      const double* src = grads + static_cast<std::size_t>(s) * block;
      std::memcpy(g.d_emb.data().data(), src, sizeof(double) * ne);
      std::memcpy(g.d_w.data().data(), src + ne, sizeof(double) * nw);
      std::memcpy(g.d_b.data(), src + ne + nw, sizeof(double) * nb);
      std::memcpy(g.d_classifier.data().data(), src + ne + nw + nb, sizeof(double) * nc);
      adam.step(p, g);
    }
    std::memcpy(params_out, p.emb.data().data(), sizeof(float) * ne);
    std::memcpy(params_out + ne, p.w.data().data(), sizeof(float) * nw);
    std::memcpy(params_out + ne + nw, p.b.data(), sizeof(float) * nb);
    std::memcpy(params_out + ne + nw + nb, p.c.data().data(), sizeof(float) * nc);
  });
}

// encode_batch + encoder_backward (encoder.cpp:64-173) on caller-supplied
// parameters and windows (CSR), with d_h supplied; outputs as oracle.h.
int ref_encoder(std::size_t catalog, std::size_t hidden, const float* emb, const float* W,
                const float* b, const int64_t* items, const int64_t* win_off, std::size_t n_windows,
                const double* dh, double* a, double* h, float* e, int64_t* targets, double* d_emb,
                double* d_W, double* d_b) {
  return guard([&] {
    ToyEncoderParams p;
    p.emb = to_matrix(emb, catalog, hidden);
    p.w = to_matrix(W, hidden, hidden);
    p.b.assign(b, b + hidden);
    p.c = DenseMatrix(hidden, catalog);
    std::vector<std::vector<int64_t>> windows(n_windows);
    for (std::size_t w = 0; w < n_windows; ++w) windows[w].assign(items + win_off[w], items + win_off[w + 1]);
    const EncodedBatch enc = encode_batch(p, windows);
    const std::size_t rows = enc.e.rows();
    std::memcpy(a, enc.a.data().data(), sizeof(double) * rows * hidden);
    std::memcpy(h, enc.h.data().data(), sizeof(double) * rows * hidden);
    std::memcpy(e, enc.e.data().data(), sizeof(float) * rows * hidden);
    std::memcpy(targets, enc.targets.data(), sizeof(int64_t) * rows);
    DenseMatrixD dhm(rows, hidden);
    std::memcpy(dhm.data().data(), dh, sizeof(double) * rows * hidden);
    EncoderGrads g(catalog, hidden);
    encoder_backward(p, windows, enc, dhm, g);
    std::memcpy(d_emb, g.d_emb.data().data(), sizeof(double) * catalog * hidden);
    std::memcpy(d_W, g.d_w.data().data(), sizeof(double) * hidden * hidden);
    std::memcpy(d_b, g.d_b.data(), sizeof(double) * hidden);
  });
}

// The initial parameters of ToyEncoderParams::Init in the same concatenated order.
int ref_encoder_init(std::size_t catalog, std::size_t hidden, uint64_t seed, float* params_out) {
  return guard([&] {
    const ToyEncoderParams p = ToyEncoderParams::Init(catalog, hidden, SplitMix64(seed));
    const std::size_t ne = catalog * hidden, nw = hidden * hidden, nb = hidden;
    std::memcpy(params_out, p.emb.data().data(), sizeof(float) * ne);
    std::memcpy(params_out + ne, p.w.data().data(), sizeof(float) * nw);
    std::memcpy(params_out + ne + nw, p.b.data(), sizeof(float) * nb);
    std::memcpy(params_out + ne + nw + nb, p.c.data().data(), sizeof(float) * hidden * catalog);
  });
}

}  // extern "C"
