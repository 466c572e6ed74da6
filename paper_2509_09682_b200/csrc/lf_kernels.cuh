// lf_kernels.cuh — internal launcher declarations shared by the C-ABI layer.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "lf_internal.cuh"

namespace lf {

// Per-(chunk,row) forward partial: running max m, rescaled sum s, target
// logit t and a has-target flag.  SIMT path: natural-log units; tensor-core
// path: float, log2 units (m = max logit * log2 e, s = sum 2^(o log2e - m)).
template <class T>
struct alignas(sizeof(T) * 4) Partial {
  T m, s, t, has;
};

// ---- SIMT (lf_simt.cu) ----
template <class T>
int simt_cce_forward_full(const T* X, const T* E, const int64_t* targets, int64_t n, int D,
                          int64_t v, double* lse, double* pos, double* loss, cudaStream_t st);
template <class T>
int simt_cce_forward_partial_log2(const T* X, const T* E, const int64_t* targets, int64_t n,
                                  int D, int64_t v, int64_t v_offset, float* out,
                                  cudaStream_t st);
template <class T>
int simt_cce_backward(const T* X, const T* E, const int64_t* targets, const double* lse,
                      double scale, double eps, int64_t n, int D, int64_t v, int64_t v_offset,
                      T* dX, T* dE, unsigned long long* skip_counter, cudaStream_t st);

// Fused forward + dX (fp32, filter off) then the dE pass: lse, pos, loss
// (optional), dX, dE in one call (lf_cce_forward_backward).
int simt_cce_fused_f32(const float* X, const float* E, const int64_t* targets, int64_t n, int D, int64_t v,
                       double scale, double eps, double* lse, double* pos, double* loss, float* dX, float* dE,
                       cudaStream_t st);

int launch_combine_f32log2(const float* part, int P, int64_t n, double* lse, double* pos,
                           double* loss, cudaStream_t st);
int launch_reduce_f32(const float* part, int P, int64_t count, float* out, cudaStream_t st);
int launch_fold_partials(const float* part, int P, int64_t n, float* out, cudaStream_t st);
int launch_negate(float* x, int64_t count, cudaStream_t st);
int launch_mean_loss(const double* lse, const double* pos, int64_t n, double* loss,
                     cudaStream_t st);

// ---- tensor-core bf16 path (lf_tc.cu) ----
// Forward partials over the local shard: writes float4 log2-unit partials
// into `part` (P blocks of n), returns P via *P_out.
int tc_cce_forward_partials(const void* X, const void* E, const int64_t* targets, int64_t n,
                            int D, int64_t v, int64_t v_offset, Scratch& ws, float** part_out,
                            int* P_out, cudaStream_t st);
// Peer-memory exchange target (lf_peer.cu): rank `rank`'s contribution goes to
// slot [rank] of every peer's buffer (peers: device array of `world`
// pointers), offset by parity_off floats (epoch double-buffering).
struct PeerPush {
  float* const* peers;
  int world, rank;
  int64_t parity_off;
};
int peer_fold_push(const float* part, int P, int64_t n, float* const* peers, int world, int rank,
                   int64_t parity_off_floats, cudaStream_t st);
int peer_reduce_push(const float* part, int P, int64_t count, float* const* peers, int world, int rank,
                     int64_t parity_off_floats, cudaStream_t st);

// With `push`, dX is not reduced into dX: the V-chunk reduction is fused with
// the store of the rank's dX partial into every peer's slot (dX is scratch).
// dX == nullptr: dE pass only (the fused forward produced dX); the skip
// statistics are then counted by the dE pass.
int tc_cce_backward(const void* X, const void* E, const int64_t* targets, const double* lse,
                    double scale, double eps, int64_t n, int D, int64_t v, int64_t v_offset,
                    float* dX, float* dE, unsigned long long* counters, cudaStream_t st,
                    const PeerPush* push = nullptr);

// Fused forward + unnormalised dX (FWDX mode; bf16, D = 64 / 128 only:
// tc_fwdx_supported).  part: [P][n] float4 {m, s, t, has} in log2 units;
// opart: [P][n][D] fp32 O = sum_j 2^(logit log2e - m) E_j over the chunk;
// tgt: local target index per row (-1 outside the shard).
int tc_fwdx_supported(int D);
int tc_cce_fwdx_partials(const void* X, const void* E, const int64_t* targets, int64_t n, int D,
                         int64_t v, int64_t v_offset, Scratch& part, Scratch& opart, Scratch& tgt,
                         int* P_out, cudaStream_t st);
// dX = scale (sum_p O_p 2^(m_p - lse2) - E_t) from those partials; lse_in ==
// nullptr: lse2 from the partials themselves, lse_out / pos_out written.
int tc_fwdx_dx(const float* part, const float* opart, int P, int64_t n, int D, const double* lse_in,
               const void* E, const int32_t* tgt, double scale, double* lse_out, double* pos_out,
               float* dX, cudaStream_t st);

// EVAL-mode partials over the shard (bf16): Et = the rows' target item rows
// (ceil(n/128)*128 rows), tl = clamped local target index; per (chunk, row)
// count (uint32), top-16 values (float) and local indices (int32).
int tc_eval_partials(const void* X, const void* E, const void* Et, const int32_t* tl, int64_t n,
                     int D, int64_t v, int k, Scratch& cnt, Scratch& val, Scratch& idx, int* P_out,
                     int* K_out, cudaStream_t st);
// Same for fp32 / fp64 (lf_simt.cu), top-K per chunk with K = k.
template <class T>
int simt_eval_partials(const T* X, const T* E, const T* Et, const int32_t* tl, int64_t n, int D,
                       int64_t v, int K, Scratch& cnt, Scratch& val, Scratch& idx, int* P_out,
                       cudaStream_t st);

// ---- full-catalog evaluation (lf_eval.cu) ----
int eval_rank_topk(int dtype, const void* X, const void* E, const int64_t* targets,
                   const void* target_rows, int64_t n, int D, int64_t v, int64_t v_offset, int k,
                   int64_t* ahead, int64_t* top_idx, double* top_score, cudaStream_t st);
int eval_merge(const int64_t* ahead, const int64_t* top_idx, const double* top_score, int P,
               int64_t n, int k, int64_t* rank, int64_t* top_idx_out, double* top_score_out,
               cudaStream_t st);
int launch_add_one(int64_t* x, int64_t n, cudaStream_t st);
int eval_summary(const int64_t* rank, const int64_t* top_idx, int64_t n, int k, const int64_t* pop,
                 int64_t v, double* out3_host, cudaStream_t st);

// ---- encoder (lf_encoder.cu) ----
int encode_batch(const int64_t* items, const int64_t* win_off, int64_t n_windows, const float* emb,
                 const float* W, const float* bias, int64_t catalog, int D, int64_t rows, int x_dtype,
                 void* X, double* a, double* h, int64_t* targets, int64_t* row_window,
                 int64_t* row_pos, cudaStream_t st);
int encoder_backward(const int64_t* items, const int64_t* win_off, int64_t n_windows, const float* W,
                     int64_t catalog, int D, const double* a, const double* h, const int64_t* row_pos,
                     int64_t rows, const void* dh, int dh_dtype, double* d_emb, double* dW, double* db,
                     cudaStream_t st);

// ---- optimizer (lf_adam.cu) ----
int adam_step(float* param, const void* grad, int grad_dtype, double* m, double* v, int64_t n,
              double lr, double b1, double b2, double eps, int64_t t, void* shadow, int shadow_dtype,
              cudaStream_t st);

// ---- CCE- (lf_ccem.cu) ----
int ccem_forward(int dtype, const void* X, const void* E, const int64_t* inds, int64_t n, int D,
                 int64_t v, int64_t w, double* lse, double* pos, double* loss, cudaStream_t st);
int ccem_backward(int dtype, const void* X, const void* E, const int64_t* inds,
                  const double* lse, const double* row_upstream, double upstream, int64_t n,
                  int D, int64_t v, int64_t w, bool atomic_de, void* dX, void* dE,
                  cudaStream_t st);
bool ccem_fused_supported(int dtype, int D, bool atomic_de);
int ccem_forward_backward(int dtype, const void* X, const void* E, const int64_t* inds, int64_t n,
                          int D, int64_t v, int64_t w, const double* row_upstream, double upstream,
                          double* lse, double* pos, double* loss, void* dX, void* dE, cudaStream_t st);

// Stable counting-by-radix sort of `count` entries by item (inds[i] in
// [0, v)): sorted_vals = entry indices grouped by item in index order,
// item_off[v + 1] = segment offsets (lf_ccem.cu).
int sort_by_item(const int64_t* inds, int64_t count, int64_t v, Scratch& sorted_vals,
                 Scratch& item_off, cudaStream_t st, const uint32_t* gate = nullptr);

// ---- materialising CE baseline (lf_ce.cu; cuBLAS GEMMs) ----
int ce_forward(int dtype, const void* X, const void* E, const int64_t* targets, int64_t n, int D,
               int64_t v, double* lse, double* pos, double* loss, cudaStream_t st);
int ce_backward(int dtype, const void* X, const void* E, const int64_t* targets, double upstream,
                int64_t n, int D, int64_t v, void* dX, void* dE, cudaStream_t st);
int cem_forward(int dtype, const void* X, const void* E, const int64_t* inds, int64_t n, int D, int64_t w,
                double* lse, double* pos, double* loss, cudaStream_t st);
int cem_backward(int dtype, const void* X, const void* E, const int64_t* inds, double upstream, int64_t n,
                 int D, int64_t v, int64_t w, void* dX, void* dE, cudaStream_t st);

// ---- negative sampler (lf_sampler.cu) ----
int sample_uniform(const int64_t* positives, int64_t n, int64_t ns, int64_t catalog,
                   uint64_t seed, int retry_cap, int64_t* inds, cudaStream_t st);
int sample_popularity(const int64_t* positives, int64_t n, int64_t ns, const int64_t* counts,
                      int64_t catalog, double exponent, uint64_t seed, int retry_cap, int64_t* inds,
                      cudaStream_t st);

// ---- validation (lf_ccem.cu) ----
int validate_targets(const int64_t* targets, int64_t n, int64_t v, cudaStream_t st);
int validate_inds(const int64_t* inds, int64_t n, int64_t w, int64_t v, cudaStream_t st);

// ---- boundary layouts (lf_layout.cu) ----
int layout_classifier_to_items(const float* C, int64_t d, int64_t v, int dtype, void* E,
                               cudaStream_t st);
int layout_convert_rows(const float* src, int64_t count, int dtype, void* dst, cudaStream_t st);
int layout_items_grad_to_classifier(const void* dE, int grad_dtype, int64_t v, int64_t d,
                                    double* dC, cudaStream_t st);
int layout_widen(const void* src, int grad_dtype, int64_t count, double* dst, cudaStream_t st);

}  // namespace lf
