/*
 * lseforge_b200.h — C-ABI of the B200-native (sm_100a) CCE / CCE- loss path.
 *
 * This is the drop-in boundary for the reference library's hot path
 * (lseforge, /root/reference/proj).  Each entry point replaces one reference
 * C++ function; the citation is given beside it.  Plain pointers and sizes
 * only; every pointer named `d_*` is DEVICE memory on the current CUDA device,
 * every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 * default stream) and does not synchronize unless documented.
 *
 * Layout (B200 naming; the reference's letters are swapped):
 *   X  [n x d]  hidden states, row-major       (reference "E", cce.hpp:36)
 *   E  [v x d]  item embeddings, row-major     (reference "C" is d x v = E^T)
 *   targets [n] int64, item index of each row's positive (reference "x")
 *   inds [n x w] int64, slot 0 = positive, w = 1 + K (NegIndexMatrix,
 *                neg_index.hpp:10-44)
 *   lse, pos [n] double (LossOutput::lse / pos_logits, losses.hpp:15-19)
 *   dX [n x d], dE [v x d]: float (dtype bf16/f32) or double (dtype f64)
 *                (GradPair, losses.hpp:24-27; dE = reference d_classifier^T)
 *
 * Element types (lf_dtype):
 *   LF_BF16 — tcgen05/TMEM/TMA tensor-core kernels, fp32 accumulate
 *             (requires d % 64 == 0, d <= 256)
 *   LF_F32  — fp32 SIMT (FFMA) kernels, any d
 *   LF_F64  — "exact" mode: fp64, reference operand order (k ascending,
 *             no FMA contraction) so pos logits are bitwise equal to the
 *             reference's double results for float-representable inputs.
 *
 * Status: every function returns 0 on success or a negative LF_E* code;
 * lf_last_error() returns a thread-local message (the reference's
 * std::invalid_argument text where one exists, e.g. "loss: row 1 targets item
 * 9, outside catalog of 8" — losses.cpp:59-66).
 */
#ifndef LSEFORGE_B200_H
#define LSEFORGE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LF_ABI_VERSION 1

#if defined(__GNUC__)
#define LF_API __attribute__((visibility("default")))
#else
#define LF_API
#endif

enum lf_status {
  LF_OK = 0,
  LF_EINVAL = -1,      /* bad argument (shape, range, config) */
  LF_EUNSUPPORTED = -2, /* valid request this build cannot serve (e.g. bf16 with d % 64) */
  LF_ECUDA = -3,       /* CUDA runtime / driver error */
  LF_ENOMEM = -4,
  LF_ERUNTIME = -5     /* the reference's std::runtime_error cases (e.g. sampler retry cap) */
};

enum lf_dtype { LF_F32 = 0, LF_F64 = 1, LF_BF16 = 2 };

/* Mirrors lseforge::CceConfig (cce.hpp:18-31).  row_block / col_block /
 * workers are CPU tiling knobs with no effect on results; they are accepted
 * and ignored (the GPU picks its own tiles, and results are bitwise identical
 * run to run for any value, matching test_cce.cpp:170-196). */
typedef struct {
  double filter_eps; /* CceConfig::filter_eps; 0 = exact backward (cce.hpp:21) */
  int32_t dtype;     /* lf_dtype of X and E */
  int32_t flags;     /* LF_FLAG_* */
} lf_cce_config;

#define LF_FLAG_NONE 0
/* CCE-: accumulate dE with red.global.add (non-deterministic bit order)
 * instead of the default deterministic bucket + ordered segment reduce. */
#define LF_FLAG_ATOMIC_DE 1
/* lf_cce_forward_backward: apply the filter to dX as well (separate dX pass,
 * 3 exps per logit instead of 2). */
#define LF_FLAG_FILTER_DX 2

/* Backward statistics (device-side counters are copied into this host struct
 * only when the caller passes a non-NULL pointer; that forces a stream sync). */
typedef struct {
  uint64_t skipped_elems;  /* off-target (row,item) pairs with softmax < eps (cce.cpp:197-200) */
  uint64_t skipped_tiles;  /* bf16: 32-row x 32-item sub-tiles of the dX pass whose exps were
                              skipped (every entry below eps; only tested while such
                              sub-tiles keep appearing — see DESIGN.md) */
  uint64_t total_tiles;    /* bf16: 32 x 32 sub-tiles visited by the dX pass */
  double skipped_fraction; /* skipped_elems / (n * (v_total - 1)), cce.cpp:264-268 */
} lf_cce_stats;

LF_API int lf_abi_version(void);
LF_API const char* lf_last_error(void);

/* ---------------------------------------------------------------- CCE ---- */

/* Replaces lseforge::cce_forward (cce.hpp:36-38, cce.cpp:65-145).
 * Writes d_lse[n], d_pos[n] and the mean loss d_loss[0] (all double). */
LF_API int lf_cce_forward(const void* d_X, const void* d_E, const int64_t* d_targets, int64_t n,
                   int64_t d, int64_t v, const lf_cce_config* cfg, double* d_lse, double* d_pos,
                   double* d_loss, void* stream);

/* Replaces lseforge::cce_backward (cce.hpp:51-54, cce.cpp:147-272) with
 * upstream = dL/dloss (scale = upstream / n, cce.cpp:174).  d_dX [n x d] and
 * d_dE [v x d] are OVERWRITTEN (the reference returns fresh zeroed matrices).
 * stats may be NULL (no sync). */
LF_API int lf_cce_backward(const void* d_X, const void* d_E, const int64_t* d_targets,
                    const double* d_lse, double upstream, int64_t n, int64_t d, int64_t v,
                    const lf_cce_config* cfg, void* d_dX, void* d_dE, lf_cce_stats* stats,
                    void* stream);

/* Fused cce_forward + cce_backward: the pair run_loss_layer issues back to
 * back on the same inputs (trainer.cpp:71-77, forward then backward with the
 * forward's lse).  Writes everything lf_cce_forward and lf_cce_backward
 * write.  For bf16 with d = 64 / 128 / 256 and filter_eps < 2^-12 it runs the
 * fused kernel: one pass over the logits computes the LSE AND the
 * softmax-weighted item sum of dX (2 exps per logit instead of 3), then the
 * item-owned dE pass.  That dX is the exact (unfiltered) softmax - onehot
 * gradient — the filter drops entries below eps, so the two differ by less
 * than eps per entry, and not at all for eps = 0 — while dE and the skip
 * statistics follow the filter exactly.  LF_FLAG_FILTER_DX (or any other
 * dtype / d / eps) runs the separate forward and backward instead. */
LF_API int lf_cce_forward_backward(const void* d_X, const void* d_E, const int64_t* d_targets,
                                   int64_t n, int64_t d, int64_t v, double upstream,
                                   const lf_cce_config* cfg, double* d_lse, double* d_pos,
                                   double* d_loss, void* d_dX, void* d_dE, lf_cce_stats* stats,
                                   void* stream);

/* ------------------------------------------------ catalog-sharded CCE ---- */
/* Rank p owns E rows [v_offset, v_offset + v_shard) of a catalog of v_total
 * items; targets are GLOBAL item indices.  Forward: per-row partial triples
 * d_part[n] = {m (max logit * log2 e), s (sum of 2^(logit*log2e - m)),
 * t (target logit if the target lies in this shard, else 0), has_t} as float4;
 * exchange them across ranks (e.g. one ncclAllGather of n*16 bytes), then
 * lf_cce_combine over the P gathered blocks gives lse/pos/loss. */
LF_API int lf_cce_forward_partial(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                           int64_t n, int64_t d, int64_t v_shard, int64_t v_offset,
                           const lf_cce_config* cfg, float* d_part, void* stream);

/* d_parts: P consecutive blocks of n float4 partials. */
LF_API int lf_cce_combine(const float* d_parts, int32_t P, int64_t n, double* d_lse, double* d_pos,
                   double* d_loss, void* stream);

/* Sharded backward: dE rows for the local shard are complete; dX is this
 * shard's PARTIAL sum over its items and must be summed across ranks
 * (ncclAllReduce sum of n*d floats).  scale = upstream / n. */
LF_API int lf_cce_backward_shard(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                          const double* d_lse, double upstream, int64_t n, int64_t d,
                          int64_t v_shard, int64_t v_offset, int64_t v_total,
                          const lf_cce_config* cfg, void* d_dX_partial, void* d_dE_shard,
                          lf_cce_stats* stats, void* stream);

/* ------------------------------- catalog sharding from C / C++ ---------- */
/* The reference's only production caller of the loss (run_loss_layer,
 * trainer.cpp:59-110) is C++; these entries let it shard the catalog over
 * GPUs without PyTorch.  lf_comm is a stream-ordered communicator: an
 * all-gather of `bytes` per rank (rank order) and an in-place float sum
 * all-reduce.  Backends: NCCL (lf_comm_nccl: wraps an ncclComm_t the caller
 * created, libnccl.so.2 bound at run time) and peer memory over CUDA IPC
 * (lf_peer_comm_*: every rank maps every rank's exchange buffer; on an
 * NVSwitch box the stores travel over NVLink).  Any other transport can
 * fill the two callbacks itself. */
typedef struct lf_comm {
  void* ctx;
  int32_t world, rank;
  int (*allgather)(void* ctx, const void* d_send, void* d_recv, uint64_t bytes, void* stream);
  int (*allreduce_sum_f32)(void* ctx, float* d_buf, uint64_t count, void* stream);
} lf_comm;

/* 1 if lf_cce_forward_backward (and the sharded variant) run the fused
 * forward + dX kernel for this config and width, else 0. */
LF_API int lf_cce_fused_supported(const lf_cce_config* cfg, int64_t d);

/* nccl_comm: an ncclComm_t of `world` ranks (this process = `rank`). */
LF_API int lf_comm_nccl(void* nccl_comm, int32_t world, int32_t rank, lf_comm* out);

/* Peer-memory communicator.  create: allocate this rank's exchange buffer
 * (two epoch halves of `world` slots of slot_bytes) and flags, export
 * lf_peer_comm_handle_bytes() bytes of CUDA IPC handles into handle_out;
 * the caller gathers every rank's handle block in rank order (any
 * bootstrap), then open maps them and fills `out`.  Barriers are bounded:
 * a peer that never arrives (LSEFORGE_PEER_TIMEOUT_MS, default 60 s) or
 * raises lf_peer_comm_abort releases the others, and lf_peer_comm_status
 * then reports LF_ERUNTIME instead of every rank spinning forever. */
typedef struct lf_peer_comm lf_peer_comm;
LF_API uint64_t lf_peer_comm_handle_bytes(void);
LF_API int lf_peer_comm_create(uint64_t slot_bytes, int32_t world, int32_t rank, lf_peer_comm** out,
                               void* handle_out);
LF_API int lf_peer_comm_open(lf_peer_comm* pc, const void* all_handles, lf_comm* out);
LF_API int lf_peer_comm_abort(lf_peer_comm* pc, void* stream);
LF_API int lf_peer_comm_status(void);
LF_API int lf_peer_comm_destroy(lf_peer_comm* pc);

/* cce_forward over a catalog shard E [v_shard x d] = items [v_offset,
 * v_offset + v_shard) of the full catalog, targets GLOBAL: local partials,
 * one all-gather of n float4, combine -> every rank holds lse / pos / loss. */
LF_API int lf_cce_forward_sharded(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                                  int64_t n, int64_t d, int64_t v_shard, int64_t v_offset,
                                  const lf_cce_config* cfg, const lf_comm* comm, double* d_lse,
                                  double* d_pos, double* d_loss, void* stream);
/* cce_backward over the shard: dE rows of the shard; dX summed over ranks
 * (one all-reduce of n x d floats; bf16 / f32).  stats: this rank's counts
 * (skipped_fraction of the GLOBAL n (v_total - 1): sum it over ranks). */
LF_API int lf_cce_backward_sharded(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                                   const double* d_lse, double upstream, int64_t n, int64_t d,
                                   int64_t v_shard, int64_t v_offset, int64_t v_total,
                                   const lf_cce_config* cfg, const lf_comm* comm, void* d_dX,
                                   void* d_dE_shard, lf_cce_stats* stats, void* stream);
/* Both, fused when lf_cce_fused_supported (one pass over the shard's logits
 * for the LSE partials and dX's item sum, the all-gather, dX normalised by
 * the global lse, the dE pass, the dX all-reduce). */
LF_API int lf_cce_forward_backward_sharded(const void* d_X, const void* d_E_shard,
                                           const int64_t* d_targets, int64_t n, int64_t d,
                                           int64_t v_shard, int64_t v_offset, int64_t v_total,
                                           double upstream, const lf_cce_config* cfg,
                                           const lf_comm* comm, double* d_lse, double* d_pos,
                                           double* d_loss, void* d_dX, void* d_dE_shard,
                                           lf_cce_stats* stats, void* stream);
/* The fused sharded step in two phases, for callers with their own
 * collectives (e.g. torch.distributed): begin writes this shard's folded
 * partials d_part[n] (float4 {m, s, t, has}, log2 units) and keeps the dX
 * partials in *work; gather the ranks' d_part blocks (rank order) and call
 * end, which writes lse / pos / loss, this shard's dX PARTIAL (sum it over
 * ranks) and dE rows, and releases *work (lf_cce_work_free on abandon). */
typedef struct lf_cce_work lf_cce_work;
LF_API int lf_cce_fwdx_shard_begin(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                                   int64_t n, int64_t d, int64_t v_shard, int64_t v_offset,
                                   const lf_cce_config* cfg, float* d_part, lf_cce_work** work,
                                   void* stream);
LF_API int lf_cce_fwdx_shard_end(lf_cce_work* work, const float* d_parts, int32_t P, double upstream,
                                 int64_t v_total, double* d_lse, double* d_pos, double* d_loss,
                                 void* d_dX_partial, void* d_dE_shard, lf_cce_stats* stats,
                                 void* stream);
LF_API int lf_cce_work_free(lf_cce_work* work);

/* ------------------------------- catalog sharding over peer memory ---- */
/* The same two exchanges without NCCL: each rank maps every peer's exchange
 * buffer (CUDA IPC: lf_peer_alloc exports a cudaMalloc'd buffer as a 64-byte
 * handle, the handles are exchanged by the caller, lf_peer_open maps them) and
 * the producing kernel stores its contribution straight into slot [rank] of
 * every peer's buffer (d_peer_*: DEVICE array of `world` pointers, this
 * rank's own buffer at index rank; parity_off = element offset of the
 * epoch-parity half, so consecutive exchanges alternate halves).
 *   forward:  lf_cce_forward_partial_peer — the per-chunk partial fold fused
 *             with the all-gather; each buffer holds [world][n] float4 —
 *             then lf_peer_barrier, then lf_cce_combine on the local block.
 *   backward: lf_cce_backward_shard_peer — the dX V-chunk reduction fused with
 *             the all-gather of the rank's partial ([world][n x d] floats),
 *             then lf_peer_barrier, then lf_peer_sum (fixed rank order: every
 *             rank gets identical bits).  bf16 / f32. */
LF_API int lf_peer_alloc(uint64_t bytes, void** d_ptr, void* ipc_handle /* 64 bytes out */);
LF_API int lf_peer_open(const void* ipc_handle, void** d_ptr);
LF_API int lf_peer_close(void* d_ptr);
LF_API int lf_peer_free(void* d_ptr);
/* Signal every peer (d_peer_flags: device array of `world` pointers to each
 * rank's uint32 flag array of `world` entries) that this rank's stores for
 * `epoch` are done, then wait (stream-ordered, on the device) for all peers'. */
LF_API int lf_peer_barrier(uint32_t* const* d_peer_flags, int32_t world, int32_t rank, uint32_t epoch,
                           void* stream);
/* The barrier waits at most LSEFORGE_PEER_TIMEOUT_MS (default 60 s) per peer
 * and then gives up instead of hanging the GPU; lf_peer_status returns
 * LF_ERUNTIME if any barrier of this process gave up (synchronizes). */
LF_API int lf_peer_status(void);
LF_API int lf_peer_sum(const float* d_slots, int32_t world, int64_t count, float* d_out, void* stream);
LF_API int lf_cce_forward_partial_peer(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                                       int64_t n, int64_t d, int64_t v_shard, int64_t v_offset,
                                       const lf_cce_config* cfg, float* const* d_peer_parts,
                                       int32_t world, int32_t rank, int64_t parity_off, void* stream);
LF_API int lf_cce_backward_shard_peer(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                                      const double* d_lse, double upstream, int64_t n, int64_t d,
                                      int64_t v_shard, int64_t v_offset, int64_t v_total,
                                      const lf_cce_config* cfg, void* d_dE_shard, lf_cce_stats* stats,
                                      float* const* d_peer_dx, int32_t world, int32_t rank,
                                      int64_t parity_off, void* stream);

/* ---------------------------------------------------------------- CCE- --- */

/* Replaces lseforge::ccem_forward (ccem.hpp:19-20, ccem.cpp:48-105). */
LF_API int lf_ccem_forward(const void* d_X, const void* d_E, const int64_t* d_inds, int64_t n,
                    int64_t d, int64_t v, int64_t w, const lf_cce_config* cfg, double* d_lse,
                    double* d_pos, double* d_loss, void* stream);

/* Replaces lseforge::ccem_backward_rows (ccem.hpp:34-36, ccem.cpp:107-194):
 * d_row_upstream[n] (double).  Passing d_row_upstream == NULL means the scalar
 * form lseforge::ccem_backward (ccem.hpp:27-29): row_upstream[i] = upstream/n.
 * Gradient filtering does not apply to CCE- (ccem.hpp:22-26).  d_dX and d_dE
 * are OVERWRITTEN; d_dE is full width (v x d) with exact zeros for untouched
 * items. */
LF_API int lf_ccem_backward(const void* d_X, const void* d_E, const int64_t* d_inds, const double* d_lse,
                     const double* d_row_upstream, double upstream, int64_t n, int64_t d,
                     int64_t v, int64_t w, const lf_cce_config* cfg, void* d_dX, void* d_dE,
                     void* stream);

/* Fused CCE- forward + backward: lf_ccem_forward followed by lf_ccem_backward
 * with the same upstream (the trainer's pairing, trainer.cpp:71-77 —
 * run_loss_layer always calls the backward right after the forward on the
 * same inputs), in ONE gather pass over the candidates' rows instead of two:
 * the pass keeps an online-softmax-weighted row sum per row, so lse, pos, dX
 * and each entry's logit come out together; the dE coefficients are formed
 * from the logits and reduced as in lf_ccem_backward (bitwise the same dE).
 * bf16 / f32 with d in {64, 128, 256} and without LF_FLAG_ATOMIC_DE run
 * fused; anything else runs the two calls in sequence.  d_row_upstream may be
 * NULL (scalar form).  d_loss may be NULL. */
LF_API int lf_ccem_forward_backward(const void* d_X, const void* d_E, const int64_t* d_inds,
                                    int64_t n, int64_t d, int64_t v, int64_t w,
                                    const double* d_row_upstream, double upstream,
                                    const lf_cce_config* cfg, double* d_lse, double* d_pos,
                                    double* d_loss, void* d_dX, void* d_dE, void* stream);

/* ------------------------------------------- materialising CE baseline ---- */
/* Replace lseforge::ce_full_forward / ce_full_backward (losses.cpp:71-140):
 * the baseline CCE is measured against.  The n x v logit matrix IS written
 * to device memory (fp32; fp64 for LF_F64) by a cuBLAS GEMM, plus a n x v
 * coefficient matrix in the backward — peak scratch ~6 n v bytes for bf16.
 * Same outputs and layouts as lf_cce_forward / lf_cce_backward (no filter). */
LF_API int lf_ce_forward(const void* d_X, const void* d_E, const int64_t* d_targets, int64_t n,
                         int64_t d, int64_t v, const lf_cce_config* cfg, double* d_lse,
                         double* d_pos, double* d_loss, void* stream);
LF_API int lf_ce_backward(const void* d_X, const void* d_E, const int64_t* d_targets,
                          double upstream, int64_t n, int64_t d, int64_t v,
                          const lf_cce_config* cfg, void* d_dX, void* d_dE, void* stream);

/* Replace lseforge::ce_sampled_forward / ce_sampled_backward (losses.cpp:142-221):
 * the materialising CE- baseline (backend "cem").  The n x w candidate logits
 * ARE written to device memory (and G over them in the backward); dE is
 * scattered with atomics (duplicate candidates accumulate).  Same outputs and
 * layouts as lf_ccem_forward / lf_ccem_backward (d_inds: n x w, slot 0 = positive). */
LF_API int lf_cem_forward(const void* d_X, const void* d_E, const int64_t* d_inds, int64_t n,
                          int64_t d, int64_t v, int64_t w, const lf_cce_config* cfg, double* d_lse,
                          double* d_pos, double* d_loss, void* stream);
LF_API int lf_cem_backward(const void* d_X, const void* d_E, const int64_t* d_inds, double upstream,
                           int64_t n, int64_t d, int64_t v, int64_t w, const lf_cce_config* cfg,
                           void* d_dX, void* d_dE, void* stream);

/* ------------------------------------------------------- negative sampler -- */
/* Replaces lseforge::sample_uniform (sampler.hpp, sampler.cpp:44-75) with a
 * device restatement that produces the SAME indices: row i draws from
 * SplitMix64(seed).derived(i) (rng.hpp:46-48; only the generator's
 * construction seed matters), slot 0 = positives[i], slots 1..ns = the next
 * in-catalog draws that differ from the positive; retry_cap consecutive
 * positive draws in one slot -> LF_ERUNTIME with the reference's message.
 * Writes d_inds[n x (1 + ns)] (int64, the NegIndexMatrix layout CCE- takes).
 * Synchronizes `stream` (validation and the retry-cap status). */
LF_API int lf_sample_uniform(const int64_t* d_positives, int64_t n, int64_t ns, int64_t catalog,
                             uint64_t seed, int32_t retry_cap, int64_t* d_inds, void* stream);

/* ------------------------------------------- full-catalog evaluation ---- */
/* The scoring and ranking of lseforge::evaluate (metrics.hpp:18-24,
 * metrics.cpp:13-103) on the device; the encoder that produces h
 * (metrics.cpp:46) is the caller's, d_X holds the encoded rows.  Scores
 * s_ij = X_i . E_j are never materialised.
 *
 * lf_eval_rank_topk: over the catalog shard E [v_shard x d] holding items
 * [v_offset, v_offset + v_shard), d_targets GLOBAL item ids:
 *   d_ahead[i]            = #{shard items j : s_ij > s_it, or s_ij == s_it and
 *                           j < t} (metrics.cpp:56-60; rank = 1 + the sum over shards)
 *   d_top_idx[i*k + e]    = the shard's top-k items by (score desc, id asc)
 *                           (metrics.cpp:63-72), global ids, -1 past the shard size
 *   d_top_score[i*k + e]  = their scores (double).
 * The target score s_it is computed on the same arithmetic path as the
 * scores it is compared with: from d_target_rows [n x d] (the rows' target
 * item rows, in dtype) when given — needed when a target lives in another
 * shard — else gathered from E (every target must then be in the shard;
 * LF_EINVAL otherwise, after a stream sync).  f64 reproduces the reference's
 * double scores bit for bit (k ascending, metrics.cpp:49-54), so ranks and
 * lists are identical; bf16 runs on the tensor cores (fp32 scores).
 * k <= 16 (bf16) / 32 (f32, f64), else LF_EUNSUPPORTED. */
LF_API int lf_eval_rank_topk(const void* d_X, const void* d_E, const int64_t* d_targets,
                             const void* d_target_rows, int64_t n, int64_t d, int64_t v_shard,
                             int64_t v_offset, int32_t k, int32_t dtype, int64_t* d_ahead,
                             int64_t* d_top_idx, double* d_top_score, void* stream);
/* Merge P shards' outputs (P consecutive blocks of n / n*k): d_rank = 1 +
 * sum of ahead, merged global top-k. */
LF_API int lf_eval_merge(const int64_t* d_ahead, const int64_t* d_top_idx, const double* d_top_score,
                         int32_t P, int64_t n, int32_t k, int64_t* d_rank, int64_t* d_top_idx_out,
                         double* d_top_score_out, void* stream);
/* Aggregation of metrics.cpp:26-33, 62, 74-103 from 1-based ranks and the
 * top-k lists (k = k_eff): out3 (HOST) = {ndcg, coverage, surprisal}.
 * d_popularity: v_total training counts.  Synchronizes `stream`; LF_EINVAL
 * with the reference's messages for a negative count / fewer than 2 events. */
LF_API int lf_eval_summary(const int64_t* d_rank, const int64_t* d_top_idx, int64_t n, int32_t k,
                           const int64_t* d_popularity, int64_t v_total, double* out3,
                           void* stream);
/* lseforge::evaluate for an unsharded catalog: k_eff = min(k, v), rank/top-k,
 * then the summary into out3 (HOST). */
LF_API int lf_evaluate(const void* d_X, const void* d_E, const int64_t* d_targets, int64_t n,
                       int64_t d, int64_t v, int32_t k, int32_t dtype, const int64_t* d_popularity,
                       double* out3, void* stream);

/* ----------------------------------------------------------------- encoder -- */
/* encode_batch (encoder.hpp:46-60, encoder.cpp:64-116) on the device.  Windows
 * as a CSR: d_items[d_win_off[w] .. d_win_off[w+1]) is window w (every window
 * >= 2 items); rows = sum (len - 1), enumerated window by window, position
 * t = 1 .. len-1.  Params in the reference layout: d_emb [catalog x d],
 * d_W [d x d], d_b [d] (float).  Outputs: d_X [rows x d] = EncodedBatch::e
 * (float(h)) converted to x_dtype (the loss input), d_a / d_h [rows x d]
 * double (pooled means — bitwise the reference's — and tanh outputs), d_targets,
 * d_row_window, d_row_pos [rows].  Synchronizes (validation); LF_EINVAL with
 * the reference's messages. */
LF_API int lf_encode_batch(const int64_t* d_items, const int64_t* d_win_off, int64_t n_windows,
                           const float* d_emb, const float* d_W, const float* d_b, int64_t catalog,
                           int64_t d, int64_t rows, int32_t x_dtype, void* d_X, double* d_a,
                           double* d_h, int64_t* d_targets, int64_t* d_row_window,
                           int64_t* d_row_pos, void* stream);
/* encoder_backward (encoder.hpp:62-66, encoder.cpp:118-173): from d_h = the
 * loss's dX [rows x d] (f32 or f64) to d_emb [catalog x d], d_W [d x d],
 * d_b [d] (double, OVERWRITTEN — the reference accumulates into a fresh
 * EncoderGrads per batch, trainer.cpp:222-223), summed in the reference's
 * order. */
LF_API int lf_encoder_backward(const int64_t* d_items, const int64_t* d_win_off, int64_t n_windows,
                               const float* d_W, int64_t catalog, int64_t d, const double* d_a,
                               const double* d_h, const int64_t* d_row_pos, int64_t rows,
                               const void* d_dh, int32_t dh_dtype, double* d_demb, double* d_dW,
                               double* d_db, void* stream);

/* -------------------------------------------------------------- optimizer -- */
/* One step of AdamState::apply (adam.hpp:18-49, adam.cpp:22-36) over `count`
 * float parameters with double moments d_m / d_v (zero before step 1), the
 * gradient in f32 or f64 (grad_dtype), t = the 1-based step number (the
 * reference's t_ after its increment; bias corrections 1 - beta^t as in
 * adam.cpp:46-47).  Bitwise equal to the reference's parameters and moments.
 * Optionally also writes the new parameters to d_shadow in shadow_dtype
 * (LF_BF16 or LF_F32; pass NULL for none) — e.g. the bf16 E the next CCE
 * step reads — in the same pass.  Layout-agnostic (elementwise): apply it to
 * E [v x d] with dE [v x d] in the B200 layout.  LF_EINVAL with the
 * reference's messages for bad betas / eps. */
LF_API int lf_adam_step(float* d_param, const void* d_grad, int32_t grad_dtype, double* d_m,
                        double* d_v, int64_t count, double lr, double beta1, double beta2,
                        double eps, int64_t t, void* d_shadow, int32_t shadow_dtype, void* stream);

/* Replaces lseforge::sample_popularity (sampler.hpp, sampler.cpp:77-127):
 * inverse CDF over the running sum of count^exponent (d_counts: catalog
 * int64 training counts), row i from SplitMix64(seed).derived(i), one
 * uniform() per attempt, retry_cap failed attempts in a row -> LF_ERUNTIME.
 * Same indices as the reference for exponent == 1 (the running sums are exact
 * integers); for other exponents the device pow may differ in the last ulp.
 * LF_EINVAL with the reference's messages (negative count, positive outside
 * the catalog, ns too large, all weights zero).  Synchronizes `stream`. */
LF_API int lf_sample_popularity(const int64_t* d_positives, int64_t n, int64_t ns,
                                const int64_t* d_counts, int64_t catalog, double exponent,
                                uint64_t seed, int32_t retry_cap, int64_t* d_inds, void* stream);

/* ----------------------------------------------------------- validation --- */
/* Replaces validate_loss_inputs' index scan (losses.cpp:58-67) for device
 * targets.  Synchronizes `stream`.  On failure returns LF_EINVAL with the
 * reference's message naming the first offending row. */
LF_API int lf_validate_targets(const int64_t* d_targets, int64_t n, int64_t v, void* stream);
/* Replaces NegIndexMatrix::validate (neg_index.cpp:8-28). Synchronizes. */
LF_API int lf_validate_inds(const int64_t* d_inds, int64_t n, int64_t w, int64_t v, void* stream);

/* ------------------------------------------------------ boundary layouts -- */
/* For callers holding the reference's host layouts (the C++ drop-in,
 * paper_2509_09682_b200/shim/lseforge_shim.cpp).  Stream-ordered, no sync. */

/* ref-C (float d x v row-major, cce.hpp:36 "C") -> E (v x d row-major) in
 * `dtype` (exact for f32/f64, round-to-nearest-even for bf16). */
LF_API int lf_classifier_to_items(const float* d_C, int64_t d, int64_t v, int32_t dtype, void* d_E,
                                  void* stream);
/* Element conversion of a float buffer (ref-E, the hidden rows) to `dtype`. */
LF_API int lf_convert_rows(const float* d_src, int64_t count, int32_t dtype, void* d_dst,
                           void* stream);
/* dE (v x d, float for bf16/f32 inputs or double for f64 — the gradient type
 * of `dtype`) -> d_classifier (double d x v, GradPair::d_classifier,
 * losses.hpp:24-27). */
LF_API int lf_items_grad_to_classifier(const void* d_dE, int32_t dtype, int64_t v, int64_t d,
                                       double* d_dC, void* stream);
/* Widen a gradient buffer of `dtype`'s gradient type to double (dX ->
 * GradPair::d_embeddings). */
LF_API int lf_widen_grad(const void* d_src, int32_t dtype, int64_t count, double* d_dst,
                         void* stream);

/* -------------------------------------------------------- accounting ----- */
/* Replaces lseforge::estimate_flops (ccem.hpp:43-49, ccem.cpp:207-235):
 * backend 0 ce, 1 cem, 2 cce, 3 ccem, 4 bce (backend.hpp:10-16). */
LF_API int lf_estimate_flops(int64_t n, int64_t d, int64_t v, int64_t ns, int32_t backend,
                      uint64_t* forward, uint64_t* backward);

/* Device scratch the library itself allocates (stream-ordered pool):
 * current and high-water bytes since the last reset, for the CALLING THREAD
 * (each call's scratch is charged to the thread that made it, so concurrent
 * callers do not see each other's). */
LF_API int lf_workspace_stats(uint64_t* current_bytes, uint64_t* peak_bytes);
LF_API int lf_workspace_reset_peak(void);

/* Number of library kernel launches issued since the last reset (for the
 * bench's gpu_launches evidence). */
LF_API uint64_t lf_launch_count(void);
LF_API void lf_launch_count_reset(void);

/* ------------------------------------------------------------ tracing ---- */
/* Per-kernel CUDA-event timing.  When enabled, the library brackets each of
 * its main kernel launches with events recorded on the launching stream;
 * lf_profile_read synchronizes those events and returns, for one kernel kind,
 * the launch count and summed device milliseconds since the last reset. */
enum lf_kernel_kind {
  LF_K_CCE_FWD = 0,    /* tcgen05 forward (online LSE epilogue) */
  LF_K_CCE_BWD_DX = 1, /* tcgen05 backward, row-owned dX pass */
  LF_K_CCE_BWD_DE = 2, /* tcgen05 backward, item-owned dE pass */
  LF_K_CCE_SIMT = 3,   /* fp32 / fp64 CUDA-core CCE kernels */
  LF_K_CCEM_FWD = 4,   /* CCE- forward gather/dot/LSE */
  LF_K_CCEM_BWD = 5,   /* CCE- backward (rows pass + sort + segment reduce) */
  LF_K_AUX = 6,        /* combine / reduce / prep kernels */
  LF_K_EVAL = 7,       /* full-catalog ranking (rank + top-K) */
  LF_K_CCE_FWD_DX = 8, /* tcgen05 fused forward + dX accumulation (lf_cce_forward_backward) */
  LF_K_COUNT = 9
};
LF_API int lf_profile_enable(int on);
LF_API int lf_profile_read(int32_t kind, uint64_t* launches, double* total_ms);
LF_API void lf_profile_reset(void);

#ifdef __cplusplus
}
#endif

#endif /* LSEFORGE_B200_H */
