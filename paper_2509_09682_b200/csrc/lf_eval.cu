// lf_eval.cu — full-catalog evaluation on the device: the reference's
// evaluate() (proj/src/metrics.cpp:13-103) minus the encoder, which is the
// caller's (X holds the encoded rows h, metrics.cpp:46).
//
//   rank_i  = 1 + #{j : s_ij > s_it, or s_ij == s_it and j < t}   (metrics.cpp:56-60)
//   top-k_i = first k of the items by (score desc, index asc)     (metrics.cpp:63-72)
//   NDCG / coverage / surprisal aggregation                       (metrics.cpp:62, 74-103)
//
// The scores are never materialised: bf16 runs the tcgen05 kernel in EVAL
// mode (lf_tc.cu), fp32 / fp64 the SIMT kernel (lf_simt.cu); both emit, per
// (V chunk, row), the count of items ranked ahead of the target and the
// chunk's top-k, which eval_combine folds.  Catalog shards compose the same
// way: counts add, top-k lists merge (lf_eval_merge).
#include <climits>
#include <cmath>
#include <cstring>
#include <string>

#include "lf_internal.cuh"
#include "lf_kernels.cuh"

namespace lf {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// tl[i] = targets[i] - v_offset clamped to [-1, v] (-1: the target precedes
// the shard, v: it follows it); Et row i = the target's item row (from
// target_rows when given, else gathered from the shard), zero past n.
// bad[0] = first row whose target is not in the shard (gather mode only).
__global__ void eval_prep(const int64_t* __restrict__ targets, const uint32_t* __restrict__ E,
                          const uint32_t* __restrict__ target_rows, int64_t n, int64_t n_pad,
                          int64_t v, int64_t v_offset, int words, int32_t* __restrict__ tl,
                          uint32_t* __restrict__ Et, unsigned long long* __restrict__ bad) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n_pad) return;
  const uint32_t* src = nullptr;
  if (i < n) {
    const int64_t local = targets[i] - v_offset;
    if (lane == 0) tl[i] = static_cast<int32_t>(local < 0 ? -1 : (local > v ? v : local));
    if (target_rows) {
      src = target_rows + i * words;
    } else if (local >= 0 && local < v) {
      src = E + local * words;
    } else if (lane == 0) {
      atomicMin(bad, static_cast<unsigned long long>(i));
    }
  } else if (lane == 0) {
    tl[i] = -1;
  }
  for (int w = lane; w < words; w += 32) Et[i * words + w] = src ? src[w] : 0u;
}

template <class TI>
__device__ __forceinline__ bool idx_empty(TI x) {
  return sizeof(TI) == 4 ? x == static_cast<TI>(INT_MAX) : x < 0;
}

// Warp per row: fold P count / top-KS blocks into ahead (or rank) and the
// row's top-k (k <= KS, k <= 32), lane e holding entry e.
template <class TC, class TV, class TI>
__global__ void eval_combine(const TC* __restrict__ cnt, const TV* __restrict__ val,
                             const TI* __restrict__ idx, int P, int KS, int64_t n, int k,
                             int64_t idx_offset, int64_t add, int64_t* __restrict__ ahead,
                             int64_t* __restrict__ top_idx, double* __restrict__ top_score) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  unsigned long long c = 0;
  for (int p = lane; p < P; p += 32) c += static_cast<unsigned long long>(cnt[p * n + row]);
  for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(kFull, c, off);
  double kv = -INFINITY;
  long long ki = LLONG_MAX;
  for (int p = 0; p < P; ++p) {
    const int64_t rp = (static_cast<int64_t>(p) * n + row) * KS;
    double cv_l = -INFINITY;
    long long ci_l = LLONG_MAX;
    int has_l = 0;
    if (lane < k) {
      const TI li = idx[rp + lane];
      if (!idx_empty(li)) {
        cv_l = static_cast<double>(val[rp + lane]);
        ci_l = static_cast<long long>(li) + idx_offset;
        has_l = 1;
      }
    }
    for (int e = 0; e < k; ++e) {  // the block's list is descending: stop at the first miss
      if (!__shfl_sync(kFull, has_l, e)) break;
      const double cv = __shfl_sync(kFull, cv_l, e);
      const long long ci = __shfl_sync(kFull, ci_l, e);
      const bool ahead_l = lane < k && (kv > cv || (kv == cv && ki < ci));
      const int pos = __popc(__ballot_sync(kFull, ahead_l));
      if (pos >= k) break;
      const double upv = __shfl_up_sync(kFull, kv, 1);
      const long long upi = __shfl_up_sync(kFull, ki, 1);
      if (lane == pos) {
        kv = cv;
        ki = ci;
      } else if (lane > pos && lane < k) {
        kv = upv;
        ki = upi;
      }
    }
  }
  if (lane == 0) ahead[row] = static_cast<int64_t>(c) + add;
  if (lane < k) {
    top_idx[row * k + lane] = ki == LLONG_MAX ? -1 : ki;
    top_score[row * k + lane] = kv;
  }
}

// ---- aggregation (metrics.cpp:26-33, 62, 74-103) ----
// One block: total = sum of the popularity counts (exact: integers in double),
// first negative entry.
__global__ void eval_pop_total(const int64_t* __restrict__ pop, int64_t v, double* __restrict__ total,
                               unsigned long long* __restrict__ neg) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < v; j += blockDim.x) {
    const int64_t c = pop[j];
    if (c < 0) atomicMin(neg, static_cast<unsigned long long>(j));
    s += static_cast<double>(c);
  }
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += red[w];
    *total = t;
  }
}

// Per row: ndcg_i, surprisal_i, and the union of the top-k lists.
__global__ void eval_rows(const int64_t* __restrict__ rank, const int64_t* __restrict__ top, int64_t n,
                          int k, const int64_t* __restrict__ pop, const double* __restrict__ total,
                          double* __restrict__ ndcg, double* __restrict__ surp,
                          uint32_t* __restrict__ seen, unsigned long long* __restrict__ distinct) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double tot = *total;
  const double log2_total = log2(tot);
  const int64_t r = rank[i];
  ndcg[i] = r <= k ? 1.0 / log2(static_cast<double>(r) + 1.0) : 0.0;
  double acc = 0.0;
  for (int e = 0; e < k; ++e) {
    const int64_t item = top[i * k + e];
    if (item < 0) continue;
    const int64_t c = pop[item] > 1 ? pop[item] : 1;
    acc += -log2(static_cast<double>(c) / tot) / log2_total;
    if (atomicOr(&seen[item >> 5], 1u << (item & 31)) & (1u << (item & 31))) continue;
    atomicAdd(distinct, 1ull);
  }
  surp[i] = acc / static_cast<double>(k);
}

// Fixed-order sums (deterministic): 1024 contiguous segments, then a tree.
__global__ void eval_means(const double* __restrict__ ndcg, const double* __restrict__ surp, int64_t n,
                           const unsigned long long* __restrict__ distinct, int64_t v,
                           double* __restrict__ out) {
  __shared__ double a[1024], b[1024];
  const int64_t seg = ceil_div(n, 1024);
  const int64_t lo = threadIdx.x * seg, hi = min(n, lo + seg);
  double x = 0.0, y = 0.0;
  for (int64_t i = lo; i < hi; ++i) {
    x += ndcg[i];
    y += surp[i];
  }
  a[threadIdx.x] = x;
  b[threadIdx.x] = y;
  __syncthreads();
  for (int s = 512; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      a[threadIdx.x] += a[threadIdx.x + s];
      b[threadIdx.x] += b[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = a[0] / static_cast<double>(n);
    out[1] = static_cast<double>(*distinct) / static_cast<double>(v);
    out[2] = b[0] / static_cast<double>(n);
  }
}

__global__ void add_one(int64_t* __restrict__ x, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] += 1;
}

size_t dtype_bytes(int dtype) { return dtype == LF_F64 ? 8 : (dtype == LF_F32 ? 4 : 2); }

}  // namespace

int eval_rank_topk(int dtype, const void* X, const void* E, const int64_t* targets,
                   const void* target_rows, int64_t n, int D, int64_t v, int64_t v_offset, int k,
                   int64_t* ahead, int64_t* top_idx, double* top_score, cudaStream_t st) {
  if (n < 0 || v < 0 || D <= 0) return fail(LF_EINVAL, "eval: negative extent");
  if (k < 1) return fail(LF_EINVAL, "evaluate: k must be >= 1");
  const bool tc = dtype == LF_BF16;
  if (k > (tc ? 16 : 32))
    return fail(LF_EUNSUPPORTED, "eval: k = " + std::to_string(k) + " exceeds the per-row top-k of this path (" +
                                     (tc ? "16 for bf16" : "32 for f32/f64") + ")");
  if (tc && (D % 64 != 0 || D > 256)) return fail(LF_EUNSUPPORTED, "eval bf16: d must be 64/128/192/256");
  if (v >= INT_MAX) return fail(LF_EUNSUPPORTED, "eval: shard too large for 32-bit item indices");
  if (n == 0) return LF_OK;
  if (v == 0) {
    // empty shard: nothing ranks ahead, no items
    LF_CUDA(cudaMemsetAsync(ahead, 0, sizeof(int64_t) * n, st));
    LF_CUDA(cudaMemsetAsync(top_idx, 0xff, sizeof(int64_t) * n * k, st));
    return LF_OK;
  }
  const int64_t n_pad = tc ? ceil_div(n, 128) * 128 : n;
  const int words = static_cast<int>(D * dtype_bytes(dtype) / 4);
  Scratch tl, Et, bad;
  int rc = tl.alloc(sizeof(int32_t) * n_pad, st);
  if (!rc) rc = Et.alloc(static_cast<size_t>(words) * 4 * n_pad, st);
  if (!rc) rc = bad.alloc(sizeof(unsigned long long), st);
  if (rc) return rc;
  LF_CUDA(cudaMemsetAsync(bad.ptr, 0xff, sizeof(unsigned long long), st));
  eval_prep<<<static_cast<unsigned>(ceil_div(n_pad, 8)), 256, 0, st>>>(
      targets, static_cast<const uint32_t*>(E), static_cast<const uint32_t*>(target_rows), n, n_pad, v,
      v_offset, words, tl.as<int32_t>(), Et.as<uint32_t>(), bad.as<unsigned long long>());
  LF_LAUNCHED();
  if (!target_rows) {
    unsigned long long h = 0;
    LF_CUDA(cudaMemcpyAsync(&h, bad.ptr, sizeof(h), cudaMemcpyDeviceToHost, st));
    LF_CUDA(cudaStreamSynchronize(st));
    if (h != ~0ull)
      return fail(LF_EINVAL, "eval: row " + std::to_string(h) +
                                 " has its target outside this catalog shard (pass target_rows)");
  }
  Scratch cnt, val, idx;
  int P = 0;
  const unsigned blocks = static_cast<unsigned>(ceil_div(n, 8));
  if (tc) {
    int K = 16;
    rc = tc_eval_partials(X, E, Et.ptr, tl.as<int32_t>(), n, D, v, k, cnt, val, idx, &P, &K, st);
    if (rc) return rc;
    eval_combine<uint32_t, float, int32_t><<<blocks, 256, 0, st>>>(
        cnt.as<uint32_t>(), val.as<float>(), idx.as<int32_t>(), P, K, n, k, v_offset, 0, ahead,
        top_idx, top_score);
  } else if (dtype == LF_F32) {
    rc = simt_eval_partials<float>(static_cast<const float*>(X), static_cast<const float*>(E),
                                   Et.as<float>(), tl.as<int32_t>(), n, D, v, k, cnt, val, idx, &P, st);
    if (rc) return rc;
    eval_combine<uint32_t, float, int32_t><<<blocks, 256, 0, st>>>(
        cnt.as<uint32_t>(), val.as<float>(), idx.as<int32_t>(), P, k, n, k, v_offset, 0, ahead,
        top_idx, top_score);
  } else {
    rc = simt_eval_partials<double>(static_cast<const double*>(X), static_cast<const double*>(E),
                                    Et.as<double>(), tl.as<int32_t>(), n, D, v, k, cnt, val, idx, &P,
                                    st);
    if (rc) return rc;
    eval_combine<uint32_t, double, int32_t><<<blocks, 256, 0, st>>>(
        cnt.as<uint32_t>(), val.as<double>(), idx.as<int32_t>(), P, k, n, k, v_offset, 0, ahead,
        top_idx, top_score);
  }
  LF_LAUNCHED();
  return LF_OK;
}

int launch_add_one(int64_t* x, int64_t n, cudaStream_t st) {
  if (n == 0) return LF_OK;
  add_one<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, st>>>(x, n);
  LF_LAUNCHED();
  return LF_OK;
}

int eval_merge(const int64_t* ahead, const int64_t* top_idx, const double* top_score, int P,
               int64_t n, int k, int64_t* rank, int64_t* top_idx_out, double* top_score_out,
               cudaStream_t st) {
  if (P < 1 || n < 0 || k < 1 || k > 32) return fail(LF_EINVAL, "eval_merge: bad P / n / k (k <= 32)");
  if (n == 0) return LF_OK;
  eval_combine<int64_t, double, int64_t><<<static_cast<unsigned>(ceil_div(n, 8)), 256, 0, st>>>(
      ahead, top_score, top_idx, P, k, n, k, 0, 1, rank, top_idx_out, top_score_out);
  LF_LAUNCHED();
  return LF_OK;
}

int eval_summary(const int64_t* rank, const int64_t* top_idx, int64_t n, int k, const int64_t* pop,
                 int64_t v, double* out3_host, cudaStream_t st) {
  if (n <= 0) return fail(LF_EINVAL, "evaluate: no eval pairs");
  if (k < 1) return fail(LF_EINVAL, "evaluate: k must be >= 1");
  if (v <= 0) return fail(LF_EINVAL, "evaluate: empty catalog");
  Scratch buf, seen, rows;
  int rc = buf.alloc(8 * 8, st);  // [0] total, [1] neg, [2] distinct, [4..6] out
  if (!rc) rc = seen.alloc(sizeof(uint32_t) * ceil_div(v, 32), st);
  if (!rc) rc = rows.alloc(sizeof(double) * 2 * n, st);
  if (rc) return rc;
  double* total = buf.as<double>();
  unsigned long long* neg = buf.as<unsigned long long>() + 1;
  unsigned long long* distinct = buf.as<unsigned long long>() + 2;
  double* out = buf.as<double>() + 4;
  LF_CUDA(cudaMemsetAsync(neg, 0xff, 8, st));
  LF_CUDA(cudaMemsetAsync(distinct, 0, 8, st));
  LF_CUDA(cudaMemsetAsync(seen.ptr, 0, sizeof(uint32_t) * ceil_div(v, 32), st));
  eval_pop_total<<<1, 1024, 0, st>>>(pop, v, total, neg);
  LF_LAUNCHED();
  double h[2];
  LF_CUDA(cudaMemcpyAsync(h, buf.ptr, 16, cudaMemcpyDeviceToHost, st));
  LF_CUDA(cudaStreamSynchronize(st));
  unsigned long long neg_h;
  memcpy(&neg_h, &h[1], 8);
  if (neg_h != ~0ull) return fail(LF_EINVAL, "evaluate: negative popularity count");
  if (h[0] < 2.0) return fail(LF_EINVAL, "evaluate: popularity table needs at least 2 training events");
  eval_rows<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, st>>>(
      rank, top_idx, n, k, pop, total, rows.as<double>(), rows.as<double>() + n, seen.as<uint32_t>(),
      distinct);
  LF_LAUNCHED();
  eval_means<<<1, 1024, 0, st>>>(rows.as<double>(), rows.as<double>() + n, n, distinct, v, out);
  LF_LAUNCHED();
  LF_CUDA(cudaMemcpyAsync(out3_host, out, 24, cudaMemcpyDeviceToHost, st));
  LF_CUDA(cudaStreamSynchronize(st));
  return LF_OK;
}

}  // namespace lf
