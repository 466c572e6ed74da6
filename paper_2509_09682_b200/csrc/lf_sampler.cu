// lf_sampler.cu — device restatement of the reference's uniform negative
// sampler (proj/src/sampler.cpp:44-75, SplitMix64 in rng.hpp:13-60), bit-exact:
// row i draws from SplitMix64(seed).derived(i); each slot takes the next draw
// that is inside the catalog (bounded()'s mask-and-reject) and differs from the
// row's positive; a slot that sees retry_cap consecutive positive draws is an
// error, as in the reference.  Produces the N x (1 + ns) index matrix CCE- takes
// (slot 0 = positive) directly in HBM, so the 210 MB int64 upload of cfg3 is not
// needed.
//
// SplitMix64 is a counter generator: draw k of a stream is mix(s + (k+1) g),
// so a warp evaluates 32 consecutive draws of one row at once and places the
// accepted ones with a ballot prefix count — same sequence as the serial loop.
#include <algorithm>
#include <cstdint>
#include <string>

#include "lf_internal.cuh"
#include "lf_kernels.cuh"

namespace lf {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // rng.hpp:51-55
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// Warp per row.  status[0]: first row that exhausted retry_cap (or n).
__global__ void __launch_bounds__(256) sample_uniform_rows(const int64_t* __restrict__ pos,
                                                           int64_t n, int64_t ns, uint64_t catalog,
                                                           uint64_t seed, int retry_cap,
                                                           int64_t* __restrict__ inds,
                                                           unsigned long long* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  const int64_t w = ns + 1;
  const int64_t p = pos[row];
  int64_t* out = inds + row * w;
  if (lane == 0) out[0] = p;
  // derived(i): SplitMix64(mix(seed + golden (i + 1))); draw k = mix(s + (k + 1) golden)
  const uint64_t s = mix64(seed + kGolden * static_cast<uint64_t>(row + 1));
  uint64_t mask = catalog - 1;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  mask |= mask >> 32;
  int64_t filled = 0;
  int run = 0;  // consecutive positive draws in the current slot (warp-uniform)
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t k0 = 0; filled < ns; k0 += 32) {
    const uint64_t v = mix64(s + (k0 + lane + 1) * kGolden) & mask;
    const bool inside = v < catalog;
    const bool hit_pos = inside && static_cast<int64_t>(v) == p;
    const bool acc = inside && !hit_pos;
    const unsigned am = __ballot_sync(0xffffffffu, acc);
    const unsigned pm = __ballot_sync(0xffffffffu, hit_pos);
    // retry cap (sampler.cpp:62-70): a slot fails after retry_cap consecutive
    // positive draws (out-of-catalog draws are bounded()'s own rejections and
    // do not count).  Walk the batch's relevant draws in order — warp-uniform,
    // and only when a positive was drawn (rare for a large catalog).
    if (pm) {
      unsigned m = am | pm;
      int64_t f = filled;
      int r = run;
      bool failed = false;
      while (m && f < ns) {
        const int b = __ffs(m) - 1;
        m &= m - 1u;
        if ((pm >> b) & 1u) {
          if (++r >= retry_cap) {
            failed = true;
            break;
          }
        } else {
          ++f;
          r = 0;
        }
      }
      if (failed) {
        if (lane == 0) atomicMin(status, static_cast<unsigned long long>(row));
        return;
      }
      run = r;
    } else if (am) {
      run = 0;
    }
    if (acc) {
      const int64_t slot = filled + __popc(am & lt) + 1;
      if (slot <= ns) out[slot] = static_cast<int64_t>(v);
    }
    filled += __popc(am);
  }
}

__global__ void first_bad_positive(const int64_t* __restrict__ pos, int64_t n, int64_t catalog,
                                   unsigned long long* __restrict__ first) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (pos[i] < 0 || pos[i] >= catalog) atomicMin(first, static_cast<unsigned long long>(i));
}

// ---- popularity sampler (sampler.cpp:77-127) ----
// Weights and their running sum for exponent != 1: a single thread keeps the
// reference's summation order (pow itself may differ from glibc's in the last
// ulp).  (exponent == 1 uses the blocked scan below.)
// flags[0] = first negative count, flags[1] = 1 if the total is not > 0.
// count^exponent for every item, in parallel (the expensive part of a
// non-unit exponent); pop_cumulative then sums them in the reference's order.
__global__ void pop_weights(const int64_t* __restrict__ counts, int64_t catalog, double exponent,
                            double* __restrict__ w, unsigned long long* __restrict__ flags) {
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < catalog;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = counts[v];
    if (c < 0) atomicMin(flags, static_cast<unsigned long long>(v));
    w[v] = pow(static_cast<double>(c), exponent);
  }
}

// Running sum over the weights already in cum (pop_weights), in place.
__global__ void pop_cumulative(const int64_t* __restrict__ counts, int64_t catalog, double exponent,
                               double* __restrict__ cum, unsigned long long* __restrict__ flags,
                               double* __restrict__ total) {
  __shared__ double seg[1024];
  const int T = blockDim.x;
  const int64_t len = ceil_div(catalog, T);
  const int64_t lo = threadIdx.x * len, hi = min(catalog, lo + len);
  double run = 0.0;
  for (int64_t v = lo; v < hi; ++v) {
    run += cum[v];
    cum[v] = run;
  }
  seg[threadIdx.x] = run;
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scan of the segment sums, in order
    double acc = 0.0;
    for (int t = 0; t < T; ++t) {
      const double x = seg[t];
      seg[t] = acc;
      acc += x;
    }
    *total = acc;
    if (!(acc > 0.0)) flags[1] = 1;
  }
  __syncthreads();
  const double off = seg[threadIdx.x];
  if (off != 0.0)
    for (int64_t v = lo; v < hi; ++v) cum[v] += off;
}

// exponent == 1: a three-kernel blocked scan over all SMs (exact: every
// partial sum of integer counts is an integer below 2^53).  Block = 256
// threads x 16 consecutive items.
constexpr int kScanPer = 16, kScanBlock = 256 * kScanPer;

__device__ __forceinline__ double block_exclusive_scan(double x, double* warp_tot, double* block_total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double inc = x;
  for (int off = 1; off < 32; off <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += y;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) {
      const double t = warp_tot[w];
      warp_tot[w] = acc;
      acc += t;
    }
    *block_total = acc;
  }
  __syncthreads();
  return warp_tot[warp] + inc - x;
}

__global__ void __launch_bounds__(256) pop_block_sums(const int64_t* __restrict__ counts, int64_t catalog,
                                                    double* __restrict__ block_sums,
                                                    unsigned long long* __restrict__ flags) {
  __shared__ double wt[8], bt;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kScanBlock + threadIdx.x * kScanPer;
  double x = 0.0;
  for (int q = 0; q < kScanPer; ++q) {
    const int64_t v = i0 + q;
    if (v < catalog) {
      const int64_t c = counts[v];
      if (c < 0) atomicMin(flags, static_cast<unsigned long long>(v));
      x += static_cast<double>(c);
    }
  }
  block_exclusive_scan(x, wt, &bt);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = bt;
}

__global__ void pop_scan_blocks(double* __restrict__ block_sums, int64_t nb, double* __restrict__ total,
                                unsigned long long* __restrict__ flags) {
  if (threadIdx.x != 0) return;
  double acc = 0.0;
  for (int64_t b = 0; b < nb; ++b) {
    const double t = block_sums[b];
    block_sums[b] = acc;
    acc += t;
  }
  *total = acc;
  if (!(acc > 0.0)) flags[1] = 1;
}

__global__ void __launch_bounds__(256) pop_block_scan(const int64_t* __restrict__ counts, int64_t catalog,
                                                    const double* __restrict__ block_off,
                                                    double* __restrict__ cum) {
  __shared__ double wt[8], bt;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kScanBlock + threadIdx.x * kScanPer;
  double w[kScanPer], x = 0.0;
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {
    const int64_t v = i0 + q;
    w[q] = v < catalog ? static_cast<double>(counts[v]) : 0.0;
    x += w[q];
  }
  double run = block_off[blockIdx.x] + block_exclusive_scan(x, wt, &bt);
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {
    run += w[q];
    if (i0 + q < catalog) cum[i0 + q] = run;
  }
}

__device__ __forceinline__ int64_t upper_bound(const double* __restrict__ cum, int64_t n, double u) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = lo + ((hi - lo) >> 1);
    if (!(u < cum[mid])) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Guide table (Chen's method): guide[j] = upper_bound(cum, (j - 1) total / G),
// so a draw u in bucket j = floor(u G / total) has its answer in
// [guide[j], guide[j + 2]); a few probes instead of ~20.  The result is
// verified against its neighbours and falls back to the full search, so it is
// always exactly upper_bound(cum, u) (the reference's std::upper_bound).
__global__ void build_guide(const double* __restrict__ cum, int64_t catalog, const double* __restrict__ total,
                            int64_t G, int64_t* __restrict__ guide) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= G) return;
  const double t = static_cast<double>(j - 1) * (*total / static_cast<double>(G));
  guide[j] = j == 0 ? 0 : upper_bound(cum, catalog, t);
}

__device__ __forceinline__ int64_t guided_upper_bound(const double* __restrict__ cum, int64_t catalog,
                                                      const int64_t* __restrict__ guide, int64_t G,
                                                      double scale, double u) {
  int64_t j = static_cast<int64_t>(u * scale);
  j = j < 0 ? 0 : (j >= G ? G - 1 : j);
  const int64_t lo = guide[j], hi = j + 2 < G ? guide[j + 2] : catalog;
  int64_t r = lo + upper_bound(cum + lo, hi - lo, u);
  const bool ok = (r == catalog || u < cum[r]) && (r == 0 || !(u < cum[r - 1]));
  return ok ? r : upper_bound(cum, catalog, u);
}

// Warp per row, 32 consecutive draws at once (one uniform() per attempt);
// every rejected draw (index past the table, or the positive) is one failed
// attempt of the current slot, retry_cap in a row is an error.
__global__ void __launch_bounds__(256) sample_popularity_rows(
    const int64_t* __restrict__ pos, int64_t n, int64_t ns, const double* __restrict__ cum,
    int64_t catalog, const double* __restrict__ total, const int64_t* __restrict__ guide, int64_t G,
    uint64_t seed, int retry_cap, int64_t* __restrict__ inds, unsigned long long* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  const int64_t w = ns + 1;
  const int64_t p = pos[row];
  const double running = *total;
  const double scale = static_cast<double>(G) / running;
  int64_t* out = inds + row * w;
  if (lane == 0) out[0] = p;
  const uint64_t s = mix64(seed + kGolden * static_cast<uint64_t>(row + 1));
  int64_t filled = 0;
  int run = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t k0 = 0; filled < ns; k0 += 32) {
    const uint64_t z = mix64(s + (k0 + lane + 1) * kGolden);
    const double u = static_cast<double>(z >> 11) * 0x1.0p-53 * running;  // rng.hpp:41
    const int64_t v = guided_upper_bound(cum, catalog, guide, G, scale, u);
    const bool acc = v < catalog && v != p;
    const unsigned am = __ballot_sync(0xffffffffu, acc);
    const unsigned fm = ~am;
    if (fm) {  // walk the batch in order (rare)
      int64_t f = filled;
      int r = run;
      bool failed = false;
      for (int b = 0; b < 32 && f < ns; ++b) {
        if ((am >> b) & 1u) {
          ++f;
          r = 0;
        } else if (++r >= retry_cap) {
          failed = true;
          break;
        }
      }
      if (failed) {
        if (lane == 0) atomicMin(status, static_cast<unsigned long long>(row));
        return;
      }
      run = r;
    } else {
      run = 0;
    }
    if (acc) {
      const int64_t slot = filled + __popc(am & lt) + 1;
      if (slot <= ns) out[slot] = v;
    }
    filled += __popc(am);
  }
}

}  // namespace

int sample_popularity(const int64_t* positives, int64_t n, int64_t ns, const int64_t* counts,
                      int64_t catalog, double exponent, uint64_t seed, int retry_cap, int64_t* inds,
                      cudaStream_t st) {
  if (catalog <= 0) return fail(LF_EINVAL, "sample_popularity: empty popularity table");
  if (n < 0 || ns < 0) return fail(LF_EINVAL, "sample_popularity: negative extent");
  Scratch flag, cum, tot;
  int rc = flag.alloc(4 * sizeof(unsigned long long), st);
  if (!rc) rc = cum.alloc(sizeof(double) * catalog, st);
  if (!rc) rc = tot.alloc(sizeof(double), st);
  if (rc) return rc;
  LF_CUDA(cudaMemsetAsync(flag.ptr, 0xFF, sizeof(unsigned long long), st));
  LF_CUDA(cudaMemsetAsync(flag.as<unsigned long long>() + 1, 0, sizeof(unsigned long long), st));
  LF_CUDA(cudaMemsetAsync(flag.as<unsigned long long>() + 2, 0xFF, 2 * sizeof(unsigned long long), st));
  unsigned long long* f = flag.as<unsigned long long>();
  Scratch bsums;
  if (exponent == 1.0) {
    const int64_t nb = ceil_div(catalog, kScanBlock);
    rc = bsums.alloc(sizeof(double) * nb, st);
    if (rc) return rc;
    pop_block_sums<<<static_cast<unsigned>(nb), 256, 0, st>>>(counts, catalog, bsums.as<double>(), f);
    pop_scan_blocks<<<1, 32, 0, st>>>(bsums.as<double>(), nb, tot.as<double>(), f);
    pop_block_scan<<<static_cast<unsigned>(nb), 256, 0, st>>>(counts, catalog, bsums.as<double>(), cum.as<double>());
  } else {  // weights in parallel, then the reference's summation order (sampler.cpp:93-99)
    pop_weights<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(catalog, 256), 8LL * num_sms())), 256, 0,
                  st>>>(counts, catalog, exponent, cum.as<double>(), f);
    pop_cumulative<<<1, 1, 0, st>>>(counts, catalog, exponent, cum.as<double>(), f, tot.as<double>());
  }
  LF_LAUNCHED();
  first_bad_positive<<<static_cast<unsigned>(std::min<int64_t>(std::max<int64_t>(ceil_div(n, 256), 1), 1024)),
                       256, 0, st>>>(positives, n, catalog, f + 2);
  LF_LAUNCHED();
  unsigned long long h[3];
  LF_CUDA(cudaMemcpyAsync(h, f, sizeof(h), cudaMemcpyDeviceToHost, st));
  LF_CUDA(cudaStreamSynchronize(st));
  if (h[0] != ~0ull) {  // PopularityTable::FromCounts (sampler.cpp:30-42)
    int64_t c = 0;
    LF_CUDA(cudaMemcpy(&c, counts + h[0], sizeof(c), cudaMemcpyDeviceToHost));
    return fail(LF_EINVAL, "PopularityTable: item " + std::to_string(h[0]) + " has negative count " +
                               std::to_string(c));
  }
  if (h[2] != ~0ull) {  // sampler.cpp:12-20
    int64_t bad = 0;
    LF_CUDA(cudaMemcpy(&bad, positives + h[2], sizeof(bad), cudaMemcpyDeviceToHost));
    return fail(LF_EINVAL, "sampler: row " + std::to_string(h[2]) + " positive " + std::to_string(bad) +
                               " outside catalog of " + std::to_string(catalog));
  }
  if (ns > catalog - 1)
    return fail(LF_EINVAL, "sample_popularity: ns = " + std::to_string(ns) +
                               " exceeds catalog minus positive (" + std::to_string(catalog - 1) + ")");
  if (h[1]) return fail(LF_EINVAL, "sample_popularity: all item weights are zero");
  if (n == 0) return LF_OK;
  if (retry_cap < 1 && ns > 0)  // no attempt is made: row 0's first slot fails (sampler.cpp:62-71)
    return fail(LF_ERUNTIME, "sampler: row 0 exhausted " + std::to_string(retry_cap) +
                                 " rejection retries; the distribution leaves no valid negative");
  const int64_t G = catalog;
  Scratch guide;
  rc = guide.alloc(sizeof(int64_t) * G, st);
  if (rc) return rc;
  build_guide<<<static_cast<unsigned>(ceil_div(G, 256)), 256, 0, st>>>(cum.as<double>(), catalog, tot.as<double>(),
                                                                       G, guide.as<int64_t>());
  LF_LAUNCHED();
  sample_popularity_rows<<<static_cast<unsigned>(ceil_div(n, 8)), 256, 0, st>>>(
      positives, n, ns, cum.as<double>(), catalog, tot.as<double>(), guide.as<int64_t>(), G, seed,
      retry_cap, inds, f + 3);
  LF_LAUNCHED();
  unsigned long long bad = 0;
  LF_CUDA(cudaMemcpyAsync(&bad, f + 3, sizeof(bad), cudaMemcpyDeviceToHost, st));
  LF_CUDA(cudaStreamSynchronize(st));
  if (bad != ~0ull)  // sampler.cpp:22-27
    return fail(LF_ERUNTIME, "sampler: row " + std::to_string(bad) + " exhausted " + std::to_string(retry_cap) +
                                 " rejection retries; the distribution leaves no valid negative");
  return LF_OK;
}

int sample_uniform(const int64_t* positives, int64_t n, int64_t ns, int64_t catalog,
                   uint64_t seed, int retry_cap, int64_t* inds, cudaStream_t st) {
  // the reference's order (sampler.cpp:44-56): catalog, positives, ns
  if (catalog <= 0) return fail(LF_EINVAL, "sample_uniform: empty catalog");
  if (n < 0 || ns < 0) return fail(LF_EINVAL, "sample_uniform: negative extent");
  auto ns_check = [&]() {
    return ns > catalog - 1
               ? fail(LF_EINVAL, "sample_uniform: ns = " + std::to_string(ns) +
                                     " exceeds catalog minus positive (" + std::to_string(catalog - 1) + ")")
               : LF_OK;
  };
  if (n == 0) return ns_check();
  Scratch flag;
  int rc = flag.alloc(2 * sizeof(unsigned long long), st);
  if (rc) return rc;
  LF_CUDA(cudaMemsetAsync(flag.ptr, 0xFF, 2 * sizeof(unsigned long long), st));
  unsigned long long* f = flag.as<unsigned long long>();
  first_bad_positive<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), 1024)), 256, 0, st>>>(
      positives, n, catalog, f);
  LF_LAUNCHED();
  unsigned long long h = 0;
  LF_CUDA(cudaMemcpyAsync(&h, f, sizeof(h), cudaMemcpyDeviceToHost, st));
  LF_CUDA(cudaStreamSynchronize(st));
  if (h != ~0ull) {  // sampler.cpp:12-20, the reference's message
    int64_t bad = 0;
    LF_CUDA(cudaMemcpy(&bad, positives + h, sizeof(bad), cudaMemcpyDeviceToHost));
    return fail(LF_EINVAL, "sampler: row " + std::to_string(h) + " positive " + std::to_string(bad) +
                               " outside catalog of " + std::to_string(catalog));
  }
  rc = ns_check();
  if (rc) return rc;
  if (retry_cap < 1 && ns > 0)  // no attempt is made: row 0's first slot fails (sampler.cpp:62-71)
    return fail(LF_ERUNTIME, "sampler: row 0 exhausted " + std::to_string(retry_cap) +
                                 " rejection retries; the distribution leaves no valid negative");
  sample_uniform_rows<<<static_cast<unsigned>(ceil_div(n, 8)), 256, 0, st>>>(
      positives, n, ns, static_cast<uint64_t>(catalog), seed, retry_cap, inds, f + 1);
  LF_LAUNCHED();
  LF_CUDA(cudaMemcpyAsync(&h, f + 1, sizeof(h), cudaMemcpyDeviceToHost, st));
  LF_CUDA(cudaStreamSynchronize(st));
  if (h != ~0ull)  // sampler.cpp:22-27
    return fail(LF_ERUNTIME, "sampler: row " + std::to_string(h) + " exhausted " +
                                 std::to_string(retry_cap) +
                                 " rejection retries; the distribution leaves no valid negative");
  return LF_OK;
}

}  // namespace lf
