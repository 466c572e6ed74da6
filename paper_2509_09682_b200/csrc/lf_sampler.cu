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

}  // namespace

int sample_uniform(const int64_t* positives, int64_t n, int64_t ns, int64_t catalog,
                   uint64_t seed, int retry_cap, int64_t* inds, cudaStream_t st) {
  if (catalog <= 0) return fail(LF_EINVAL, "sample_uniform: empty catalog");
  if (n < 0 || ns < 0) return fail(LF_EINVAL, "sample_uniform: negative extent");
  if (ns > catalog - 1)
    return fail(LF_EINVAL, "sample_uniform: ns = " + std::to_string(ns) +
                               " exceeds catalog minus positive (" + std::to_string(catalog - 1) +
                               ")");
  if (n == 0) return LF_OK;
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
