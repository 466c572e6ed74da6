// lf_capi.cu — extern "C" entry points of liblseforge_b200.so (declared in
// include/lseforge_b200.h) plus the library's error, scratch and launch
// bookkeeping.  Argument checks reproduce the reference's validation
// (losses.cpp:48-69, cce.cpp:17-27, ccem.cpp:16-31) with the same messages;
// the index scans themselves are separate calls (lf_validate_*) because they
// need a device->host sync.
#include <nvtx3/nvToolsExt.h>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "lf_internal.cuh"
#include "lf_kernels.cuh"

#ifndef LF_SIMT_FUSED
#define LF_SIMT_FUSED 1  // fp32 lf_cce_forward_backward with the filter off: fused SIMT forward + dX
#endif

namespace lf {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
// Scratch accounting is per calling thread: every Scratch lives on the stack
// of the call that allocated it, so concurrent callers (e.g. the reference's
// sweep running points in parallel, sweep.cpp:101) never charge each other's
// scratch to their own MemAccountant.
thread_local uint64_t g_ws_current = 0;
thread_local uint64_t g_ws_peak = 0;
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? LF_ENOMEM : LF_ECUDA;
}
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
std::atomic<int> g_prof_on{0};
std::mutex g_prof_mu;
struct ProfRec {
  int kind;
  cudaEvent_t a, b;
};
std::vector<ProfRec> g_prof_pending;
uint64_t g_prof_launches[LF_K_COUNT] = {};
double g_prof_ms[LF_K_COUNT] = {};
}  // namespace

// NVTX ranges (header-only NVTX3: a no-op unless a tool such as nsys or
// ncu --nvtx is attached) name each library phase on the host timeline.
static const char* const kKindNames[LF_K_COUNT] = {
    "lf.cce_fwd", "lf.cce_bwd_dx", "lf.cce_bwd_de", "lf.cce_simt", "lf.ccem_fwd",
    "lf.ccem_bwd", "lf.aux", "lf.eval", "lf.cce_fwd_dx"};

ProfScope::ProfScope(int k, cudaStream_t s) : kind(k), st(s) {
  nvtxRangePushA(k >= 0 && k < LF_K_COUNT ? kKindNames[k] : "lf.kernel");
  if (g_prof_on.load() && cudaEventCreate(&start) == cudaSuccess) cudaEventRecord(start, st);
}
ProfScope::~ProfScope() {
  nvtxRangePop();
  if (!start) return;
  cudaEvent_t end;
  if (cudaEventCreate(&end) != cudaSuccess) return;
  cudaEventRecord(end, st);
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_pending.push_back({kind, start, end});
}

static void prof_drain() {
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& r : g_prof_pending) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess && r.kind >= 0 && r.kind < LF_K_COUNT) {
      g_prof_ms[r.kind] += ms;
      g_prof_launches[r.kind] += 1;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof_pending.clear();
}

// The library's scratch comes from the device's default stream-ordered pool.
// Its default release threshold (0) hands freed memory back to the driver at
// every synchronization, so the next call would pay a full cudaMalloc again;
// keep the pool's high-water mark resident instead (once per device).
static void keep_pool_resident() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> g(mu);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev] = true;
}

int Scratch::alloc(size_t nbytes, cudaStream_t s) {
  if (ptr) return fail(LF_EINVAL, "internal: scratch reused");
  if (nbytes == 0) nbytes = 16;
  keep_pool_resident();
  cudaError_t e = cudaMallocAsync(&ptr, nbytes, s);
  if (e != cudaSuccess) {
    ptr = nullptr;
    return cuda_fail(e, "cudaMallocAsync(scratch)");
  }
  bytes = nbytes;
  stream = s;
  g_ws_current += nbytes;
  if (g_ws_current > g_ws_peak) g_ws_peak = g_ws_current;
  return LF_OK;
}
Scratch::~Scratch() {
  if (ptr) {
    cudaFreeAsync(ptr, stream);
    g_ws_current -= bytes;
  }
}

int num_sms() {
  static int cached = [] {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
  }();
  return cached;
}

namespace {

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int check_cfg(const lf_cce_config* cfg) {
  if (!cfg) return fail(LF_EINVAL, "CceConfig: null config");
  if (!(cfg->filter_eps >= 0.0))  // cce.cpp:23-26 (also rejects NaN)
    return fail(LF_EINVAL, "CceConfig: filter_eps must be >= 0, got " + std::to_string(cfg->filter_eps));
  if (cfg->dtype != LF_F32 && cfg->dtype != LF_F64 && cfg->dtype != LF_BF16)
    return fail(LF_EINVAL, "lf_cce_config: unknown dtype " + std::to_string(cfg->dtype));
  return LF_OK;
}

// losses.cpp:48-57 shape checks (index range: lf_validate_targets).
int check_shapes(int64_t n, int64_t d, int64_t v) {
  if (n <= 0) return fail(LF_EINVAL, "loss: embedding matrix has zero rows; the mean loss is undefined");
  if (d <= 0) return fail(LF_EINVAL, "loss: embedding width must be >= 1");
  if (v <= 0) return fail(LF_EINVAL, "loss: catalog must hold at least one item");
  return LF_OK;
}

int check_bf16_d(int64_t d) {
  if (d % 64 != 0 || d > 256)
    return fail(LF_EUNSUPPORTED,
                "bf16 tensor-core path needs d in {64, 128, 192, 256} (got " + std::to_string(d) +
                    "); use dtype f32 or f64");
  return LF_OK;
}

struct Counters {
  Scratch buf;
  int init(cudaStream_t st) {
    int rc = buf.alloc(4 * sizeof(unsigned long long), st);
    if (rc) return rc;
    LF_CUDA(cudaMemsetAsync(buf.ptr, 0, 4 * sizeof(unsigned long long), st));
    return LF_OK;
  }
  unsigned long long* ptr() { return buf.as<unsigned long long>(); }
};

int read_stats(Counters& c, lf_cce_stats* stats, int64_t n, int64_t v_total, cudaStream_t st) {
  unsigned long long h[4] = {0, 0, 0, 0};
  LF_CUDA(cudaMemcpyAsync(h, c.ptr(), sizeof(h), cudaMemcpyDeviceToHost, st));
  LF_CUDA(cudaStreamSynchronize(st));
  stats->skipped_elems = h[0];
  stats->skipped_tiles = h[1];
  stats->total_tiles = h[2];
  const double off_target = static_cast<double>(n) * static_cast<double>(v_total - 1);
  stats->skipped_fraction = off_target == 0.0 ? 0.0 : static_cast<double>(h[0]) / off_target;
  return LF_OK;
}

int backward_impl(const void* X, const void* E, const int64_t* targets, const double* lse,
                  double upstream, int64_t n, int64_t d, int64_t v_shard, int64_t v_offset,
                  int64_t v_total, const lf_cce_config* cfg, void* dX, void* dE,
                  lf_cce_stats* stats, cudaStream_t st, const PeerPush* push = nullptr) {
  int rc = check_cfg(cfg);
  if (!rc) rc = check_shapes(n, d, v_shard);
  if (rc) return rc;
  if (!lse) return fail(LF_EINVAL, "cce_backward: LSE vector is null");
  const double scale = upstream / static_cast<double>(n);  // cce.cpp:174
  Counters c;
  rc = c.init(st);
  if (rc) return rc;
  switch (cfg->dtype) {
    case LF_BF16:
      rc = check_bf16_d(d);
      if (!rc)
        rc = tc_cce_backward(X, E, targets, lse, scale, cfg->filter_eps, n, static_cast<int>(d),
                             v_shard, v_offset, static_cast<float*>(dX), static_cast<float*>(dE),
                             stats ? c.ptr() : nullptr, st, push);
      break;
    case LF_F32:
      rc = simt_cce_backward<float>(static_cast<const float*>(X), static_cast<const float*>(E),
                                    targets, lse, scale, cfg->filter_eps, n, static_cast<int>(d),
                                    v_shard, v_offset, static_cast<float*>(dX),
                                    static_cast<float*>(dE), c.ptr(), st);
      if (!rc && push)
        rc = peer_reduce_push(static_cast<const float*>(dX), 1, n * d, push->peers, push->world,
                              push->rank, push->parity_off, st);
      break;
    default:
      rc = simt_cce_backward<double>(static_cast<const double*>(X),
                                     static_cast<const double*>(E), targets, lse, scale,
                                     cfg->filter_eps, n, static_cast<int>(d), v_shard, v_offset,
                                     static_cast<double*>(dX), static_cast<double*>(dE), c.ptr(),
                                     st);
  }
  if (rc) return rc;
  if (stats) return read_stats(c, stats, n, v_total, st);
  return LF_OK;
}

}  // namespace
}  // namespace lf

using namespace lf;

extern "C" {

int lf_abi_version(void) { return LF_ABI_VERSION; }

// The fused forward + dX kernel serves lf_cce_forward_backward when dX may
// ignore the filter: bf16, d = 64 / 128 / 256, and eps below 2^-12 (entries it
// would drop are < eps each; eps = 0 is exact) unless the caller asks for
// the filtered dX pass (LF_FLAG_FILTER_DX).
int lf_cce_fused_supported(const lf_cce_config* cfg, int64_t d) {
  return cfg && cfg->dtype == LF_BF16 && tc_fwdx_supported(static_cast<int>(d)) &&
         cfg->filter_eps < 0x1p-12 && !(cfg->flags & LF_FLAG_FILTER_DX);
}
const char* lf_last_error(void) { return g_last_error.c_str(); }

int lf_cce_forward(const void* d_X, const void* d_E, const int64_t* d_targets, int64_t n,
                   int64_t d, int64_t v, const lf_cce_config* cfg, double* d_lse, double* d_pos,
                   double* d_loss, void* stream) {
  int rc = check_cfg(cfg);
  if (!rc) rc = check_shapes(n, d, v);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  switch (cfg->dtype) {
    case LF_BF16: {
      rc = check_bf16_d(d);
      if (rc) return rc;
      Scratch ws;
      float* part = nullptr;
      int P = 0;
      rc = tc_cce_forward_partials(d_X, d_E, d_targets, n, static_cast<int>(d), v, 0, ws, &part,
                                   &P, st);
      if (rc) return rc;
      return launch_combine_f32log2(part, P, n, d_lse, d_pos, d_loss, st);
    }
    case LF_F32:
      return simt_cce_forward_full<float>(static_cast<const float*>(d_X),
                                          static_cast<const float*>(d_E), d_targets, n,
                                          static_cast<int>(d), v, d_lse, d_pos, d_loss, st);
    default:
      return simt_cce_forward_full<double>(static_cast<const double*>(d_X),
                                           static_cast<const double*>(d_E), d_targets, n,
                                           static_cast<int>(d), v, d_lse, d_pos, d_loss, st);
  }
}

int lf_cce_backward(const void* d_X, const void* d_E, const int64_t* d_targets,
                    const double* d_lse, double upstream, int64_t n, int64_t d, int64_t v,
                    const lf_cce_config* cfg, void* d_dX, void* d_dE, lf_cce_stats* stats,
                    void* stream) {
  return backward_impl(d_X, d_E, d_targets, d_lse, upstream, n, d, v, 0, v, cfg, d_dX, d_dE,
                       stats, as_stream(stream));
}

int lf_cce_forward_backward(const void* d_X, const void* d_E, const int64_t* d_targets, int64_t n,
                            int64_t d, int64_t v, double upstream, const lf_cce_config* cfg,
                            double* d_lse, double* d_pos, double* d_loss, void* d_dX, void* d_dE,
                            lf_cce_stats* stats, void* stream) {
  int rc = check_cfg(cfg);
  if (!rc) rc = check_shapes(n, d, v);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  if (cfg->dtype == LF_F32 && cfg->filter_eps == 0.0 && !(cfg->flags & LF_FLAG_FILTER_DX) &&
      LF_SIMT_FUSED) {
    // fp32, filter off: the fused SIMT forward + dX, then the dE pass (no
    // entry is filtered, so the skip counts are zero)
    if (!d_lse || !d_pos || !d_dX || !d_dE) return fail(LF_EINVAL, "cce_forward_backward: null output");
    rc = simt_cce_fused_f32(static_cast<const float*>(d_X), static_cast<const float*>(d_E), d_targets, n,
                            static_cast<int>(d), v, upstream / static_cast<double>(n), 0.0, d_lse, d_pos,
                            d_loss, static_cast<float*>(d_dX), static_cast<float*>(d_dE), st);
    if (rc) return rc;
    if (stats) {
      Counters c;
      rc = c.init(st);
      if (!rc) rc = read_stats(c, stats, n, v, st);
    }
    return rc;
  }
  if (!lf_cce_fused_supported(cfg, d)) {
    rc = lf_cce_forward(d_X, d_E, d_targets, n, d, v, cfg, d_lse, d_pos, d_loss, stream);
    if (rc) return rc;
    return lf_cce_backward(d_X, d_E, d_targets, d_lse, upstream, n, d, v, cfg, d_dX, d_dE, stats,
                           stream);
  }
  const double scale = upstream / static_cast<double>(n);  // cce.cpp:174
  {
    Scratch part, opart, tgt;
    int P = 0;
    rc = tc_cce_fwdx_partials(d_X, d_E, d_targets, n, static_cast<int>(d), v, 0, part, opart, tgt,
                              &P, st);
    if (!rc)
      rc = tc_fwdx_dx(part.as<float>(), opart.as<float>(), P, n, static_cast<int>(d), nullptr, d_E,
                      tgt.as<int32_t>(), scale, d_lse, d_pos, static_cast<float*>(d_dX), st);
    if (!rc && d_loss) rc = launch_mean_loss(d_lse, d_pos, n, d_loss, st);
    if (rc) return rc;
  }  // the O partials go back to the pool before the dE pass
  Counters c;
  rc = c.init(st);
  if (!rc)
    rc = tc_cce_backward(d_X, d_E, d_targets, d_lse, scale, cfg->filter_eps, n, static_cast<int>(d), v,
                         0, nullptr, static_cast<float*>(d_dE), stats ? c.ptr() : nullptr, st);
  if (rc) return rc;
  if (stats) return read_stats(c, stats, n, v, st);
  return LF_OK;
}

int lf_cce_forward_partial(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                           int64_t n, int64_t d, int64_t v_shard, int64_t v_offset,
                           const lf_cce_config* cfg, float* d_part, void* stream) {
  int rc = check_cfg(cfg);
  if (!rc) rc = check_shapes(n, d, v_shard);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  switch (cfg->dtype) {
    case LF_BF16: {
      rc = check_bf16_d(d);
      if (rc) return rc;
      Scratch ws;
      float* part = nullptr;
      int P = 0;
      rc = tc_cce_forward_partials(d_X, d_E_shard, d_targets, n, static_cast<int>(d), v_shard,
                                   v_offset, ws, &part, &P, st);
      if (rc) return rc;
      // fold the per-chunk partials into one per row (log2 units)
      return launch_fold_partials(part, P, n, d_part, st);
    }
    case LF_F32:
      return simt_cce_forward_partial_log2<float>(static_cast<const float*>(d_X),
                                                  static_cast<const float*>(d_E_shard), d_targets,
                                                  n, static_cast<int>(d), v_shard, v_offset,
                                                  d_part, st);
    default:
      return simt_cce_forward_partial_log2<double>(static_cast<const double*>(d_X),
                                                   static_cast<const double*>(d_E_shard),
                                                   d_targets, n, static_cast<int>(d), v_shard,
                                                   v_offset, d_part, st);
  }
}

int lf_cce_combine(const float* d_parts, int32_t P, int64_t n, double* d_lse, double* d_pos,
                   double* d_loss, void* stream) {
  if (P < 1) return fail(LF_EINVAL, "combine: P must be >= 1");
  return launch_combine_f32log2(d_parts, P, n, d_lse, d_pos, d_loss, as_stream(stream));
}

int lf_cce_backward_shard(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                          const double* d_lse, double upstream, int64_t n, int64_t d,
                          int64_t v_shard, int64_t v_offset, int64_t v_total,
                          const lf_cce_config* cfg, void* d_dX_partial, void* d_dE_shard,
                          lf_cce_stats* stats, void* stream) {
  return backward_impl(d_X, d_E_shard, d_targets, d_lse, upstream, n, d, v_shard, v_offset,
                       v_total, cfg, d_dX_partial, d_dE_shard, stats, as_stream(stream));
}

int lf_cce_forward_partial_peer(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                                int64_t n, int64_t d, int64_t v_shard, int64_t v_offset,
                                const lf_cce_config* cfg, float* const* d_peer_parts, int32_t world,
                                int32_t rank, int64_t parity_off, void* stream) {
  int rc = check_cfg(cfg);
  if (!rc) rc = check_shapes(n, d, v_shard);
  if (rc) return rc;
  if (world < 1 || rank < 0 || rank >= world || !d_peer_parts)
    return fail(LF_EINVAL, "peer exchange: bad world / rank / peer table");
  cudaStream_t st = as_stream(stream);
  Scratch ws;
  float* part = nullptr;
  int P = 1;
  if (cfg->dtype == LF_BF16) {
    rc = check_bf16_d(d);
    if (!rc)
      rc = tc_cce_forward_partials(d_X, d_E_shard, d_targets, n, static_cast<int>(d), v_shard, v_offset,
                                   ws, &part, &P, st);
  } else {
    rc = ws.alloc(sizeof(float) * 4 * n, st);
    part = ws.as<float>();
    if (!rc && cfg->dtype == LF_F32)
      rc = simt_cce_forward_partial_log2<float>(static_cast<const float*>(d_X),
                                                static_cast<const float*>(d_E_shard), d_targets, n,
                                                static_cast<int>(d), v_shard, v_offset, part, st);
    else if (!rc)
      rc = simt_cce_forward_partial_log2<double>(static_cast<const double*>(d_X),
                                                 static_cast<const double*>(d_E_shard), d_targets, n,
                                                 static_cast<int>(d), v_shard, v_offset, part, st);
  }
  if (rc) return rc;
  // the chunk fold fused with the all-gather: each row's partial lands in
  // slot [rank] of every peer's buffer
  return peer_fold_push(part, P, n, d_peer_parts, world, rank, parity_off, st);
}

int lf_cce_backward_shard_peer(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                               const double* d_lse, double upstream, int64_t n, int64_t d,
                               int64_t v_shard, int64_t v_offset, int64_t v_total,
                               const lf_cce_config* cfg, void* d_dE_shard, lf_cce_stats* stats,
                               float* const* d_peer_dx, int32_t world, int32_t rank,
                               int64_t parity_off, void* stream) {
  if (!cfg || (cfg->dtype != LF_BF16 && cfg->dtype != LF_F32))
    return fail(LF_EUNSUPPORTED, "peer exchange: bf16 or f32 only (fp32 dX slots)");
  if (world < 1 || rank < 0 || rank >= world || !d_peer_dx)
    return fail(LF_EINVAL, "peer exchange: bad world / rank / peer table");
  if (n < 0 || d < 0) return fail(LF_EINVAL, "cce: negative extent");
  cudaStream_t st = as_stream(stream);
  Scratch dx;
  int rc = dx.alloc(sizeof(float) * std::max<int64_t>(n * d, 1), st);
  if (rc) return rc;
  const PeerPush push{d_peer_dx, world, rank, parity_off};
  return backward_impl(d_X, d_E_shard, d_targets, d_lse, upstream, n, d, v_shard, v_offset, v_total,
                       cfg, dx.ptr, d_dE_shard, stats, st, &push);
}

int lf_ccem_forward(const void* d_X, const void* d_E, const int64_t* d_inds, int64_t n,
                    int64_t d, int64_t v, int64_t w, const lf_cce_config* cfg, double* d_lse,
                    double* d_pos, double* d_loss, void* stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (n <= 0) return fail(LF_EINVAL, "fused sampled loss: zero rows; the mean loss is undefined");
  if (w < 1) return fail(LF_EINVAL, "NegIndexMatrix: width must be at least 1 (the positive slot)");
  if (d <= 0 || v <= 0) return fail(LF_EINVAL, "fused sampled loss: empty embedding or catalog");
  return ccem_forward(cfg->dtype, d_X, d_E, d_inds, n, static_cast<int>(d), v, w, d_lse, d_pos,
                      d_loss, as_stream(stream));
}

int lf_ccem_backward(const void* d_X, const void* d_E, const int64_t* d_inds, const double* d_lse,
                     const double* d_row_upstream, double upstream, int64_t n, int64_t d,
                     int64_t v, int64_t w, const lf_cce_config* cfg, void* d_dX, void* d_dE,
                     void* stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (n <= 0) return fail(LF_EINVAL, "fused sampled loss: zero rows; the mean loss is undefined");
  if (w < 1) return fail(LF_EINVAL, "NegIndexMatrix: width must be at least 1 (the positive slot)");
  if (d <= 0 || v <= 0) return fail(LF_EINVAL, "fused sampled loss: empty embedding or catalog");
  if (!d_lse) return fail(LF_EINVAL, "ccem_backward: LSE vector is null");
  return ccem_backward(cfg->dtype, d_X, d_E, d_inds, d_lse, d_row_upstream, upstream, n,
                       static_cast<int>(d), v, w, (cfg->flags & LF_FLAG_ATOMIC_DE) != 0, d_dX,
                       d_dE, as_stream(stream));
}

int lf_ccem_forward_backward(const void* d_X, const void* d_E, const int64_t* d_inds, int64_t n,
                             int64_t d, int64_t v, int64_t w, const double* d_row_upstream,
                             double upstream, const lf_cce_config* cfg, double* d_lse, double* d_pos,
                             double* d_loss, void* d_dX, void* d_dE, void* stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (n <= 0) return fail(LF_EINVAL, "fused sampled loss: zero rows; the mean loss is undefined");
  if (w < 1) return fail(LF_EINVAL, "NegIndexMatrix: width must be at least 1 (the positive slot)");
  if (d <= 0 || v <= 0) return fail(LF_EINVAL, "fused sampled loss: empty embedding or catalog");
  if (!d_lse || !d_pos) return fail(LF_EINVAL, "ccem_forward_backward: lse / pos outputs are null");
  const bool atomic = (cfg->flags & LF_FLAG_ATOMIC_DE) != 0;
  cudaStream_t st = as_stream(stream);
  if (ccem_fused_supported(cfg->dtype, static_cast<int>(d), atomic))
    return ccem_forward_backward(cfg->dtype, d_X, d_E, d_inds, n, static_cast<int>(d), v, w,
                                 d_row_upstream, upstream, d_lse, d_pos, d_loss, d_dX, d_dE, st);
  rc = ccem_forward(cfg->dtype, d_X, d_E, d_inds, n, static_cast<int>(d), v, w, d_lse, d_pos, d_loss, st);
  if (rc) return rc;
  return ccem_backward(cfg->dtype, d_X, d_E, d_inds, d_lse, d_row_upstream, upstream, n,
                       static_cast<int>(d), v, w, atomic, d_dX, d_dE, st);
}

int lf_validate_targets(const int64_t* d_targets, int64_t n, int64_t v, void* stream) {
  if (n <= 0) return fail(LF_EINVAL, "loss: embedding matrix has zero rows; the mean loss is undefined");
  return validate_targets(d_targets, n, v, as_stream(stream));
}

int lf_validate_inds(const int64_t* d_inds, int64_t n, int64_t w, int64_t v, void* stream) {
  return validate_inds(d_inds, n, w, v, as_stream(stream));
}

int lf_classifier_to_items(const float* d_C, int64_t d, int64_t v, int32_t dtype, void* d_E,
                           void* stream) {
  if (d < 0 || v < 0) return fail(LF_EINVAL, "lf_classifier_to_items: negative extent");
  return layout_classifier_to_items(d_C, d, v, dtype, d_E, as_stream(stream));
}

int lf_convert_rows(const float* d_src, int64_t count, int32_t dtype, void* d_dst, void* stream) {
  if (count < 0) return fail(LF_EINVAL, "lf_convert_rows: negative count");
  return layout_convert_rows(d_src, count, dtype, d_dst, as_stream(stream));
}

int lf_items_grad_to_classifier(const void* d_dE, int32_t dtype, int64_t v, int64_t d,
                                double* d_dC, void* stream) {
  if (d < 0 || v < 0) return fail(LF_EINVAL, "lf_items_grad_to_classifier: negative extent");
  return layout_items_grad_to_classifier(d_dE, dtype == LF_F64 ? LF_F64 : LF_F32, v, d, d_dC,
                                         as_stream(stream));
}

int lf_widen_grad(const void* d_src, int32_t dtype, int64_t count, double* d_dst, void* stream) {
  if (count < 0) return fail(LF_EINVAL, "lf_widen_grad: negative count");
  return layout_widen(d_src, dtype == LF_F64 ? LF_F64 : LF_F32, count, d_dst, as_stream(stream));
}

int lf_ce_forward(const void* d_X, const void* d_E, const int64_t* d_targets, int64_t n,
                  int64_t d, int64_t v, const lf_cce_config* cfg, double* d_lse, double* d_pos,
                  double* d_loss, void* stream) {
  int rc = check_cfg(cfg);
  if (!rc) rc = check_shapes(n, d, v);
  if (rc) return rc;
  return ce_forward(cfg->dtype, d_X, d_E, d_targets, n, static_cast<int>(d), v, d_lse, d_pos,
                    d_loss, as_stream(stream));
}

int lf_ce_backward(const void* d_X, const void* d_E, const int64_t* d_targets, double upstream,
                   int64_t n, int64_t d, int64_t v, const lf_cce_config* cfg, void* d_dX,
                   void* d_dE, void* stream) {
  int rc = check_cfg(cfg);
  if (!rc) rc = check_shapes(n, d, v);
  if (rc) return rc;
  return ce_backward(cfg->dtype, d_X, d_E, d_targets, upstream, n, static_cast<int>(d), v, d_dX,
                     d_dE, as_stream(stream));
}

int lf_cem_forward(const void* d_X, const void* d_E, const int64_t* d_inds, int64_t n, int64_t d,
                   int64_t v, int64_t w, const lf_cce_config* cfg, double* d_lse, double* d_pos,
                   double* d_loss, void* stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (n <= 0) return fail(LF_EINVAL, "loss: embedding matrix has zero rows; the mean loss is undefined");
  if (w < 1) return fail(LF_EINVAL, "NegIndexMatrix: width must be at least 1 (the positive slot)");
  if (d <= 0 || v <= 0) return fail(LF_EINVAL, "loss: empty embedding or catalog");
  if (!d_X || !d_E || !d_inds || !d_lse || !d_pos) return fail(LF_EINVAL, "ce_sampled_forward: null pointer");
  return cem_forward(cfg->dtype, d_X, d_E, d_inds, n, static_cast<int>(d), w, d_lse, d_pos, d_loss,
                     as_stream(stream));
}

int lf_cem_backward(const void* d_X, const void* d_E, const int64_t* d_inds, double upstream, int64_t n,
                    int64_t d, int64_t v, int64_t w, const lf_cce_config* cfg, void* d_dX, void* d_dE,
                    void* stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (n <= 0) return fail(LF_EINVAL, "loss: embedding matrix has zero rows; the mean loss is undefined");
  if (w < 1) return fail(LF_EINVAL, "NegIndexMatrix: width must be at least 1 (the positive slot)");
  if (d <= 0 || v <= 0) return fail(LF_EINVAL, "loss: empty embedding or catalog");
  if (!d_X || !d_E || !d_inds || !d_dX || !d_dE) return fail(LF_EINVAL, "ce_sampled_backward: null pointer");
  return cem_backward(cfg->dtype, d_X, d_E, d_inds, upstream, n, static_cast<int>(d), v, w, d_dX, d_dE,
                      as_stream(stream));
}

int lf_sample_uniform(const int64_t* d_positives, int64_t n, int64_t ns, int64_t catalog,
                      uint64_t seed, int32_t retry_cap, int64_t* d_inds, void* stream) {
  return sample_uniform(d_positives, n, ns, catalog, seed, retry_cap, d_inds, as_stream(stream));
}

int lf_eval_rank_topk(const void* d_X, const void* d_E, const int64_t* d_targets,
                      const void* d_target_rows, int64_t n, int64_t d, int64_t v_shard,
                      int64_t v_offset, int32_t k, int32_t dtype, int64_t* d_ahead,
                      int64_t* d_top_idx, double* d_top_score, void* stream) {
  if (dtype != LF_F32 && dtype != LF_F64 && dtype != LF_BF16)
    return fail(LF_EINVAL, "eval: unknown dtype " + std::to_string(dtype));
  if (d < 1 || d > 4096) return fail(LF_EINVAL, "eval: d must be in [1, 4096]");
  return eval_rank_topk(dtype, d_X, d_E, d_targets, d_target_rows, n, static_cast<int>(d), v_shard,
                        v_offset, k, d_ahead, d_top_idx, d_top_score, as_stream(stream));
}

int lf_eval_merge(const int64_t* d_ahead, const int64_t* d_top_idx, const double* d_top_score,
                  int32_t P, int64_t n, int32_t k, int64_t* d_rank, int64_t* d_top_idx_out,
                  double* d_top_score_out, void* stream) {
  return eval_merge(d_ahead, d_top_idx, d_top_score, P, n, k, d_rank, d_top_idx_out,
                    d_top_score_out, as_stream(stream));
}

int lf_eval_summary(const int64_t* d_rank, const int64_t* d_top_idx, int64_t n, int32_t k,
                    const int64_t* d_popularity, int64_t v_total, double* out3, void* stream) {
  return eval_summary(d_rank, d_top_idx, n, k, d_popularity, v_total, out3, as_stream(stream));
}

int lf_evaluate(const void* d_X, const void* d_E, const int64_t* d_targets, int64_t n, int64_t d,
                int64_t v, int32_t k, int32_t dtype, const int64_t* d_popularity, double* out3,
                void* stream) {
  // metrics.cpp:16-33 argument checks, then k_eff = min(k, v) (metrics.cpp:34)
  if (n <= 0) return fail(LF_EINVAL, "evaluate: no eval pairs");
  if (k < 1) return fail(LF_EINVAL, "evaluate: k must be >= 1");
  if (v < 1) return fail(LF_EINVAL, "evaluate: empty catalog");
  const int32_t k_eff = static_cast<int32_t>(std::min<int64_t>(k, v));
  cudaStream_t st = as_stream(stream);
  Scratch rank, top, score;
  int rc = rank.alloc(sizeof(int64_t) * n, st);
  if (!rc) rc = top.alloc(sizeof(int64_t) * n * k_eff, st);
  if (!rc) rc = score.alloc(sizeof(double) * n * k_eff, st);
  if (!rc)
    rc = lf_eval_rank_topk(d_X, d_E, d_targets, nullptr, n, d, v, 0, k_eff, dtype, rank.as<int64_t>(),
                           top.as<int64_t>(), score.as<double>(), stream);
  if (!rc) rc = launch_add_one(rank.as<int64_t>(), n, st);
  if (!rc) rc = eval_summary(rank.as<int64_t>(), top.as<int64_t>(), n, k_eff, d_popularity, v, out3, st);
  return rc;
}

int lf_encode_batch(const int64_t* d_items, const int64_t* d_win_off, int64_t n_windows,
                    const float* d_emb, const float* d_W, const float* d_b, int64_t catalog, int64_t d,
                    int64_t rows, int32_t x_dtype, void* d_X, double* d_a, double* d_h,
                    int64_t* d_targets, int64_t* d_row_window, int64_t* d_row_pos, void* stream) {
  if (x_dtype != LF_F32 && x_dtype != LF_F64 && x_dtype != LF_BF16)
    return fail(LF_EINVAL, "encode_batch: unknown dtype " + std::to_string(x_dtype));
  return encode_batch(d_items, d_win_off, n_windows, d_emb, d_W, d_b, catalog, static_cast<int>(d), rows,
                      x_dtype, d_X, d_a, d_h, d_targets, d_row_window, d_row_pos, as_stream(stream));
}

int lf_encoder_backward(const int64_t* d_items, const int64_t* d_win_off, int64_t n_windows,
                        const float* d_W, int64_t catalog, int64_t d, const double* d_a,
                        const double* d_h, const int64_t* d_row_pos, int64_t rows, const void* d_dh,
                        int32_t dh_dtype, double* d_demb, double* d_dW, double* d_db, void* stream) {
  return encoder_backward(d_items, d_win_off, n_windows, d_W, catalog, static_cast<int>(d), d_a, d_h,
                          d_row_pos, rows, d_dh, dh_dtype, d_demb, d_dW, d_db, as_stream(stream));
}

int lf_adam_step(float* d_param, const void* d_grad, int32_t grad_dtype, double* d_m, double* d_v,
                 int64_t count, double lr, double beta1, double beta2, double eps, int64_t t,
                 void* d_shadow, int32_t shadow_dtype, void* stream) {
  return adam_step(d_param, d_grad, grad_dtype, d_m, d_v, count, lr, beta1, beta2, eps, t, d_shadow,
                   shadow_dtype, as_stream(stream));
}

int lf_sample_popularity(const int64_t* d_positives, int64_t n, int64_t ns, const int64_t* d_counts,
                         int64_t catalog, double exponent, uint64_t seed, int32_t retry_cap,
                         int64_t* d_inds, void* stream) {
  return sample_popularity(d_positives, n, ns, d_counts, catalog, exponent, seed, retry_cap, d_inds,
                           as_stream(stream));
}

int lf_estimate_flops(int64_t n, int64_t d, int64_t v, int64_t ns, int32_t backend,
                      uint64_t* forward, uint64_t* backward) {
  // ccem.cpp:207-235
  if (n < 1 || d < 1 || v < 1) return fail(LF_EINVAL, "estimate_flops: N, D, V must all be >= 1");
  uint64_t scored = 0, factor = 2;
  switch (backend) {
    case 0: scored = static_cast<uint64_t>(v); break;
    case 1: scored = 1 + static_cast<uint64_t>(ns); break;
    case 2: scored = static_cast<uint64_t>(v); factor = 3; break;
    case 3: scored = 1 + static_cast<uint64_t>(ns); factor = 3; break;
    case 4: scored = 2; break;
    default: return fail(LF_EINVAL, "estimate_flops: unknown backend " + std::to_string(backend));
  }
  const uint64_t f = static_cast<uint64_t>(n) * static_cast<uint64_t>(d) * scored;
  if (forward) *forward = f;
  if (backward) *backward = factor * f;
  return LF_OK;
}

int lf_workspace_stats(uint64_t* current_bytes, uint64_t* peak_bytes) {
  if (current_bytes) *current_bytes = g_ws_current;
  if (peak_bytes) *peak_bytes = g_ws_peak;
  return LF_OK;
}
int lf_workspace_reset_peak(void) {
  g_ws_peak = g_ws_current;
  return LF_OK;
}
uint64_t lf_launch_count(void) { return g_launches.load(); }

int lf_profile_enable(int on) {
  g_prof_on.store(on ? 1 : 0);
  return LF_OK;
}
int lf_profile_read(int32_t kind, uint64_t* launches, double* total_ms) {
  if (kind < 0 || kind >= LF_K_COUNT) return fail(LF_EINVAL, "lf_profile_read: bad kind");
  prof_drain();
  if (launches) *launches = g_prof_launches[kind];
  if (total_ms) *total_ms = g_prof_ms[kind];
  return LF_OK;
}
void lf_profile_reset(void) {
  prof_drain();
  for (int k = 0; k < LF_K_COUNT; ++k) {
    g_prof_launches[k] = 0;
    g_prof_ms[k] = 0.0;
  }
}
void lf_launch_count_reset(void) { g_launches.store(0); }

}  // extern "C"
