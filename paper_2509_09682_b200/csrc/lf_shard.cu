// lf_shard.cu — catalog sharding without PyTorch: the C communicator
// (lf_comm: all-gather + float sum all-reduce, stream-ordered), its NCCL and
// peer-memory backends, and the sharded CCE entry points that run the two
// exchanges of SURVEY.md 8(e) through it:
//
//   forward   local (m, s, t) partials over the shard -> ONE all-gather of
//             n float4 -> combine (every rank gets the global lse / pos / loss)
//   backward  dE rows of the shard are complete locally; dX is the shard's
//             partial sum -> ONE sum all-reduce of n x d floats
//
// lf_cce_forward_backward_sharded runs the fused kernel (FWDX) when the
// configuration allows (bf16, d = 64 / 128, eps < 2^-12): local partials +
// the unnormalised dX sum in one pass, the all-gather, then dX normalised by
// the global lse (lf_cce_fwdx_shard_end) and the dE pass.  The phase API
// (lf_cce_fwdx_shard_begin / _end) lets a caller use its own collectives.
//
// The NCCL backend binds libnccl.so.2 at run time (dlopen: a process that
// already loaded NCCL — e.g. PyTorch's — hands its own ncclComm_t over and
// the same library serves it).  The peer backend maps every rank's exchange
// buffer through CUDA IPC; handles are exchanged by the caller (any
// bootstrap: files, sockets, MPI), and the flag barrier is bounded.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "lf_internal.cuh"
#include "lf_kernels.cuh"

namespace lf {

// ------------------------------------------------------------------ NCCL --
namespace {
// Declarations mirror nccl.h (2.x): opaque communicator, int result codes.
using nccl_comm_t = void*;
using nccl_allgather_t = int (*)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t);
using nccl_allreduce_t = int (*)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t);
using nccl_errstr_t = const char* (*)(int);
constexpr int kNcclUint8 = 1, kNcclFloat32 = 7, kNcclSum = 0;

struct NcclSyms {
  nccl_allgather_t allgather = nullptr;
  nccl_allreduce_t allreduce = nullptr;
  nccl_errstr_t errstr = nullptr;
};

const NcclSyms* nccl_syms() {
  static NcclSyms s;
  static bool tried = false;
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the one already in the process
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      s.allgather = reinterpret_cast<nccl_allgather_t>(dlsym(h, "ncclAllGather"));
      s.allreduce = reinterpret_cast<nccl_allreduce_t>(dlsym(h, "ncclAllReduce"));
      s.errstr = reinterpret_cast<nccl_errstr_t>(dlsym(h, "ncclGetErrorString"));
    }
  }
  return s.allgather && s.allreduce ? &s : nullptr;
}

int nccl_fail(int r, const char* what) {
  const NcclSyms* s = nccl_syms();
  return fail(LF_ECUDA, std::string("NCCL ") + what + " failed: " + (s && s->errstr ? s->errstr(r) : "?"));
}

int nccl_allgather(void* ctx, const void* send, void* recv, uint64_t bytes, void* stream) {
  const int r = nccl_syms()->allgather(send, recv, bytes, kNcclUint8, ctx, static_cast<cudaStream_t>(stream));
  return r ? nccl_fail(r, "ncclAllGather") : LF_OK;
}
int nccl_allreduce(void* ctx, float* buf, uint64_t count, void* stream) {
  const int r = nccl_syms()->allreduce(buf, buf, count, kNcclFloat32, kNcclSum, ctx,
                                       static_cast<cudaStream_t>(stream));
  return r ? nccl_fail(r, "ncclAllReduce") : LF_OK;
}

// ------------------------------------------------------------------ peer --
// One exchange buffer per rank: two epoch-parity halves of `cap` bytes, each
// holding `world` slots; flags: one uint32 per peer plus an abort word.
struct PeerComm {
  int world = 0, rank = 0;
  uint64_t cap = 0;  // bytes per slot
  void* own = nullptr;        // this rank's buffer (cudaMalloc, exported)
  uint32_t* own_flags = nullptr;
  void** peers_h = nullptr;   // host copies of the mapped pointers
  void** d_peers = nullptr;   // device array [world] of data buffers
  uint32_t** d_flags = nullptr;  // device array [world] of flag arrays
  uint32_t epoch = 0;
  bool opened = false;
};

__device__ unsigned g_peer_error = 0;  // set when a barrier timed out or saw an abort

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Bounded barrier: thread q signals peer q, then waits for peer q's signal
// for `epoch`, for at most timeout_ns, or until some rank raised the abort
// word (flags[world]) — then it records the failure and returns.
__global__ void bounded_barrier(uint32_t* const* __restrict__ flags, int world, int rank, uint32_t epoch,
                                uint64_t timeout_ns) {
  const int q = threadIdx.x;
  if (q >= world) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags[q] + rank), "r"(epoch) : "memory");
  const uint32_t* mine = flags[rank] + q;
  const uint32_t* abort_word = flags[rank] + world;
  const uint64_t t0 = global_ns();
  for (uint32_t spin = 0;; ++spin) {
    uint32_t seen, ab;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(seen) : "l"(mine) : "memory");
    if (static_cast<int32_t>(seen - epoch) >= 0) return;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(ab) : "l"(abort_word) : "memory");
    if (ab != 0 || ((spin & 255) == 0 && global_ns() - t0 > timeout_ns)) {
      atomicOr(&g_peer_error, ab != 0 ? 2u : 1u);
      return;
    }
  }
}

__global__ void raise_abort(uint32_t* const* __restrict__ flags, int world) {
  const int q = threadIdx.x;
  if (q < world) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags[q] + world), "r"(1u) : "memory");
  }
}

// d_recv[r] <- slot r of this rank's buffer, after every rank stored into it
__global__ void push_slot(const uint4* __restrict__ src, uint64_t n16, void* const* __restrict__ peers,
                          int world, int rank, uint64_t slot_off) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint4 v = src[i];
    for (int r = 0; r < world; ++r)
      reinterpret_cast<uint4*>(static_cast<unsigned char*>(peers[r]) + slot_off)[i] = v;
  }
}

__global__ void sum_slots_f32(const float* __restrict__ slots, int world, uint64_t count, uint64_t stride,
                              float* __restrict__ out) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    float acc = slots[i];
    for (int r = 1; r < world; ++r) acc += slots[r * stride + i];  // fixed rank order
    out[i] = acc;
  }
}

uint64_t peer_timeout_ns() {
  const char* e = std::getenv("LSEFORGE_PEER_TIMEOUT_MS");
  const double ms = e ? std::atof(e) : 60000.0;
  return static_cast<uint64_t>((ms > 0 ? ms : 60000.0) * 1e6);
}

int peer_barrier_bounded(PeerComm* pc, cudaStream_t st) {
  ++pc->epoch;
  bounded_barrier<<<1, 32 * ((pc->world + 31) / 32), 0, st>>>(pc->d_flags, pc->world, pc->rank, pc->epoch,
                                                             peer_timeout_ns());
  LF_LAUNCHED();
  return LF_OK;
}

// Slot layout inside a buffer: [parity][rank][cap bytes]
uint64_t slot_offset(const PeerComm* pc, int rank) {
  return (static_cast<uint64_t>(pc->epoch & 1u) * pc->world + rank) * pc->cap;
}

int peer_allgather(void* ctx, const void* send, void* recv, uint64_t bytes, void* stream) {
  auto* pc = static_cast<PeerComm*>(ctx);
  if (bytes > pc->cap || bytes % 16) return fail(LF_EINVAL, "peer comm: all-gather size exceeds capacity or is not 16-B aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t off = slot_offset(pc, pc->rank);
  const uint64_t n16 = bytes / 16;
  if (n16) {
    push_slot<<<static_cast<unsigned>(std::min<uint64_t>(ceil_div(n16, 256), 4ull * num_sms())), 256, 0, st>>>(
        static_cast<const uint4*>(send), n16, pc->d_peers, pc->world, pc->rank, off);
    LF_LAUNCHED();
  }
  const uint64_t base = slot_offset(pc, 0);
  int rc = peer_barrier_bounded(pc, st);
  if (rc) return rc;
  // this rank's buffer now holds every rank's block for the old parity
  for (int r = 0; r < pc->world; ++r)
    LF_CUDA(cudaMemcpyAsync(static_cast<unsigned char*>(recv) + r * bytes,
                            static_cast<unsigned char*>(pc->own) + base + r * pc->cap, bytes,
                            cudaMemcpyDeviceToDevice, st));
  return LF_OK;
}

int peer_allreduce(void* ctx, float* buf, uint64_t count, void* stream) {
  auto* pc = static_cast<PeerComm*>(ctx);
  const uint64_t bytes = count * sizeof(float);
  if (bytes > pc->cap || bytes % 16) return fail(LF_EINVAL, "peer comm: all-reduce size exceeds capacity or is not 16-B aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t off = slot_offset(pc, pc->rank);
  const uint64_t n16 = bytes / 16;
  if (n16) {
    push_slot<<<static_cast<unsigned>(std::min<uint64_t>(ceil_div(n16, 256), 4ull * num_sms())), 256, 0, st>>>(
        reinterpret_cast<const uint4*>(buf), n16, pc->d_peers, pc->world, pc->rank, off);
    LF_LAUNCHED();
  }
  const uint64_t base = slot_offset(pc, 0);
  int rc = peer_barrier_bounded(pc, st);
  if (rc) return rc;
  if (count) {
    sum_slots_f32<<<static_cast<unsigned>(std::min<uint64_t>(ceil_div(count, 256), 8ull * num_sms())), 256, 0,
                    st>>>(reinterpret_cast<const float*>(static_cast<unsigned char*>(pc->own) + base), pc->world,
                          count, pc->cap / sizeof(float), buf);
    LF_LAUNCHED();
  }
  return LF_OK;
}

constexpr uint64_t kHandleBytes = 2 * sizeof(cudaIpcMemHandle_t);  // data + flags

}  // namespace
}  // namespace lf

// ------------------------------------------------------------------ C-ABI --
using namespace lf;

struct lf_peer_comm {
  PeerComm pc;
};

struct lf_cce_work {
  Scratch part, opart, tgt;
  int P = 0;
  const void* X = nullptr;
  const void* E = nullptr;
  const int64_t* targets = nullptr;
  int64_t n = 0, d = 0, v_shard = 0, v_offset = 0;
  lf_cce_config cfg{};
};

namespace {
cudaStream_t sst(void* s) { return static_cast<cudaStream_t>(s); }
// Sum this rank's skip counters over the ranks (one all-gather of 32 bytes;
// the stats read-out already synchronised the stream).
int gather_stats(const lf_comm* c, lf_cce_stats* stats, int64_t n, int64_t v_total, cudaStream_t st) {
  if (!stats || c->world == 1) return LF_OK;
  Scratch buf;
  int rc = buf.alloc(sizeof(uint64_t) * 4 * (c->world + 1), st);
  if (rc) return rc;
  const uint64_t mine[4] = {stats->skipped_elems, stats->skipped_tiles, stats->total_tiles, 0};
  LF_CUDA(cudaMemcpyAsync(buf.ptr, mine, sizeof(mine), cudaMemcpyHostToDevice, st));
  rc = c->allgather(c->ctx, buf.ptr, buf.as<uint64_t>() + 4, sizeof(mine), st);
  if (rc) return rc;
  std::vector<uint64_t> all(4 * c->world);
  LF_CUDA(cudaMemcpyAsync(all.data(), buf.as<uint64_t>() + 4, sizeof(uint64_t) * all.size(),
                          cudaMemcpyDeviceToHost, st));
  LF_CUDA(cudaStreamSynchronize(st));
  stats->skipped_elems = stats->skipped_tiles = stats->total_tiles = 0;
  for (int r = 0; r < c->world; ++r) {
    stats->skipped_elems += all[4 * r];
    stats->skipped_tiles += all[4 * r + 1];
    stats->total_tiles += all[4 * r + 2];
  }
  const double off = static_cast<double>(n) * static_cast<double>(v_total - 1);
  stats->skipped_fraction = off == 0.0 ? 0.0 : static_cast<double>(stats->skipped_elems) / off;
  return LF_OK;
}

int check_comm(const lf_comm* c) {
  if (!c || !c->allgather || !c->allreduce_sum_f32 || c->world < 1 || c->rank < 0 || c->rank >= c->world)
    return fail(LF_EINVAL, "lf_comm: incomplete communicator (callbacks, world, rank)");
  return LF_OK;
}
}  // namespace

extern "C" {

LF_API int lf_comm_nccl(void* nccl_comm, int32_t world, int32_t rank, lf_comm* out) {
  if (!nccl_comm || !out || world < 1 || rank < 0 || rank >= world)
    return fail(LF_EINVAL, "lf_comm_nccl: null communicator / output or bad world / rank");
  if (!nccl_syms()) return fail(LF_EUNSUPPORTED, "lf_comm_nccl: libnccl.so.2 not found");
  out->ctx = nccl_comm;
  out->world = world;
  out->rank = rank;
  out->allgather = nccl_allgather;
  out->allreduce_sum_f32 = nccl_allreduce;
  return LF_OK;
}

LF_API int lf_peer_comm_create(uint64_t slot_bytes, int32_t world, int32_t rank, lf_peer_comm** out,
                               void* handle_out) {
  if (!out || !handle_out || world < 1 || world > 1024 || rank < 0 || rank >= world)
    return fail(LF_EINVAL, "lf_peer_comm_create: bad arguments");
  auto* h = new lf_peer_comm;
  PeerComm& pc = h->pc;
  pc.world = world;
  pc.rank = rank;
  pc.cap = (slot_bytes + 15) / 16 * 16;
  const uint64_t data_bytes = 2 * static_cast<uint64_t>(world) * pc.cap;
  cudaIpcMemHandle_t hd, hf;
  cudaError_t e = cudaMalloc(&pc.own, data_bytes ? data_bytes : 16);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&pc.own_flags), sizeof(uint32_t) * (world + 1));
  if (e == cudaSuccess) e = cudaMemset(pc.own_flags, 0, sizeof(uint32_t) * (world + 1));
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hd, pc.own);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hf, pc.own_flags);
  if (e != cudaSuccess) {
    cudaFree(pc.own);
    cudaFree(pc.own_flags);
    delete h;
    return cuda_fail(e, "lf_peer_comm_create");
  }
  std::memcpy(handle_out, &hd, sizeof(hd));
  std::memcpy(static_cast<unsigned char*>(handle_out) + sizeof(hd), &hf, sizeof(hf));
  *out = h;
  return LF_OK;
}

LF_API uint64_t lf_peer_comm_handle_bytes(void) { return kHandleBytes; }

LF_API int lf_peer_comm_open(lf_peer_comm* h, const void* all_handles, lf_comm* out) {
  if (!h || !all_handles || !out) return fail(LF_EINVAL, "lf_peer_comm_open: null argument");
  PeerComm& pc = h->pc;
  const int W = pc.world;
  pc.peers_h = new void*[2 * W]();
  void** flags_h = pc.peers_h + W;
  for (int r = 0; r < W; ++r) {
    const unsigned char* hr = static_cast<const unsigned char*>(all_handles) + r * kHandleBytes;
    if (r == pc.rank) {
      pc.peers_h[r] = pc.own;
      flags_h[r] = pc.own_flags;
      continue;
    }
    cudaIpcMemHandle_t hd, hf;
    std::memcpy(&hd, hr, sizeof(hd));
    std::memcpy(&hf, hr + sizeof(hd), sizeof(hf));
    LF_CUDA(cudaIpcOpenMemHandle(&pc.peers_h[r], hd, cudaIpcMemLazyEnablePeerAccess));
    LF_CUDA(cudaIpcOpenMemHandle(&flags_h[r], hf, cudaIpcMemLazyEnablePeerAccess));
  }
  LF_CUDA(cudaMalloc(reinterpret_cast<void**>(&pc.d_peers), sizeof(void*) * W));
  LF_CUDA(cudaMalloc(reinterpret_cast<void**>(&pc.d_flags), sizeof(void*) * W));
  LF_CUDA(cudaMemcpy(pc.d_peers, pc.peers_h, sizeof(void*) * W, cudaMemcpyHostToDevice));
  LF_CUDA(cudaMemcpy(pc.d_flags, flags_h, sizeof(void*) * W, cudaMemcpyHostToDevice));
  pc.opened = true;
  out->ctx = &pc;
  out->world = W;
  out->rank = pc.rank;
  out->allgather = peer_allgather;
  out->allreduce_sum_f32 = peer_allreduce;
  return LF_OK;
}

LF_API int lf_peer_comm_abort(lf_peer_comm* h, void* stream) {
  if (!h || !h->pc.opened) return fail(LF_EINVAL, "lf_peer_comm_abort: not opened");
  raise_abort<<<1, 32 * ((h->pc.world + 31) / 32), 0, sst(stream)>>>(h->pc.d_flags, h->pc.world);
  LF_LAUNCHED();
  return LF_OK;
}

LF_API int lf_peer_comm_status(void) {
  unsigned v = 0;
  LF_CUDA(cudaMemcpyFromSymbol(&v, g_peer_error, sizeof(v)));
  if (v & 2u) return fail(LF_ERUNTIME, "peer exchange: a rank raised the abort word");
  if (v & 1u) return fail(LF_ERUNTIME, "peer exchange: barrier timed out (LSEFORGE_PEER_TIMEOUT_MS)");
  return LF_OK;
}

LF_API int lf_peer_comm_destroy(lf_peer_comm* h) {
  if (!h) return LF_OK;
  PeerComm& pc = h->pc;
  if (pc.opened) {
    void** flags_h = pc.peers_h + pc.world;
    for (int r = 0; r < pc.world; ++r) {
      if (r == pc.rank) continue;
      if (pc.peers_h[r]) cudaIpcCloseMemHandle(pc.peers_h[r]);
      if (flags_h[r]) cudaIpcCloseMemHandle(flags_h[r]);
    }
    cudaFree(pc.d_peers);
    cudaFree(pc.d_flags);
  }
  delete[] pc.peers_h;
  cudaFree(pc.own);
  cudaFree(pc.own_flags);
  delete h;
  return LF_OK;
}

// ---------------------------------------------------------- fused phases --
LF_API int lf_cce_fwdx_shard_begin(const void* d_X, const void* d_E_shard, const int64_t* d_targets, int64_t n,
                                   int64_t d, int64_t v_shard, int64_t v_offset, const lf_cce_config* cfg,
                                   float* d_part, lf_cce_work** work, void* stream) {
  if (!cfg || !work || !d_part) return fail(LF_EINVAL, "lf_cce_fwdx_shard_begin: null argument");
  if (n <= 0) return fail(LF_EINVAL, "loss: embedding matrix has zero rows; the mean loss is undefined");
  if (v_shard <= 0) return fail(LF_EINVAL, "loss: catalog must hold at least one item");
  if (!(cfg->filter_eps >= 0.0))
    return fail(LF_EINVAL, "CceConfig: filter_eps must be >= 0, got " + std::to_string(cfg->filter_eps));
  if (!lf_cce_fused_supported(cfg, d))
    return fail(LF_EUNSUPPORTED, "fused sharded step: needs bf16, d = 64 / 128, filter_eps < 2^-12 "
                                 "(use lf_cce_forward_partial / lf_cce_backward_shard)");
  cudaStream_t st = sst(stream);
  auto* w = new lf_cce_work;
  w->X = d_X;
  w->E = d_E_shard;
  w->targets = d_targets;
  w->n = n;
  w->d = d;
  w->v_shard = v_shard;
  w->v_offset = v_offset;
  w->cfg = *cfg;
  int rc = tc_cce_fwdx_partials(d_X, d_E_shard, d_targets, n, static_cast<int>(d), v_shard, v_offset, w->part,
                                w->opart, w->tgt, &w->P, st);
  if (!rc) rc = launch_fold_partials(w->part.as<float>(), w->P, n, d_part, st);
  if (rc) {
    delete w;
    return rc;
  }
  *work = w;
  return LF_OK;
}

LF_API int lf_cce_fwdx_shard_end(lf_cce_work* w, const float* d_parts, int32_t P, double upstream,
                                 int64_t v_total, double* d_lse, double* d_pos, double* d_loss,
                                 void* d_dX_partial, void* d_dE_shard, lf_cce_stats* stats, void* stream) {
  if (!w) return fail(LF_EINVAL, "lf_cce_fwdx_shard_end: null work");
  cudaStream_t st = sst(stream);
  int rc = P < 1 ? fail(LF_EINVAL, "combine: P must be >= 1") : LF_OK;
  if (!rc) rc = launch_combine_f32log2(d_parts, P, w->n, d_lse, d_pos, d_loss, st);
  const double scale = upstream / static_cast<double>(w->n);  // cce.cpp:174
  if (!rc)
    rc = tc_fwdx_dx(w->part.as<float>(), w->opart.as<float>(), w->P, w->n, static_cast<int>(w->d), d_lse,
                    w->E, w->tgt.as<int32_t>(), scale, nullptr, nullptr, static_cast<float*>(d_dX_partial), st);
  // the O partials go back to the pool before the dE pass
  const void* X = w->X;
  const void* E = w->E;
  const int64_t* targets = w->targets;
  const int64_t n = w->n, d = w->d, v_shard = w->v_shard, v_offset = w->v_offset;
  const double eps = w->cfg.filter_eps;
  delete w;
  if (rc) return rc;
  Scratch counters;
  rc = counters.alloc(4 * sizeof(unsigned long long), st);
  if (rc) return rc;
  LF_CUDA(cudaMemsetAsync(counters.ptr, 0, 4 * sizeof(unsigned long long), st));
  rc = tc_cce_backward(X, E, targets, d_lse, scale, eps, n, static_cast<int>(d), v_shard, v_offset, nullptr,
                       static_cast<float*>(d_dE_shard), stats ? counters.as<unsigned long long>() : nullptr, st);
  if (rc) return rc;
  if (stats) {
    unsigned long long h[4] = {0, 0, 0, 0};
    LF_CUDA(cudaMemcpyAsync(h, counters.ptr, sizeof(h), cudaMemcpyDeviceToHost, st));
    LF_CUDA(cudaStreamSynchronize(st));
    stats->skipped_elems = h[0];
    stats->skipped_tiles = h[1];
    stats->total_tiles = h[2];
    const double off = static_cast<double>(n) * static_cast<double>(v_total - 1);
    stats->skipped_fraction = off == 0.0 ? 0.0 : static_cast<double>(h[0]) / off;
  }
  return LF_OK;
}

LF_API int lf_cce_work_free(lf_cce_work* w) {
  delete w;
  return LF_OK;
}

// ------------------------------------------------------- one-shot sharded --
LF_API int lf_cce_forward_sharded(const void* d_X, const void* d_E_shard, const int64_t* d_targets, int64_t n,
                                  int64_t d, int64_t v_shard, int64_t v_offset, const lf_cce_config* cfg,
                                  const lf_comm* comm, double* d_lse, double* d_pos, double* d_loss,
                                  void* stream) {
  int rc = check_comm(comm);
  if (rc) return rc;
  cudaStream_t st = sst(stream);
  Scratch mine, all;
  rc = mine.alloc(sizeof(float) * 4 * std::max<int64_t>(n, 1), st);
  if (!rc) rc = all.alloc(sizeof(float) * 4 * std::max<int64_t>(n, 1) * comm->world, st);
  if (!rc) rc = lf_cce_forward_partial(d_X, d_E_shard, d_targets, n, d, v_shard, v_offset, cfg, mine.as<float>(), stream);
  if (!rc) rc = comm->allgather(comm->ctx, mine.ptr, all.ptr, sizeof(float) * 4 * n, stream);
  if (!rc) rc = lf_cce_combine(all.as<float>(), comm->world, n, d_lse, d_pos, d_loss, stream);
  return rc;
}

LF_API int lf_cce_backward_sharded(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                                   const double* d_lse, double upstream, int64_t n, int64_t d, int64_t v_shard,
                                   int64_t v_offset, int64_t v_total, const lf_cce_config* cfg,
                                   const lf_comm* comm, void* d_dX, void* d_dE_shard, lf_cce_stats* stats,
                                   void* stream) {
  int rc = check_comm(comm);
  if (rc) return rc;
  if (cfg && cfg->dtype == LF_F64)
    return fail(LF_EUNSUPPORTED, "sharded backward: the dX exchange sums fp32 (bf16 / f32 only)");
  rc = lf_cce_backward_shard(d_X, d_E_shard, d_targets, d_lse, upstream, n, d, v_shard, v_offset, v_total, cfg,
                             d_dX, d_dE_shard, stats, stream);
  if (!rc) rc = comm->allreduce_sum_f32(comm->ctx, static_cast<float*>(d_dX), static_cast<uint64_t>(n * d), stream);
  if (!rc) rc = gather_stats(comm, stats, n, v_total, sst(stream));
  return rc;
}

LF_API int lf_cce_forward_backward_sharded(const void* d_X, const void* d_E_shard, const int64_t* d_targets,
                                           int64_t n, int64_t d, int64_t v_shard, int64_t v_offset,
                                           int64_t v_total, double upstream, const lf_cce_config* cfg,
                                           const lf_comm* comm, double* d_lse, double* d_pos, double* d_loss,
                                           void* d_dX, void* d_dE_shard, lf_cce_stats* stats, void* stream) {
  int rc = check_comm(comm);
  if (rc) return rc;
  if (!cfg) return fail(LF_EINVAL, "CceConfig: null config");
  if (!lf_cce_fused_supported(cfg, d)) {
    rc = lf_cce_forward_sharded(d_X, d_E_shard, d_targets, n, d, v_shard, v_offset, cfg, comm, d_lse, d_pos,
                                d_loss, stream);
    if (!rc)
      rc = lf_cce_backward_sharded(d_X, d_E_shard, d_targets, d_lse, upstream, n, d, v_shard, v_offset, v_total,
                                   cfg, comm, d_dX, d_dE_shard, stats, stream);
    return rc;
  }
  cudaStream_t st = sst(stream);
  Scratch mine, all;
  rc = mine.alloc(sizeof(float) * 4 * n, st);
  if (!rc) rc = all.alloc(sizeof(float) * 4 * n * comm->world, st);
  if (rc) return rc;
  lf_cce_work* w = nullptr;
  rc = lf_cce_fwdx_shard_begin(d_X, d_E_shard, d_targets, n, d, v_shard, v_offset, cfg, mine.as<float>(), &w,
                               stream);
  if (!rc) rc = comm->allgather(comm->ctx, mine.ptr, all.ptr, sizeof(float) * 4 * n, stream);
  if (rc) {
    lf_cce_work_free(w);
    return rc;
  }
  rc = lf_cce_fwdx_shard_end(w, all.as<float>(), comm->world, upstream, v_total, d_lse, d_pos, d_loss, d_dX,
                             d_dE_shard, stats, stream);
  if (!rc) rc = comm->allreduce_sum_f32(comm->ctx, static_cast<float*>(d_dX), static_cast<uint64_t>(n * d), stream);
  if (!rc) rc = gather_stats(comm, stats, n, v_total, st);
  return rc;
}

}  // extern "C"
