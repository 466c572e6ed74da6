// lf_peer.cu — the catalog-sharded exchanges over peer memory instead of
// NCCL: every rank maps every other rank's exchange buffer (CUDA IPC; on an
// NVSwitch box the stores travel over NVLink), and the kernels that produce a
// rank's contribution store it straight into all peers' buffers:
//
//   forward   fold of the per-chunk (m, s, t) partials -> each peer's slot
//             [rank][row] (the all-gather fused into the fold kernel), then a
//             flag barrier, then lf_cce_combine over the local P x n block;
//   backward  the dX chunk reduce -> each peer's slot [rank] (the all-gather
//             half of an all-reduce fused into the reduce), barrier, then a
//             fixed-order sum of the P slots (identical bits on every rank).
//
// Buffers alternate by epoch parity, so a rank can run ahead into the next
// exchange without overwriting a slot a slower peer is still reading.
// Flags: flag[q] on rank p = the last epoch rank q finished writing into p;
// signalled with a system-scope release after a system fence, waited on with
// system-scope acquires.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "lf_internal.cuh"
#include "lf_kernels.cuh"

namespace lf {
namespace {

__global__ void fold_push(const float4* __restrict__ part, int P, int64_t n, float4* const* __restrict__ peers,
                          int world, int rank, int64_t parity_off) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // same arithmetic as fold_partials (lf_simt.cu)
  float M = -INFINITY;
  for (int p = 0; p < P; ++p) M = fmaxf(M, part[p * n + i].x);
  float S = 0.f, t = 0.f, h = 0.f;
  for (int p = 0; p < P; ++p) {
    const float4 q = part[p * n + i];
    if (q.x != -INFINITY) S += q.y * exp2f(q.x - M);
    if (q.w != 0.f) {
      t = q.z;
      h = 1.f;
    }
  }
  const float4 o = make_float4(M, S, t, h);
  for (int r = 0; r < world; ++r) peers[r][parity_off + static_cast<int64_t>(rank) * n + i] = o;
}

__global__ void reduce_push(const float* __restrict__ part, int P, int64_t count, float* const* __restrict__ peers,
                            int world, int rank, int64_t parity_off) {
  // fixed chunk order, as reduce_chunks (lf_simt.cu); 4 floats per thread
  const int64_t n4 = count / 4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(part)[i];
    for (int p = 1; p < P; ++p) {
      const float4 q = reinterpret_cast<const float4*>(part + p * count)[i];
      acc.x += q.x;
      acc.y += q.y;
      acc.z += q.z;
      acc.w += q.w;
    }
    for (int r = 0; r < world; ++r)
      reinterpret_cast<float4*>(peers[r] + parity_off + static_cast<int64_t>(rank) * count)[i] = acc;
  }
  if (blockIdx.x == 0 && threadIdx.x < count - n4 * 4) {  // tail
    const int64_t i = n4 * 4 + threadIdx.x;
    float acc = part[i];
    for (int p = 1; p < P; ++p) acc += part[p * count + i];
    for (int r = 0; r < world; ++r) peers[r][parity_off + static_cast<int64_t>(rank) * count + i] = acc;
  }
}

__device__ unsigned g_barrier_timeout = 0;  // a barrier gave up waiting (lf_peer_status)

// One block: thread q < world signals peer q, then waits for peer q's signal
// — for at most timeout_ns (a rank that died or raised an error before its
// signal must not hang every other rank's GPU): then it records the timeout
// and returns, and lf_peer_status reports it.
__global__ void peer_barrier(uint32_t* const* __restrict__ flags, int world, int rank, uint32_t epoch,
                             uint64_t timeout_ns) {
  const int q = threadIdx.x;
  if (q >= world) return;
  __threadfence_system();
  uint32_t* remote = flags[q] + rank;
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(remote), "r"(epoch) : "memory");
  const uint32_t* mine = flags[rank] + q;
  uint64_t t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (uint32_t spin = 0;; ++spin) {
    uint32_t seen;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(seen) : "l"(mine) : "memory");
    if (static_cast<int32_t>(seen - epoch) >= 0) return;
    if ((spin & 255) == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicExch(&g_barrier_timeout, 1u);
        return;
      }
    }
  }
}

__global__ void sum_slots(const float* __restrict__ slots, int world, int64_t count, float* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = slots[i];
    for (int r = 1; r < world; ++r) acc += slots[static_cast<int64_t>(r) * count + i];
    out[i] = acc;
  }
}

}  // namespace

int peer_fold_push(const float* part, int P, int64_t n, float* const* peers, int world, int rank,
                   int64_t parity_off_floats, cudaStream_t st) {
  if (n == 0) return LF_OK;
  fold_push<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, st>>>(
      reinterpret_cast<const float4*>(part), P, n, reinterpret_cast<float4* const*>(peers), world, rank,
      parity_off_floats / 4);
  LF_LAUNCHED();
  return LF_OK;
}

int peer_reduce_push(const float* part, int P, int64_t count, float* const* peers, int world, int rank,
                     int64_t parity_off_floats, cudaStream_t st) {
  if (count == 0) return LF_OK;
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(count / 4 + 1, 256), 8LL * num_sms()));
  reduce_push<<<grid, 256, 0, st>>>(part, P, count, peers, world, rank, parity_off_floats);
  LF_LAUNCHED();
  return LF_OK;
}

}  // namespace lf

// ------------------------------------------------------------------ C-ABI --
using namespace lf;

namespace {
cudaStream_t as_st(void* s) { return static_cast<cudaStream_t>(s); }
}  // namespace

extern "C" {

LF_API int lf_peer_alloc(uint64_t bytes, void** d_ptr, void* ipc_handle) {
  if (!d_ptr || !ipc_handle) return fail(LF_EINVAL, "lf_peer_alloc: null output");
  LF_CUDA(cudaMalloc(d_ptr, bytes));
  LF_CUDA(cudaMemset(*d_ptr, 0, bytes));
  cudaIpcMemHandle_t h;
  LF_CUDA(cudaIpcGetMemHandle(&h, *d_ptr));
  std::memcpy(ipc_handle, &h, sizeof(h));
  return LF_OK;
}

LF_API int lf_peer_open(const void* ipc_handle, void** d_ptr) {
  if (!d_ptr || !ipc_handle) return fail(LF_EINVAL, "lf_peer_open: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, ipc_handle, sizeof(h));
  LF_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return LF_OK;
}

LF_API int lf_peer_close(void* d_ptr) {
  LF_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return LF_OK;
}

LF_API int lf_peer_free(void* d_ptr) {
  LF_CUDA(cudaFree(d_ptr));
  return LF_OK;
}

LF_API int lf_peer_barrier(uint32_t* const* d_peer_flags, int32_t world, int32_t rank, uint32_t epoch,
                           void* stream) {
  if (world < 1 || world > 1024 || rank < 0 || rank >= world) return fail(LF_EINVAL, "lf_peer_barrier: bad world/rank");
  const char* e = std::getenv("LSEFORGE_PEER_TIMEOUT_MS");
  const double ms = e && std::atof(e) > 0 ? std::atof(e) : 60000.0;
  peer_barrier<<<1, 32 * ((world + 31) / 32), 0, as_st(stream)>>>(d_peer_flags, world, rank, epoch,
                                                                  static_cast<uint64_t>(ms * 1e6));
  LF_LAUNCHED();
  return LF_OK;
}

LF_API int lf_peer_status(void) {
  unsigned v = 0;
  LF_CUDA(cudaMemcpyFromSymbol(&v, g_barrier_timeout, sizeof(v)));
  if (v) return fail(LF_ERUNTIME, "peer exchange: lf_peer_barrier timed out waiting for a peer (LSEFORGE_PEER_TIMEOUT_MS)");
  return LF_OK;
}

LF_API int lf_peer_sum(const float* d_slots, int32_t world, int64_t count, float* d_out, void* stream) {
  if (world < 1 || count < 0) return fail(LF_EINVAL, "lf_peer_sum: bad world/count");
  if (count == 0) return LF_OK;
  sum_slots<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(count, 256), 8LL * num_sms())), 256, 0,
              as_st(stream)>>>(d_slots, world, count, d_out);
  LF_LAUNCHED();
  return LF_OK;
}

}  // extern "C"
