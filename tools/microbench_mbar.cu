// microbench_mbar.cu — latency of mbarrier waits on an already-completed
// phase (the MMA-issuer's per-tile cost), and of arrive + wait round trips.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int OP>
__global__ void bench(long long* out) {
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[0])) : "memory");
  }
  __syncthreads();
  const uint32_t a = smem_u32(&bar[0]);
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) {
    uint32_t ok;
    if (OP == 0) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(a), "r"(0u) : "memory");
    } else if (OP == 1) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(a), "r"(0u), "r"(0x989680) : "memory");
    } else {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(a), "r"(0u) : "memory");
    }
    acc += ok;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) * 1000 + acc % 1000;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 148);
  const char* names[3] = {"try_wait(done phase)", "try_wait+hint(done phase)", "test_wait(done phase)"};
  for (int op = 0; op < 3; ++op) {
    for (int threads : {32, 320}) {
      if (op == 0) bench<0><<<148, threads>>>(d);
      if (op == 1) bench<1><<<148, threads>>>(d);
      if (op == 2) bench<2><<<148, threads>>>(d);
      cudaDeviceSynchronize();
      long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("{\"op\": \"%s\", \"threads\": %d, \"cycles_per_wait\": %.1f}\n", names[op], threads,
             (h / 1000) / 1000.0);
    }
  }
  return 0;
}
