// microbench_pipes.cu — measures per-SM issue rates of the instructions that
// bound the CCE epilogue on B200 (sm_100a): MUFU.EX2 (f32 / f16x2 / bf16x2),
// FFMA, FMNMX3, F2FP pack, mixed f32+f16 add.  Prints one JSON line per op:
// {"op":..., "elems_per_clk_per_sm":...}.  Results are committed under
// profiles/ and feed the exp-roofline figure in DESIGN.md.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
#define CHAINS 8

template <int OP>
__global__ void __launch_bounds__(256) bench(float* out, long long* cyc, unsigned long long* ns) {
  uint32_t r[CHAINS];
  float f[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    f[c] = 0.001f * (threadIdx.x + c);
    r[c] = 0x3c003c00u + c;
  }
  long long t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[c]));
      if (OP == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r[c]));
      if (OP == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r[c]));
      if (OP == 3) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3F000000;" : "+f"(f[c]));
      if (OP == 4) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(f[(c + 1) % CHAINS]), "f"(f[(c + 2) % CHAINS]));
      if (OP == 5) asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r[c]) : "f"(f[c]), "f"(__uint_as_float(r[(c + 1) % CHAINS])));
      if (OP == 6) asm volatile("add.f32.f16 %0, %1, %0;" : "+f"(f[c]) : "h"((unsigned short)r[c]));
      if (OP == 7) asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(r[c]) : "r"(r[(c + 1) % CHAINS]));
      if (OP == 8) asm volatile("fma.rn.f32 %0, %0, %1, 0f3F000000;" : "+f"(f[c]) : "f"(f[(c + 3) % CHAINS]));
      if (OP == 9) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r[c]) : "f"(f[c]), "f"(__uint_as_float(r[(c + 1) % CHAINS])));
      if (OP == 10) asm volatile("fma.rn.f16x2 %0, %0, %1, %0;" : "+r"(r[c]) : "r"(r[(c + 1) % CHAINS]));
    }
  }
  long long t1 = clock64();
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc += f[c] + __uint_as_float(r[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = t1 - t0;
    ns[blockIdx.x] = g1 - g0;
  }
}

template <int OP>
void run(const char* name, int elems_per_op, int sms) {
  const int blocks = sms * 8, threads = 256;
  float* out;
  long long* cyc;
  unsigned long long* ns;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  cudaMalloc(&ns, sizeof(unsigned long long) * blocks);
  bench<OP><<<blocks, threads>>>(out, cyc, ns);  // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<OP><<<blocks, threads>>>(out, cyc, ns);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long hc[4096];
  unsigned long long hn[4096];
  cudaMemcpy(hc, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  cudaMemcpy(hn, ns, sizeof(unsigned long long) * blocks, cudaMemcpyDeviceToHost);
  double mhz = 0;
  for (int i = 0; i < blocks; ++i) mhz += (double)hc[i] / (double)hn[i] * 1e3;
  mhz /= blocks;
  const double total = (double)blocks * threads * ITERS * CHAINS * elems_per_op;
  const double per_s = total / (ms * 1e-3);
  const double per_clk_sm = per_s / (mhz * 1e6) / sms;
  printf("{\"op\": \"%s\", \"elems_per_s\": %.4e, \"sm_mhz\": %.0f, \"elems_per_clk_per_sm\": %.2f, \"ms\": %.3f}\n",
         name, per_s, mhz, per_clk_sm, ms);
  cudaFree(out);
  cudaFree(cyc);
  cudaFree(ns);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("ex2.approx.ftz.f32", 1, sms);
  run<1>("ex2.approx.f16x2", 2, sms);
  run<2>("ex2.approx.ftz.bf16x2", 2, sms);
  run<3>("fma.f32(imm)", 1, sms);
  run<8>("fma.f32(reg)", 1, sms);
  run<4>("max3.f32", 1, sms);
  run<5>("cvt.rn.f16x2.f32", 2, sms);
  run<9>("cvt.rn.bf16x2.f32", 2, sms);
  run<6>("add.f32.f16", 1, sms);
  run<7>("add.f16x2", 2, sms);
  run<10>("fma.f16x2", 2, sms);
  return 0;
}
