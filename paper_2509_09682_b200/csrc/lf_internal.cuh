// lf_internal.cuh — shared host/device helpers for the lseforge_b200 library:
// error plumbing (thread-local message, status codes), launch accounting,
// the stream-ordered scratch allocator, and small device utilities.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/lseforge_b200.h"

namespace lf {

// ------------------------------------------------------------ errors -------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define LF_CUDA(expr)                                    \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return ::lf::cuda_fail(_e, #expr); \
  } while (0)

#define LF_LAUNCHED()                                  \
  do {                                                 \
    ::lf::note_launch();                               \
    cudaError_t _e = cudaGetLastError();               \
    if (_e != cudaSuccess) return ::lf::cuda_fail(_e, "kernel launch"); \
  } while (0)

void note_launch();

// Event bracket around one kernel launch when profiling is on (lf_profile_*).
struct ProfScope {
  int kind;
  cudaStream_t st;
  cudaEvent_t start = nullptr;
  ProfScope(int k, cudaStream_t s);
  ~ProfScope();
};

// --------------------------------------------------- scratch allocator ------
// Stream-ordered device scratch (cudaMallocAsync on the default mempool);
// tracks current and peak bytes for the peak-HBM figure.
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch();
  int alloc(size_t nbytes, cudaStream_t s);
  template <class T>
  T* as() const { return static_cast<T*>(ptr); }
};

int num_sms();

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ------------------------------------------------------- device utils ------
__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ double to_f64(double x) { return x; }
__device__ __forceinline__ float to_f32_or_self(float x) { return x; }
__device__ __forceinline__ float to_f32_or_self(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ double to_f32_or_self(double x) { return x; }

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

}  // namespace lf
