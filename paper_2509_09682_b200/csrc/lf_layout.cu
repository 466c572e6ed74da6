// lf_layout.cu — boundary layout conversions for callers that hold the
// reference's host layouts (the C++ drop-in shim, shim/lseforge_shim.cpp).
//
// The reference stores the item table as ref-C, a float D x V row-major
// matrix (proj/tests/support.hpp:19, cce.hpp:36), and returns d_classifier as
// a double D x V matrix (losses.hpp:24-27).  The kernels want E = ref-C^T,
// V x D row-major (one contiguous 2D-byte row per item, which CCE- gathers
// need), so the shim uploads ref-C once and converts it here on the device:
// a 32 x 32 shared-memory tile transpose with coalesced reads and writes on
// both sides.  Element conversion is exact float->double / float->float, or
// round-to-nearest-even float->bf16.
#include <cuda_bf16.h>

#include <algorithm>

#include "lf_internal.cuh"

namespace lf {
namespace {

template <class T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ double from_f32<double>(float x) { return static_cast<double>(x); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// out[c][r] = cvt(in[r][c]) for an R x Cn row-major input.
template <class Tin, class Tout, class Cvt>
__global__ void __launch_bounds__(256) transpose_tiles(const Tin* __restrict__ in, int64_t R,
                                                       int64_t Cn, Tout* __restrict__ out, Cvt cvt) {
  __shared__ Tin tile[32][33];
  const int64_t ctiles = (Cn + 31) / 32;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) / ctiles * 32;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) % ctiles * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int64_t r = r0 + ty + k, c = c0 + tx;
    if (r < R && c < Cn) tile[ty + k][tx] = in[r * Cn + c];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int64_t c = c0 + ty + k, r = r0 + tx;
    if (r < R && c < Cn) out[c * R + r] = cvt(tile[tx][ty + k]);
  }
}

template <class Tout>
struct CvtF32 {
  __device__ __forceinline__ Tout operator()(float x) const { return from_f32<Tout>(x); }
};
struct CvtToF64 {
  __device__ __forceinline__ double operator()(float x) const { return static_cast<double>(x); }
  __device__ __forceinline__ double operator()(double x) const { return x; }
};

template <class Tout>
__global__ void convert_f32(const float* __restrict__ in, int64_t count, Tout* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = from_f32<Tout>(in[i]);
}

__global__ void widen_f32(const float* __restrict__ in, int64_t count, double* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<double>(in[i]);
}

template <class Tin, class Tout, class Cvt>
int launch_transpose(const Tin* in, int64_t R, int64_t Cn, Tout* out, Cvt cvt, cudaStream_t st) {
  if (R == 0 || Cn == 0) return LF_OK;
  const int64_t tiles = ceil_div(R, 32) * ceil_div(Cn, 32);
  if (tiles > 0x7fffffff) return fail(LF_EUNSUPPORTED, "layout: transpose too large");
  transpose_tiles<<<static_cast<unsigned>(tiles), 256, 0, st>>>(in, R, Cn, out, cvt);
  LF_LAUNCHED();
  return LF_OK;
}

int grid_for(int64_t count) {
  return static_cast<int>(std::min<int64_t>(ceil_div(count, 256), 148 * 16));
}

}  // namespace

int layout_classifier_to_items(const float* C, int64_t d, int64_t v, int dtype, void* E,
                               cudaStream_t st) {
  switch (dtype) {
    case LF_F32: return launch_transpose(C, d, v, static_cast<float*>(E), CvtF32<float>{}, st);
    case LF_F64: return launch_transpose(C, d, v, static_cast<double*>(E), CvtF32<double>{}, st);
    case LF_BF16:
      return launch_transpose(C, d, v, static_cast<__nv_bfloat16*>(E), CvtF32<__nv_bfloat16>{}, st);
    default: return fail(LF_EINVAL, "layout: unknown dtype");
  }
}

int layout_convert_rows(const float* src, int64_t count, int dtype, void* dst, cudaStream_t st) {
  if (count == 0) return LF_OK;
  switch (dtype) {
    case LF_F32:
      LF_CUDA(cudaMemcpyAsync(dst, src, sizeof(float) * count, cudaMemcpyDeviceToDevice, st));
      return LF_OK;
    case LF_F64:
      convert_f32<double><<<grid_for(count), 256, 0, st>>>(src, count, static_cast<double*>(dst));
      break;
    case LF_BF16:
      convert_f32<__nv_bfloat16><<<grid_for(count), 256, 0, st>>>(
          src, count, static_cast<__nv_bfloat16*>(dst));
      break;
    default: return fail(LF_EINVAL, "layout: unknown dtype");
  }
  LF_LAUNCHED();
  return LF_OK;
}

int layout_items_grad_to_classifier(const void* dE, int grad_dtype, int64_t v, int64_t d,
                                    double* dC, cudaStream_t st) {
  if (grad_dtype == LF_F64)
    return launch_transpose(static_cast<const double*>(dE), v, d, dC, CvtToF64{}, st);
  if (grad_dtype == LF_F32)
    return launch_transpose(static_cast<const float*>(dE), v, d, dC, CvtToF64{}, st);
  return fail(LF_EINVAL, "layout: gradients are float or double");
}

int layout_widen(const void* src, int grad_dtype, int64_t count, double* dst, cudaStream_t st) {
  if (count == 0) return LF_OK;
  if (grad_dtype == LF_F64) {
    LF_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * count, cudaMemcpyDeviceToDevice, st));
    return LF_OK;
  }
  if (grad_dtype != LF_F32) return fail(LF_EINVAL, "layout: gradients are float or double");
  widen_f32<<<grid_for(count), 256, 0, st>>>(static_cast<const float*>(src), count, dst);
  LF_LAUNCHED();
  return LF_OK;
}

}  // namespace lf
