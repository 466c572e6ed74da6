// lf_ce.cu — the MATERIALISING cross-entropy baseline on the GPU: the
// reference's ce_full_forward / ce_full_backward (proj/src/losses.cpp:71-140),
// i.e. what CCE avoids.  The n x v logit matrix is written to HBM (fp32) by a
// cuBLAS GEMM (a plain library GEMM — this is the baseline, not the product),
// the softmax / log-sum-exp are row kernels over it, and the gradients are two
// more GEMMs over a materialised bf16 coefficient matrix G.  Used to reproduce
// the paper's CE-vs-CCE memory and time comparisons on B200;
// peak scratch is n * v * 6 bytes.  Also the sampled variant ce_sampled_forward /
// backward (losses.cpp:142-221): the n x (1+K) candidate logits written to HBM,
// G written over them, dE scattered with atomics.
#include <cublas_v2.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "lf_internal.cuh"
#include "lf_kernels.cuh"

namespace lf {
namespace {

cublasHandle_t handle_for_thread() {
  thread_local cublasHandle_t h = nullptr;
  if (!h && cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) h = nullptr;
  return h;
}

int blas_fail(cublasStatus_t s, const char* what) {
  return fail(LF_ECUDA, std::string("cuBLAS ") + what + " failed: status " + std::to_string(s));
}

cudaDataType_t blas_type(int dtype) {
  return dtype == LF_BF16 ? CUDA_R_16BF : (dtype == LF_F32 ? CUDA_R_32F : CUDA_R_64F);
}

// logits[n x v] (row-major, fp32 or fp64) = X[n x d] . E[v x d]^T.  Column-major
// view: logits^T (v x n) = E (d x v)^T . X (d x n).
template <class T>
int logits_gemm(cublasHandle_t h, int dtype, const void* X, const void* E, int64_t n, int d,
                int64_t v, T* logits) {
  const T one = 1, zero = 0;
  const cudaDataType_t ct = sizeof(T) == 8 ? CUDA_R_64F : CUDA_R_32F;
  const cublasComputeType_t comp = sizeof(T) == 8 ? CUBLAS_COMPUTE_64F : CUBLAS_COMPUTE_32F;
  cublasStatus_t s = cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(v),
                                  static_cast<int>(n), d, &one, E, blas_type(dtype), d, X,
                                  blas_type(dtype), d, &zero, logits, ct, static_cast<int>(v), comp,
                                  CUBLAS_GEMM_DEFAULT);
  return s == CUBLAS_STATUS_SUCCESS ? LF_OK : blas_fail(s, "logits GEMM");
}

// Block per row: numerically stable log-sum-exp over v logits (two passes
// over the row, which sits in L2) in the logits' own precision (fp32 for the
// bf16/f32 baseline, as a framework CE would), and the target logit gather.
template <class T>
__global__ void __launch_bounds__(256) row_lse_pos(const T* __restrict__ logits, int64_t v,
                                                   const int64_t* __restrict__ targets,
                                                   double* __restrict__ lse, double* __restrict__ pos) {
  __shared__ T red[8];
  const int64_t row = blockIdx.x;
  const T* l = logits + row * v;
  T mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < v; j += blockDim.x) mx = max(mx, l[j]);
  for (int off = 16; off > 0; off >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int i = 1; i < 8; ++i) mx = max(mx, red[i]);
  __syncthreads();
  T s = 0;
  for (int64_t j = threadIdx.x; j < v; j += blockDim.x) s += exp(l[j] - mx);
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += static_cast<double>(red[i]);
    lse[row] = static_cast<double>(mx) + log(t);
    pos[row] = static_cast<double>(l[targets[row]]);
  }
}

// G[i][j] = (exp(logit - lse_i) - [j == x_i]) * scale (losses.cpp:117-121),
// stored in the gradient GEMMs' input type.
template <class T, class TG>
__global__ void softmax_grad(const T* __restrict__ logits, int64_t n, int64_t v,
                             const int64_t* __restrict__ targets, const double* __restrict__ lse,
                             double scale, TG* __restrict__ g) {
  const int64_t total = n * v;
  const T sc = static_cast<T>(scale);
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = k / v, j = k - i * v;
    T x = exp(logits[k] - static_cast<T>(lse[i]));
    if (j == targets[i]) x -= T(1);
    g[k] = static_cast<TG>(x * sc);
  }
}

int grid_for(int64_t count) { return static_cast<int>(std::min<int64_t>(ceil_div(count, 256), 148 * 32)); }

// ---- materialising sampled CE (losses.cpp:142-221) ----
template <class TI>
__device__ __forceinline__ double to_d(TI x) { return static_cast<double>(x); }
template <>
__device__ __forceinline__ double to_d<__nv_bfloat16>(__nv_bfloat16 x) { return static_cast<double>(__bfloat162float(x)); }

// Warp per row: the n x w candidate logits are WRITTEN (this is the baseline).
template <class TI, class T>
__global__ void __launch_bounds__(256) cem_logits(const TI* __restrict__ X, const TI* __restrict__ E,
                                                 const int64_t* __restrict__ inds, int64_t n, int D,
                                                 int64_t w, T* __restrict__ logits) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  for (int64_t s = lane; s < w; s += 32) {
    const TI* er = E + inds[row * w + s] * D;
    const TI* xr = X + row * D;
    T acc = 0;
    for (int k = 0; k < D; ++k) acc += static_cast<T>(to_d(xr[k])) * static_cast<T>(to_d(er[k]));
    logits[row * w + s] = acc;
  }
}

// Warp per row: lse, pos (slot 0); optionally G = (softmax - [s == 0]) * scale
// written back over the logits.
template <class T>
__global__ void __launch_bounds__(256) cem_rows(T* __restrict__ logits, int64_t n, int64_t w,
                                               double* __restrict__ lse, double* __restrict__ pos,
                                               double scale, bool grad) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  T* o = logits + row * w;
  T mx = -INFINITY;
  for (int64_t s = lane; s < w; s += 32) mx = max(mx, o[s]);
  for (int off = 16; off > 0; off >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  double sum = 0.0;
  for (int64_t s = lane; s < w; s += 32) sum += exp(static_cast<double>(o[s] - mx));
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  const double l = static_cast<double>(mx) + log(sum);
  if (!grad) {
    if (lane == 0) {
      lse[row] = l;
      pos[row] = static_cast<double>(o[0]);
    }
    return;
  }
  for (int64_t s = lane; s < w; s += 32) {
    const double g = exp(static_cast<double>(o[s]) - l) * scale;
    o[s] = static_cast<T>(s == 0 ? g - scale : g);
  }
}

// dX row = sum_s G[s] E[inds[s]] (warp per row, lanes over k); dE scattered
// with atomics (duplicates accumulate, losses.cpp:211-218).
template <class TI, class T>
__global__ void __launch_bounds__(256) cem_grads(const TI* __restrict__ X, const TI* __restrict__ E,
                                                const int64_t* __restrict__ inds, const T* __restrict__ G,
                                                int64_t n, int D, int64_t w, T* __restrict__ dX,
                                                T* __restrict__ dE) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  for (int k = lane; k < D; k += 32) {
    T acc = 0;
    const T xk = static_cast<T>(to_d(X[row * D + k]));
    for (int64_t s = 0; s < w; ++s) {
      const int64_t item = inds[row * w + s];
      const T g = G[row * w + s];
      acc += g * static_cast<T>(to_d(E[item * D + k]));
      atomicAdd(dE + item * D + k, g * xk);
    }
    dX[row * D + k] = acc;
  }
}

}  // namespace

int cem_forward(int dtype, const void* X, const void* E, const int64_t* inds, int64_t n, int D, int64_t w,
                double* lse, double* pos, double* loss, cudaStream_t st) {
  const bool f64 = dtype == LF_F64;
  Scratch logits;
  int rc = logits.alloc((f64 ? 8 : 4) * n * w, st);
  if (rc) return rc;
  const unsigned blocks = static_cast<unsigned>(ceil_div(n, 8));
  if (f64) {
    cem_logits<double, double><<<blocks, 256, 0, st>>>(static_cast<const double*>(X), static_cast<const double*>(E),
                                                      inds, n, D, w, logits.as<double>());
    cem_rows<double><<<blocks, 256, 0, st>>>(logits.as<double>(), n, w, lse, pos, 0.0, false);
  } else if (dtype == LF_F32) {
    cem_logits<float, float><<<blocks, 256, 0, st>>>(static_cast<const float*>(X), static_cast<const float*>(E),
                                                    inds, n, D, w, logits.as<float>());
    cem_rows<float><<<blocks, 256, 0, st>>>(logits.as<float>(), n, w, lse, pos, 0.0, false);
  } else {
    cem_logits<__nv_bfloat16, float><<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(X),
                                                            static_cast<const __nv_bfloat16*>(E), inds, n, D,
                                                            w, logits.as<float>());
    cem_rows<float><<<blocks, 256, 0, st>>>(logits.as<float>(), n, w, lse, pos, 0.0, false);
  }
  LF_LAUNCHED();
  return launch_mean_loss(lse, pos, n, loss, st);
}

int cem_backward(int dtype, const void* X, const void* E, const int64_t* inds, double upstream, int64_t n,
                 int D, int64_t v, int64_t w, void* dX, void* dE, cudaStream_t st) {
  const bool f64 = dtype == LF_F64;
  Scratch logits;
  int rc = logits.alloc((f64 ? 8 : 4) * n * w, st);
  if (rc) return rc;
  LF_CUDA(cudaMemsetAsync(dE, 0, (f64 ? 8 : 4) * v * D, st));
  const double scale = upstream / static_cast<double>(n);
  const unsigned blocks = static_cast<unsigned>(ceil_div(n, 8));
  if (f64) {
    cem_logits<double, double><<<blocks, 256, 0, st>>>(static_cast<const double*>(X), static_cast<const double*>(E),
                                                      inds, n, D, w, logits.as<double>());
    cem_rows<double><<<blocks, 256, 0, st>>>(logits.as<double>(), n, w, nullptr, nullptr, scale, true);
    cem_grads<double, double><<<blocks, 256, 0, st>>>(static_cast<const double*>(X), static_cast<const double*>(E),
                                                     inds, logits.as<double>(), n, D, w,
                                                     static_cast<double*>(dX), static_cast<double*>(dE));
  } else if (dtype == LF_F32) {
    cem_logits<float, float><<<blocks, 256, 0, st>>>(static_cast<const float*>(X), static_cast<const float*>(E),
                                                    inds, n, D, w, logits.as<float>());
    cem_rows<float><<<blocks, 256, 0, st>>>(logits.as<float>(), n, w, nullptr, nullptr, scale, true);
    cem_grads<float, float><<<blocks, 256, 0, st>>>(static_cast<const float*>(X), static_cast<const float*>(E), inds,
                                                   logits.as<float>(), n, D, w, static_cast<float*>(dX),
                                                   static_cast<float*>(dE));
  } else {
    cem_logits<__nv_bfloat16, float><<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(X),
                                                            static_cast<const __nv_bfloat16*>(E), inds, n, D,
                                                            w, logits.as<float>());
    cem_rows<float><<<blocks, 256, 0, st>>>(logits.as<float>(), n, w, nullptr, nullptr, scale, true);
    cem_grads<__nv_bfloat16, float><<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(X),
                                                           static_cast<const __nv_bfloat16*>(E), inds,
                                                           logits.as<float>(), n, D, w, static_cast<float*>(dX),
                                                           static_cast<float*>(dE));
  }
  LF_LAUNCHED();
  return LF_OK;
}

int ce_forward(int dtype, const void* X, const void* E, const int64_t* targets, int64_t n, int D,
               int64_t v, double* lse, double* pos, double* loss, cudaStream_t st) {
  cublasHandle_t h = handle_for_thread();
  if (!h) return fail(LF_ECUDA, "cublasCreate failed");
  cublasSetStream(h, st);
  Scratch logits;
  const size_t eb = dtype == LF_F64 ? 8 : 4;
  int rc = logits.alloc(eb * n * v, st);
  if (rc) return rc;
  if (dtype == LF_F64) {
    rc = logits_gemm<double>(h, dtype, X, E, n, D, v, logits.as<double>());
    if (!rc) row_lse_pos<double><<<static_cast<unsigned>(n), 256, 0, st>>>(logits.as<double>(), v,
                                                                          targets, lse, pos);
  } else {
    rc = logits_gemm<float>(h, dtype, X, E, n, D, v, logits.as<float>());
    if (!rc) row_lse_pos<float><<<static_cast<unsigned>(n), 256, 0, st>>>(logits.as<float>(), v,
                                                                         targets, lse, pos);
  }
  if (rc) return rc;
  LF_LAUNCHED();
  return launch_mean_loss(lse, pos, n, loss, st);
}

int ce_backward(int dtype, const void* X, const void* E, const int64_t* targets, double upstream,
                int64_t n, int D, int64_t v, void* dX, void* dE, cudaStream_t st) {
  cublasHandle_t h = handle_for_thread();
  if (!h) return fail(LF_ECUDA, "cublasCreate failed");
  cublasSetStream(h, st);
  const bool f64 = dtype == LF_F64;
  Scratch logits, g, lse, pos;
  int rc = logits.alloc((f64 ? 8 : 4) * n * v, st);
  // G in the GEMM input type: bf16 for bf16 inputs (fp32 accumulate), else the input type
  const size_t gb = dtype == LF_BF16 ? 2 : (f64 ? 8 : 4);
  if (!rc) rc = g.alloc(gb * n * v, st);
  if (!rc) rc = lse.alloc(sizeof(double) * n, st);
  if (!rc) rc = pos.alloc(sizeof(double) * n, st);
  if (rc) return rc;
  const double scale = upstream / static_cast<double>(n);  // losses.cpp:114
  if (f64) {
    rc = logits_gemm<double>(h, dtype, X, E, n, D, v, logits.as<double>());
    if (rc) return rc;
    row_lse_pos<double><<<static_cast<unsigned>(n), 256, 0, st>>>(logits.as<double>(), v, targets,
                                                                 lse.as<double>(), pos.as<double>());
    softmax_grad<double, double><<<grid_for(n * v), 256, 0, st>>>(
        logits.as<double>(), n, v, targets, lse.as<double>(), scale, g.as<double>());
  } else {
    rc = logits_gemm<float>(h, dtype, X, E, n, D, v, logits.as<float>());
    if (rc) return rc;
    row_lse_pos<float><<<static_cast<unsigned>(n), 256, 0, st>>>(logits.as<float>(), v, targets,
                                                                lse.as<double>(), pos.as<double>());
    if (dtype == LF_BF16)
      softmax_grad<float, __nv_bfloat16><<<grid_for(n * v), 256, 0, st>>>(
          logits.as<float>(), n, v, targets, lse.as<double>(), scale, g.as<__nv_bfloat16>());
    else
      softmax_grad<float, float><<<grid_for(n * v), 256, 0, st>>>(
          logits.as<float>(), n, v, targets, lse.as<double>(), scale, g.as<float>());
  }
  LF_LAUNCHED();
  // dX (n x d) = G . E; column-major: dX^T (d x n) = E^T-view (d x v) . G^T-view (v x n)
  // dE (v x d) = G^T . X; column-major: dE^T (d x v) = X^T-view (d x n) . G-view (n x v)^T
  const cudaDataType_t gt = dtype == LF_BF16 ? CUDA_R_16BF : (f64 ? CUDA_R_64F : CUDA_R_32F);
  const cudaDataType_t ot = f64 ? CUDA_R_64F : CUDA_R_32F;
  const cublasComputeType_t comp = f64 ? CUBLAS_COMPUTE_64F : CUBLAS_COMPUTE_32F;
  const double one64 = 1.0, zero64 = 0.0;
  const float one32 = 1.f, zero32 = 0.f;
  const void* one = f64 ? static_cast<const void*>(&one64) : static_cast<const void*>(&one32);
  const void* zero = f64 ? static_cast<const void*>(&zero64) : static_cast<const void*>(&zero32);
  cublasStatus_t s = cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, D, static_cast<int>(n),
                                  static_cast<int>(v), one, E, blas_type(dtype), D, g.ptr, gt,
                                  static_cast<int>(v), zero, dX, ot, D, comp, CUBLAS_GEMM_DEFAULT);
  if (s != CUBLAS_STATUS_SUCCESS) return blas_fail(s, "dX GEMM");
  s = cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_T, D, static_cast<int>(v), static_cast<int>(n), one,
                   X, blas_type(dtype), D, g.ptr, gt, static_cast<int>(v), zero, dE, ot, D, comp,
                   CUBLAS_GEMM_DEFAULT);
  if (s != CUBLAS_STATUS_SUCCESS) return blas_fail(s, "dE GEMM");
  return LF_OK;
}

}  // namespace lf
