// lf_adam.cu — the optimizer step that consumes dE (and the encoder's
// gradients) on the device: AdamState::apply (proj/src/adam.cpp:22-36),
// element for element.  Parameters are float, moments and all update
// arithmetic double, each operation rounded once in the reference's order
// (no contraction: __dmul_rn / __dadd_rn / __ddiv_rn / __dsqrt_rn), so the
// parameters after any number of steps are bitwise those of the reference.
//
// HBM-bound elementwise pass: per element read param 4 B + grad 4|8 B + m, v
// 16 B, write param 4 B + m, v 16 B (+ an optional bf16 / fp32 shadow of the
// new parameter for the next step's CCE kernels, fused so it costs 2|4 B
// instead of another pass).  Grid-stride over SM-count multiples.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "lf_internal.cuh"
#include "lf_kernels.cuh"

namespace lf {
namespace {

template <class G, class S>
__device__ __forceinline__ void adam_one(float* __restrict__ param, double* __restrict__ m,
                                         double* __restrict__ v, int64_t i, float p0, double g,
                                         double m0, double v0, double b1, double b2, double c1,
                                         double c2, double lr, double eps, double corr1,
                                         double corr2, S* __restrict__ shadow) {
  // adam.cpp:28-33, left to right, one rounding per operation
  const double mi = __dadd_rn(__dmul_rn(b1, m0), __dmul_rn(c1, g));
  const double vi = __dadd_rn(__dmul_rn(b2, v0), __dmul_rn(__dmul_rn(c2, g), g));
  m[i] = mi;
  v[i] = vi;
  const double mhat = __ddiv_rn(mi, corr1);
  const double vhat = __ddiv_rn(vi, corr2);
  const double step = __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps));
  const float p = __double2float_rn(__dadd_rn(static_cast<double>(p0), -step));
  param[i] = p;
  if constexpr (sizeof(S) == 2) {
    shadow[i] = __float2bfloat16_rn(p);
  } else if constexpr (sizeof(S) == 4) {
    shadow[i] = p;
  }
}

// Each thread takes U elements one grid-stride apart and issues all their
// loads before any arithmetic (the pass is latency-bound on scalar loads
// otherwise).
template <class G, class S>
__global__ void __launch_bounds__(256) adam_apply(float* __restrict__ param, const G* __restrict__ grad,
                                                  double* __restrict__ m, double* __restrict__ v,
                                                  int64_t n, double b1, double b2, double lr, double eps,
                                                  double corr1, double corr2, S* __restrict__ shadow) {
  constexpr int U = 4;
  const double c1 = __dadd_rn(1.0, -b1), c2 = __dadd_rn(1.0, -b2);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    float p0[U];
    double g[U], m0[U], v0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        p0[u] = param[i];
        g[u] = static_cast<double>(grad[i]);
        m0[u] = m[i];
        v0[u] = v[i];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n)
        adam_one<G, S>(param, m, v, i, p0[u], g[u], m0[u], v0[u], b1, b2, c1, c2, lr, eps, corr1,
                       corr2, shadow);
    }
  }
}

struct NoShadow {
  char pad;
};

template <class G>
int launch(float* param, const void* grad, double* m, double* v, int64_t n, double b1, double b2,
           double lr, double eps, double corr1, double corr2, void* shadow, int shadow_dtype,
           cudaStream_t st) {
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(n, 256), 4LL * num_sms()));
  const G* g = static_cast<const G*>(grad);
  if (shadow && shadow_dtype == LF_BF16)
    adam_apply<G, __nv_bfloat16><<<grid, 256, 0, st>>>(param, g, m, v, n, b1, b2, lr, eps, corr1,
                                                       corr2, static_cast<__nv_bfloat16*>(shadow));
  else if (shadow && shadow_dtype == LF_F32)
    adam_apply<G, float><<<grid, 256, 0, st>>>(param, g, m, v, n, b1, b2, lr, eps, corr1, corr2,
                                               static_cast<float*>(shadow));
  else
    adam_apply<G, NoShadow><<<grid, 256, 0, st>>>(param, g, m, v, n, b1, b2, lr, eps, corr1, corr2,
                                                  nullptr);
  LF_LAUNCHED();
  return LF_OK;
}

}  // namespace

int adam_step(float* param, const void* grad, int grad_dtype, double* m, double* v, int64_t n,
              double lr, double b1, double b2, double eps, int64_t t, void* shadow, int shadow_dtype,
              cudaStream_t st) {
  // AdamState's checks (adam.cpp:8-19) with its messages
  if (b1 < 0.0 || b1 >= 1.0 || b2 < 0.0 || b2 >= 1.0)
    return fail(LF_EINVAL, "adam: betas must lie in [0, 1)");
  if (!(eps > 0.0)) return fail(LF_EINVAL, "adam: eps must be positive");
  if (t < 1) return fail(LF_EINVAL, "adam: step count t must be >= 1");
  if (n < 0) return fail(LF_EINVAL, "adam: negative element count");
  if (grad_dtype != LF_F32 && grad_dtype != LF_F64)
    return fail(LF_EINVAL, "adam: gradients must be f32 or f64");
  if (shadow && shadow_dtype != LF_BF16 && shadow_dtype != LF_F32)
    return fail(LF_EINVAL, "adam: shadow copy must be bf16 or f32");
  if (n == 0) return LF_OK;
  // adam.cpp:46-47, on the host exactly as the reference computes them
  const double corr1 = 1.0 - std::pow(b1, static_cast<double>(t));
  const double corr2 = 1.0 - std::pow(b2, static_cast<double>(t));
  return grad_dtype == LF_F64
             ? launch<double>(param, grad, m, v, n, b1, b2, lr, eps, corr1, corr2, shadow, shadow_dtype, st)
             : launch<float>(param, grad, m, v, n, b1, b2, lr, eps, corr1, corr2, shadow, shadow_dtype, st);
}

}  // namespace lf
