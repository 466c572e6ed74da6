// lf_simt.cu — CUDA-core (SIMT) CCE kernels for the fp32 and fp64 "exact"
// element types, plus the partial-combine and dX-reduce kernels shared with
// the tensor-core path.
//
// Semantics follow the reference exactly (proj/src/cce.cpp):
//   logit  o_ij = sum_k X_ik * E_jk, k ascending                (cce.cpp:40-55)
//   lse_i  = log sum_j exp(o_ij); pos_i = o_{i, x_i} taken from the SAME
//            tile value that feeds the LSE                       (cce.cpp:111-131)
//   g_ij   = s*scale, (s-1)*scale at the target, 0 (and counted) for
//            off-target s < eps                                  (cce.cpp:189-204)
//   dX = G E (row-owned), dE = G^T X (item-owned): two recompute passes with
//            single ownership and NO atomics on the gradients    (cce.cpp:206-262)
// In exact mode (T = double) every product/sum is __dmul_rn/__dadd_rn in the
// reference's order, so pos is bitwise equal to the CPU's double result.
#include <cfloat>
#include <cmath>

#include "lf_internal.cuh"
#include "lf_kernels.cuh"

namespace lf {

namespace {

constexpr int kThreads = 256;
#ifndef LF_SIMT_KUNROLL
#define LF_SIMT_KUNROLL 4  // logit tiles: k steps unrolled (shared-memory reads issued ahead of the FMAs)
#endif
constexpr int kKUnroll = LF_SIMT_KUNROLL;

template <class T>
__device__ __forceinline__ T mul_rn(T a, T b) { return a * b; }
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <class T>
__device__ __forceinline__ T add_rn(T a, T b) { return a + b; }
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <class T>
__device__ __forceinline__ T fma_acc(T acc, T a, T b) { return fmaf(a, b, acc); }
template <>
__device__ __forceinline__ double fma_acc<double>(double acc, double a, double b) {
  return __dadd_rn(acc, __dmul_rn(a, b));  // reference order: acc += a*b, no contraction
}
template <class T>
__device__ __forceinline__ T t_exp(T x) { return expf(x); }
template <>
__device__ __forceinline__ double t_exp<double>(double x) { return exp(x); }
template <class T>
__device__ __forceinline__ T t_log(T x) { return logf(x); }
template <>
__device__ __forceinline__ double t_log<double>(double x) { return log(x); }
template <class T>
__device__ __forceinline__ T neg_inf() { return -INFINITY; }

// Stage rows [r0, r0+R) of a row-major [rows x D] matrix into smem laid out
// [D][R+PAD] (transposed, padded); rows past `rows` are zero.  PAD = 1: one
// element per thread, k fastest (conflict-free stores).  PAD = 4 (fp32 tile
// rows 16-byte aligned for vector reads): 16-byte global loads along k with
// the row fastest, so a warp's four stores per load hit 32 distinct banks.
template <class T, int R, int PAD = 1>
__device__ __forceinline__ void stage_T(T* s, const T* __restrict__ g, int64_t r0, int64_t rows,
                                        int D) {
  constexpr int LD = R + PAD;
  if constexpr (PAD == 4 && sizeof(T) == 4) {
    if ((D & 3) == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
      const int nk4 = D / 4;
      for (int idx = threadIdx.x; idx < R * nk4; idx += kThreads) {
        const int r = idx % R, kq = idx / R;
        const int64_t row = r0 + r;
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < rows) q = *reinterpret_cast<const float4*>(g + row * D + 4 * kq);
        T* c = s + 4 * kq * LD + r;
        c[0] = q.x;
        c[LD] = q.y;
        c[2 * LD] = q.z;
        c[3 * LD] = q.w;
      }
      return;
    }
  }
  for (int idx = threadIdx.x; idx < R * D; idx += kThreads) {
    const int r = idx / D, k = idx % D;
    const int64_t row = r0 + r;
    s[k * LD + r] = row < rows ? g[row * D + k] : T(0);
  }
}

// R x C logit tile from staged Xs [D][R+PAD] and Es [D][C+PAD]; each of the
// 256 threads owns RPT rows x CPT columns.  PAD = 1: columns CG apart
// (scalar reads); PAD = 4 (RPT = CPT = 4): four consecutive rows and columns,
// one 16-byte read of each per k.  Exact mode: k ascending either way.
// Four consecutive smem values (16-byte aligned): one LDS.128 for float.
template <class T>
__device__ __forceinline__ void ld4(const T* p, T (&v)[4]) {
#pragma unroll
  for (int r = 0; r < 4; ++r) v[r] = p[r];
}
template <>
__device__ __forceinline__ void ld4<float>(const float* p, float (&v)[4]) {
  const float4 q = *reinterpret_cast<const float4*>(p);
  v[0] = q.x;
  v[1] = q.y;
  v[2] = q.z;
  v[3] = q.w;
}
// Gradient-tile stride (4 owners of one stream element contiguous, rows
// 16-byte aligned) and the tile's offset, rounded up to 16 bytes.
constexpr int gstride(int owners) { return owners + 4; }
template <class T>
__device__ __host__ constexpr size_t align16(size_t elems) {
  return (elems * sizeof(T) + 15) / 16 * 16 / sizeof(T);
}

template <class T, int R, int C, int RPT_ = 2, int CPT_ = 4, int PAD = 1>
struct TileMap {
  static constexpr int RPT = RPT_;
  static constexpr int CPT = CPT_;
  static constexpr int CG = C / CPT;
  static constexpr bool kVec = PAD == 4 && RPT == 4 && CPT == 4;
  static_assert((R / RPT) * CG == kThreads, "tile map must cover 256 threads");
  __device__ static int row(int i) { return (threadIdx.x / CG) * RPT + i; }
  __device__ static int col(int q) { return kVec ? (threadIdx.x % CG) * CPT + q : (threadIdx.x % CG) + CG * q; }
  __device__ static void logits(const T* Xs, const T* Es, int D, T (&o)[RPT][CPT]) {
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
      for (int q = 0; q < CPT; ++q) o[i][q] = T(0);
#pragma unroll kKUnroll
    for (int k = 0; k < D; ++k) {
      T xv[RPT], ev[CPT];
      if constexpr (kVec) {
        ld4(Xs + k * (R + PAD) + row(0), xv);
        ld4(Es + k * (C + PAD) + col(0), ev);
      } else {
#pragma unroll
        for (int i = 0; i < RPT; ++i) xv[i] = Xs[k * (R + PAD) + row(i)];
#pragma unroll
        for (int q = 0; q < CPT; ++q) ev[q] = Es[k * (C + PAD) + col(q)];
      }
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int q = 0; q < CPT; ++q) o[i][q] = fma_acc(o[i][q], xv[i], ev[q]);
    }
  }
};

// Tile geometry per element type.  fp64 (exact mode) keeps 32 x 64 tiles
// (D = 256 must fit in shared memory); fp32 uses 4 x 4 register tiles with
// 16-byte operand reads on twice the tile area.
template <class T>
struct Lay {
  static constexpr int RPT = 2, CPT = 4, PAD = 1;
  static constexpr int FR = 32, FC = 64;  // forward: rows x columns per tile
  static constexpr int XR = 32, XC = 64;  // dX pass
  static constexpr int ER = 64, EC = 32;  // dE pass (rows per step x items per block)
};
template <>
struct Lay<float> {
  static constexpr int RPT = 4, CPT = 4, PAD = 4;
  static constexpr int FR = 32, FC = 128;
  static constexpr int XR = 32, XC = 128;
  static constexpr int ER = 128, EC = 32;
};
template <class T, int R, int C>
using LayMap = TileMap<T, R, C, Lay<T>::RPT, Lay<T>::CPT, Lay<T>::PAD>;

// Online LSE update, numeric.hpp:19-27 (branch structure kept).
template <class T>
__device__ __forceinline__ void lse_update(T& m, T& s, T o) {
  if (o <= m) {
    s += t_exp(o - m);
  } else {
    s = s * t_exp(m - o) + T(1);
    m = o;
  }
}
template <class T>
__device__ __forceinline__ void lse_merge(T& m, T& s, T m2, T s2) {
  if (m2 == neg_inf<T>()) return;
  if (m == neg_inf<T>()) { m = m2; s = s2; return; }
  const T M = m > m2 ? m : m2;
  s = s * t_exp(m - M) + s2 * t_exp(m2 - M);
  m = M;
}

// ---------------------------------------------------------------------------
// Forward: block = 32 rows x one V chunk; writes Partial<T> per (chunk, row).
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kThreads) cce_simt_fwd(const T* __restrict__ X,
                                                         const T* __restrict__ E,
                                                         const int64_t* __restrict__ targets,
                                                         int64_t n, int D, int64_t v,
                                                         int64_t v_offset, int64_t chunk,
                                                         Partial<T>* __restrict__ part) {
  constexpr int R = Lay<T>::FR, C = Lay<T>::FC, PAD = Lay<T>::PAD;
  using M = LayMap<T, R, C>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Xs = reinterpret_cast<T*>(smem_raw);
  T* Es = Xs + D * (R + PAD);
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * R;
  const int64_t c_begin = static_cast<int64_t>(blockIdx.y) * chunk;
  const int64_t c_end = min(v, c_begin + chunk);
  stage_T<T, R, PAD>(Xs, X, r0, n, D);

  T m[M::RPT], s[M::RPT], t[M::RPT], has[M::RPT];
  int64_t tgt[M::RPT];
#pragma unroll
  for (int i = 0; i < M::RPT; ++i) {
    m[i] = neg_inf<T>();
    s[i] = T(0);
    t[i] = T(0);
    has[i] = T(0);
    const int64_t row = r0 + M::row(i);
    tgt[i] = row < n ? targets[row] - v_offset : -1;
  }
  for (int64_t c0 = c_begin; c0 < c_end; c0 += C) {
    __syncthreads();
    stage_T<T, C, PAD>(Es, E, c0, c_end, D);
    __syncthreads();
    T o[M::RPT][M::CPT];
    M::logits(Xs, Es, D, o);
#pragma unroll
    for (int i = 0; i < M::RPT; ++i)
#pragma unroll
      for (int q = 0; q < M::CPT; ++q) {
        const int64_t col = c0 + M::col(q);
        if (col < c_end) {
          lse_update(m[i], s[i], o[i][q]);
          if (col == tgt[i]) { t[i] = o[i][q]; has[i] = T(1); }
        }
      }
  }
  // Merge the CG threads that share each row (consecutive lanes).
#pragma unroll
  for (int i = 0; i < M::RPT; ++i) {
    for (int off = M::CG / 2; off > 0; off >>= 1) {
      const T m2 = __shfl_xor_sync(0xffffffffu, m[i], off);
      const T s2 = __shfl_xor_sync(0xffffffffu, s[i], off);
      const T t2 = __shfl_xor_sync(0xffffffffu, t[i], off);
      const T h2 = __shfl_xor_sync(0xffffffffu, has[i], off);
      lse_merge(m[i], s[i], m2, s2);
      if (h2 != T(0)) { t[i] = t2; has[i] = T(1); }
    }
    const int64_t row = r0 + M::row(i);
    if ((threadIdx.x % M::CG) == 0 && row < n) {
      Partial<T> p;
      p.m = m[i];
      p.s = s[i];
      p.t = t[i];
      p.has = has[i];
      part[static_cast<int64_t>(blockIdx.y) * n + row] = p;
    }
  }
}

// Coefficient of one element (cce.cpp:189-204).
template <class T>
__device__ __forceinline__ T coeff(T o, T row_lse, bool is_target, T eps, T scale,
                                   unsigned& skips) {
  const T s = t_exp(o - row_lse);
  if (is_target) return (s - T(1)) * scale;
  if (eps > T(0) && s < eps) {
    ++skips;
    return T(0);
  }
  return s * scale;
}

// ---------------------------------------------------------------------------
// Backward dX: block = 32 rows x one V chunk; dX partial per chunk.  NQ =
// ceil(D / 32): the dims each thread accumulates (register arrays sized to D).
// ---------------------------------------------------------------------------
template <class T, int NQ>
__global__ void __launch_bounds__(kThreads, NQ <= 2 ? 3 : 1) cce_simt_bwd_dx(
    const T* __restrict__ X, const T* __restrict__ E, const int64_t* __restrict__ targets,
    const double* __restrict__ lse, int64_t n, int D, int64_t v, int64_t v_offset, int64_t chunk,
    T scale, T eps, T* __restrict__ dx_part, unsigned long long* __restrict__ skip_counter) {
  constexpr int R = Lay<T>::XR, C = Lay<T>::XC, PAD = Lay<T>::PAD;
  using M = LayMap<T, R, C>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int GS = gstride(R);
  T* Xs = reinterpret_cast<T*>(smem_raw);
  T* Es = Xs + D * (R + PAD);
  T* Gs = Xs + align16<T>(static_cast<size_t>(D) * (R + PAD + C + PAD));  // [C][GS]: column-major G
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * R;
  const int64_t c_begin = static_cast<int64_t>(blockIdx.y) * chunk;
  const int64_t c_end = min(v, c_begin + chunk);
  stage_T<T, R, PAD>(Xs, X, r0, n, D);

  T row_lse[M::RPT];
  int64_t tgt[M::RPT];
#pragma unroll
  for (int i = 0; i < M::RPT; ++i) {
    const int64_t row = r0 + M::row(i);
    row_lse[i] = row < n ? static_cast<T>(lse[row]) : T(0);
    tgt[i] = row < n ? targets[row] - v_offset : -1;
  }
  // dX accumulators: rows 4 (tid / 32) + r (the warp's four rows, one
  // 16-byte G load per column), dims (tid % 32) + 32 q (conflict-free E
  // reads): 4 + nq smem loads per 4 nq FMAs.
  const int arow = (threadIdx.x / 32) * 4, adim = threadIdx.x % 32;
  const int nq = (D - adim + 31) / 32;
  T acc[4][NQ];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[r][q] = T(0);
  unsigned skips = 0;

  for (int64_t c0 = c_begin; c0 < c_end; c0 += C) {
    __syncthreads();
    stage_T<T, C, PAD>(Es, E, c0, c_end, D);
    __syncthreads();
    T o[M::RPT][M::CPT];
    M::logits(Xs, Es, D, o);
    T gt[M::RPT][M::CPT];
#pragma unroll
    for (int i = 0; i < M::RPT; ++i)
#pragma unroll
      for (int q = 0; q < M::CPT; ++q) {
        const int64_t col = c0 + M::col(q);
        const bool valid = col < c_end && (r0 + M::row(i)) < n;
        gt[i][q] = valid ? coeff(o[i][q], row_lse[i], col == tgt[i], eps, scale, skips) : T(0);
      }
#pragma unroll
    for (int q = 0; q < M::CPT; ++q) {
      if constexpr (M::kVec) {  // the thread's four rows of column q: one 16-byte store
        *reinterpret_cast<float4*>(Gs + M::col(q) * GS + M::row(0)) =
            make_float4(gt[0][q], gt[1][q], gt[2][q], gt[3][q]);
      } else {
#pragma unroll
        for (int i = 0; i < M::RPT; ++i) Gs[M::col(q) * GS + M::row(i)] = gt[i][q];
      }
    }
    __syncthreads();
    const int cn = static_cast<int>((c_end - c0 < C ? c_end - c0 : C));
    if constexpr (PAD == 4) {
      // four columns per step (16-byte E reads along the column; a column
      // past cn has G = 0 and a zero-staged E row, adding exact zeros)
      for (int j = 0; j < cn; j += 4) {
        T gv[4][4], ev[NQ][4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) ld4(Gs + (j + jj) * GS + arow, gv[jj]);
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (q < nq) ld4(Es + (adim + 32 * q) * (C + PAD) + j, ev[q]);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            if (q < nq) {
#pragma unroll
              for (int r = 0; r < 4; ++r) acc[r][q] = fma_acc(acc[r][q], gv[jj][r], ev[q][jj]);
            }
      }
    } else {
      for (int j = 0; j < cn; ++j) {
        T gv[4];
        ld4(Gs + j * GS + arow, gv);
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (q < nq) {
            const T ev = Es[(adim + 32 * q) * (C + PAD) + j];
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[r][q] = fma_acc(acc[r][q], gv[r], ev);
          }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t row = r0 + arow + r;
    if (row < n) {
      T* out = dx_part + static_cast<int64_t>(blockIdx.y) * n * D + row * D;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < nq) out[adim + 32 * q] = acc[r][q];
    }
  }
  if (skip_counter) {
    for (int off = 16; off > 0; off >>= 1) skips += __shfl_xor_sync(0xffffffffu, skips, off);
    if ((threadIdx.x & 31) == 0 && skips) atomicAdd(skip_counter, static_cast<unsigned long long>(skips));
  }
}

// ---------------------------------------------------------------------------
// Backward dE: block = 32 items, loops over all rows (ascending row tiles).
// ---------------------------------------------------------------------------
template <class T, int NQ>
__global__ void __launch_bounds__(kThreads) cce_simt_bwd_de(
    const T* __restrict__ X, const T* __restrict__ E, const int64_t* __restrict__ targets,
    const double* __restrict__ lse, int64_t n, int D, int64_t v, int64_t v_offset, T scale,
    T eps, T* __restrict__ dE, int64_t rows_per, const double* __restrict__ omp = nullptr) {
  // rows_per: the rows this block's y-slice sums (gridDim.y > 1: a partial
  // dE per slice at dE + y v D, reduced afterwards; fp32 only)
  // omp (optional, the fused fp32 forward's): 1 - p_t per row in full
  // precision, so a target entry is -(1 - p_t) scale even where exp(o - lse)
  // rounds to 1 (well-fit rows)
  constexpr int R = Lay<T>::ER, C = Lay<T>::EC, PAD = Lay<T>::PAD;
  using M = LayMap<T, R, C>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int GS = gstride(C);
  T* Es = reinterpret_cast<T*>(smem_raw);
  T* Xs = Es + D * (C + PAD);
  T* Gs = Es + align16<T>(static_cast<size_t>(D) * (C + PAD + R + PAD));  // [R][GS]
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * C;
  stage_T<T, C, PAD>(Es, E, c0, v, D);
  // dE accumulators: items 4 (tid / 32) + r (one 16-byte G load per row),
  // dims (tid % 32) + 32 q (conflict-free X reads).
  const int aitem = (threadIdx.x / 32) * 4, adim = threadIdx.x % 32;
  const int nq = (D - adim + 31) / 32;
  T acc[4][NQ];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[r][q] = T(0);
  unsigned skips = 0;

  const int64_t r_begin = static_cast<int64_t>(blockIdx.y) * rows_per;
  const int64_t r_end = min(n, r_begin + rows_per);
  dE += static_cast<int64_t>(blockIdx.y) * v * D;
  for (int64_t r0 = r_begin; r0 < r_end; r0 += R) {
    __syncthreads();
    stage_T<T, R, PAD>(Xs, X, r0, r_end, D);
    __syncthreads();
    T o[M::RPT][M::CPT];
    M::logits(Xs, Es, D, o);
#pragma unroll
    for (int i = 0; i < M::RPT; ++i) {
      const int64_t row = r0 + M::row(i);
      const bool rvalid = row < r_end;
      const T rl = rvalid ? static_cast<T>(lse[row]) : T(0);
      const int64_t tg = rvalid ? targets[row] - v_offset : -1;
      T gt[M::CPT];
#pragma unroll
      for (int q = 0; q < M::CPT; ++q) {
        const int64_t col = c0 + M::col(q);
        gt[q] = rvalid && col < v ? coeff(o[i][q], rl, col == tg, eps, scale, skips) : T(0);
        if (omp && rvalid && col == tg) gt[q] = static_cast<T>(-omp[row] * static_cast<double>(scale));
      }
      if constexpr (M::kVec) {  // four consecutive items of row i: one 16-byte store
        *reinterpret_cast<float4*>(Gs + M::row(i) * GS + M::col(0)) = make_float4(gt[0], gt[1], gt[2], gt[3]);
      } else {
#pragma unroll
        for (int q = 0; q < M::CPT; ++q) Gs[M::row(i) * GS + M::col(q)] = gt[q];
      }
    }
    __syncthreads();
    const int rn = static_cast<int>((r_end - r0 < R ? r_end - r0 : R));
    if constexpr (PAD == 4) {
      // four rows per step (16-byte X reads; a row past rn has G = 0 and a
      // zero-staged X row, adding exact zeros)
      for (int i = 0; i < rn; i += 4) {
        T gv[4][4], xv[NQ][4];
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) ld4(Gs + (i + ii) * GS + aitem, gv[ii]);
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (q < nq) ld4(Xs + (adim + 32 * q) * (R + PAD) + i, xv[q]);
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            if (q < nq) {
#pragma unroll
              for (int r = 0; r < 4; ++r) acc[r][q] = fma_acc(acc[r][q], gv[ii][r], xv[q][ii]);
            }
      }
    } else {
      for (int i = 0; i < rn; ++i) {
        T gv[4];
        ld4(Gs + i * GS + aitem, gv);
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (q < nq) {
            const T xv = Xs[(adim + 32 * q) * (R + PAD) + i];
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[r][q] = fma_acc(acc[r][q], gv[r], xv);
          }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t item = c0 + aitem + r;
    if (item < v) {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < nq) dE[item * D + adim + 32 * q] = acc[r][q];
    }
  }
}


// ---------------------------------------------------------------------------
// Fused forward + dX, fp32 (lf_cce_forward_backward with the filter off): one
// pass over the logits instead of the forward and the dX recompute.  Block =
// 32 rows x one V chunk on the fp32 4 x 4 tile map, so warp w owns rows
// 4w..4w+3 of every tile — in the logits and in the dX accumulation alike —
// and keeps their running max warp-uniform: per tile, P = exp(o - M) (the
// target entry left out, as in the tensor-core read-out form), the row sums
// and the O accumulator (O_i = sum_j P_ij E_j) are rescaled by exp(M_old -
// M_new).  Output per (chunk, row): Partial {M, S, t, has} + the O row; the
// combine below normalises dX = scale (sum_p O_p e^(M_p - lse) - (1 - p_t) E_t).
// ---------------------------------------------------------------------------
// D <= 64: three resident blocks per SM (80 registers, a few bytes spilled)
// measured 6 % faster at cfg1 than two at 128 registers
template <int NQ>
__global__ void __launch_bounds__(kThreads, NQ <= 2 ? 3 : 1) cce_simt_fwdx(const float* __restrict__ X,
                                                          const float* __restrict__ E,
                                                          const int64_t* __restrict__ targets,
                                                          int64_t n, int D, int64_t v, int64_t chunk,
                                                          Partial<float>* __restrict__ part,
                                                          float* __restrict__ sxpart,
                                                          float* __restrict__ opart) {
  using L = Lay<float>;
  constexpr int R = L::XR, C = L::XC, PAD = L::PAD;
  using M = LayMap<float, R, C>;
  static_assert(M::kVec && M::CG == 32, "a warp owns four whole rows of the tile");
  constexpr int GS = gstride(R);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* Xs = reinterpret_cast<float*>(smem_raw);
  float* Es = Xs + D * (R + PAD);
  float* Gs = Xs + align16<float>(static_cast<size_t>(D) * (R + PAD + C + PAD));  // [C][GS]
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * R;
  const int64_t c_begin = static_cast<int64_t>(blockIdx.y) * chunk;
  const int64_t c_end = min(v, c_begin + chunk);
  stage_T<float, R, PAD>(Xs, X, r0, n, D);
  const int lane = threadIdx.x % 32, wr = (threadIdx.x / 32) * 4;  // == M::row(0)
  int64_t tgt[4];
  float mx[4], sm[4], sx[4], tv[4], has[4];  // sx: the row sum without the target entry
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = r0 + wr + i;
    tgt[i] = row < n ? targets[row] : -1;
    mx[i] = -INFINITY;
    sm[i] = 0.f;
    sx[i] = 0.f;
    tv[i] = 0.f;
    has[i] = 0.f;
  }
  const int nq = (D - lane + 31) / 32;
  float acc[4][NQ];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[r][q] = 0.f;

  for (int64_t c0 = c_begin; c0 < c_end; c0 += C) {
    __syncthreads();
    stage_T<float, C, PAD>(Es, E, c0, c_end, D);
    __syncthreads();
    float o[4][4];
    M::logits(Xs, Es, D, o);
    float alpha[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float tm = -INFINITY;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (c0 + M::col(q) >= c_end) o[i][q] = -INFINITY;
        tm = fmaxf(tm, o[i][q]);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, off));
      const float nm = fmaxf(mx[i], tm);  // finite: every tile has a valid column
      alpha[i] = mx[i] == -INFINITY ? 0.f : expf(mx[i] - nm);
      mx[i] = nm;
    }
    float pe[4][4];  // P with the target entry left out
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float ps = 0.f, pxs = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float pv = expf(o[i][q] - mx[i]);  // 0 for a masked column
        ps += pv;
        const bool t = c0 + M::col(q) == tgt[i];
        if (t) {
          tv[i] = o[i][q];
          has[i] = 1.f;
        }
        pe[i][q] = t ? 0.f : pv;
        pxs += pe[i][q];
      }
      sm[i] = sm[i] * alpha[i] + ps;
      sx[i] = sx[i] * alpha[i] + pxs;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<float4*>(Gs + M::col(q) * GS + wr) = make_float4(pe[0][q], pe[1][q], pe[2][q], pe[3][q]);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < NQ; ++q) acc[r][q] *= alpha[r];
    const int cn = static_cast<int>((c_end - c0 < C ? c_end - c0 : C));
    for (int j = 0; j < cn; j += 4) {
      float gv[4][4], ev[NQ][4];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) ld4(Gs + (j + jj) * GS + wr, gv[jj]);
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < nq) ld4(Es + (lane + 32 * q) * (C + PAD) + j, ev[q]);
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (q < nq) {
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[r][q] = fmaf(gv[jj][r], ev[q][jj], acc[r][q]);
          }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float si = sm[i], xi = sx[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      si += __shfl_xor_sync(0xffffffffu, si, off);
      xi += __shfl_xor_sync(0xffffffffu, xi, off);
    }
    const unsigned hb = __ballot_sync(0xffffffffu, has[i] != 0.f);
    const float ti = __shfl_sync(0xffffffffu, tv[i], hb ? __ffs(hb) - 1 : 0);
    const int64_t row = r0 + wr + i;
    if (row < n) {
      if (lane == 0) {
        Partial<float> pp;
        pp.m = mx[i];
        pp.s = si;
        pp.t = hb ? ti : 0.f;
        pp.has = hb ? 1.f : 0.f;
        part[static_cast<int64_t>(blockIdx.y) * n + row] = pp;
        sxpart[static_cast<int64_t>(blockIdx.y) * n + row] = xi;
      }
      float* out = opart + (static_cast<int64_t>(blockIdx.y) * n + row) * D;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < nq) out[lane + 32 * q] = acc[i][q];
    }
  }
}

// Warp per row: lse / pos from the chunk partials, then dX (see above).
// lse = t + log1p(Sx / e^(t - M)) and 1 - p_t = Sx / (e^(t - M) + Sx) from the
// sum without the target (Sx), so both keep full precision when the target
// dominates the row (a total sum rounded to e^(t - M) would lose them).
__global__ void simt_fwdx_combine(const Partial<float>* __restrict__ part, const float* __restrict__ sxpart,
                                  const float* __restrict__ opart, int P, int64_t n, int D,
                                  const float* __restrict__ E, const int64_t* __restrict__ targets,
                                  double scale, double* __restrict__ lse, double* __restrict__ pos,
                                  double* __restrict__ omp_out, float* __restrict__ dX) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= n) return;
  double Mx = -INFINITY;
  for (int p = 0; p < P; ++p) Mx = fmax(Mx, static_cast<double>(part[p * n + row].m));
  double Sx = 0.0, t = 0.0;
  bool found = false;
  for (int p = 0; p < P; ++p) {
    const Partial<float> q = part[p * n + row];
    Sx += static_cast<double>(sxpart[p * n + row]) * exp(static_cast<double>(q.m) - Mx);
    if (q.has != 0.f) {
      t = q.t;
      found = true;
    }
  }
  const double St = found ? exp(t - Mx) : 0.0;  // the target's own term
  const double l = found ? t + log1p(Sx / St) : Mx + log(Sx);
  const double omp = found ? Sx / (St + Sx) : 1.0;  // 1 - p_t
  if (lane == 0) {
    lse[row] = l;
    pos[row] = t;
    omp_out[row] = omp;
  }
  const float* et = E + targets[row] * D;
  for (int k = lane; k < D; k += 32) {
    double acc = 0.0;
    for (int p = 0; p < P; ++p)
      acc += static_cast<double>(opart[(static_cast<int64_t>(p) * n + row) * D + k]) *
             exp(static_cast<double>(part[p * n + row].m) - l);
    dX[row * D + k] = static_cast<float>(scale * (acc - omp * static_cast<double>(et[k])));
  }
}
}  // namespace

// ---------------------------------------------------------------------------
// Combine / reduce (shared with the tensor-core path).
// ---------------------------------------------------------------------------
template <class T, bool LOG2>
__global__ void combine_partials(const Partial<T>* __restrict__ part, int P, int64_t n,
                                 double* __restrict__ lse, double* __restrict__ pos) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double M = -INFINITY;
  for (int p = 0; p < P; ++p) M = fmax(M, static_cast<double>(part[p * n + i].m));
  double S = 0.0, t = 0.0;
  for (int p = 0; p < P; ++p) {
    const Partial<T> q = part[p * n + i];
    if (q.m != -INFINITY) S += static_cast<double>(q.s) * (LOG2 ? exp2(static_cast<double>(q.m) - M)
                                                               : exp(static_cast<double>(q.m) - M));
    if (q.has != T(0)) t = static_cast<double>(q.t);
  }
  lse[i] = LOG2 ? (M + log2(S)) * 0.6931471805599453 : M + log(S);
  pos[i] = t;
}

// loss = mean(lse - pos), one block, fixed summation order (deterministic).
__global__ void mean_loss(const double* __restrict__ lse, const double* __restrict__ pos,
                          int64_t n, double* __restrict__ loss) {
  __shared__ double red[1024];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += lse[i] - pos[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = red[0] / static_cast<double>(n);
}

template <class Tin, class Tout>
__global__ void reduce_chunks(const Tin* __restrict__ part, int P, int64_t count,
                              Tout* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    Tin acc = part[i];
    for (int p = 1; p < P; ++p) acc += part[p * count + i];
    out[i] = static_cast<Tout>(acc);
  }
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
int launch_combine_f32log2(const float* part, int P, int64_t n, double* lse, double* pos,
                           double* loss, cudaStream_t st) {
  if (n <= 0) return fail(LF_EINVAL, "combine: n must be >= 1");
  combine_partials<float, true><<<ceil_div(n, 256), 256, 0, st>>>(
      reinterpret_cast<const Partial<float>*>(part), P, n, lse, pos);
  LF_LAUNCHED();
  if (loss) {
    mean_loss<<<1, 1024, 0, st>>>(lse, pos, n, loss);
    LF_LAUNCHED();
  }
  return LF_OK;
}

template <class T>
static size_t fwd_smem(int D) {
  using L = Lay<T>;
  return sizeof(T) * D * (L::FR + L::PAD + L::FC + L::PAD);
}
template <class T>
static size_t dx_smem(int D) {  // Xs, Es, then the XC x gstride(XR) G tile
  using L = Lay<T>;
  return sizeof(T) * (align16<T>(static_cast<size_t>(D) * (L::XR + L::PAD + L::XC + L::PAD)) + L::XC * gstride(L::XR));
}
template <class T>
static size_t de_smem(int D) {  // Es, Xs, then the ER x gstride(EC) G tile
  using L = Lay<T>;
  return sizeof(T) * (align16<T>(static_cast<size_t>(D) * (L::EC + L::PAD + L::ER + L::PAD)) + L::ER * gstride(L::EC));
}

static int64_t pick_chunks(int64_t row_tiles, int64_t v, int64_t min_cols) {
  const int64_t want = 4 * num_sms();
  int64_t chunks = ceil_div(want, row_tiles);
  chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, ceil_div(v, min_cols)));
  return chunks;
}

// V chunks for a (row tiles x chunks) grid: the count in [1, max_chunks]
// (chunks of at least min_cols columns) that minimises the per-SM serial work
// waves(P) / P, waves = ceil(rt P / (SMs x resident blocks)) — a second
// wave that is mostly empty costs as much as a full one.
template <class K>
static int64_t balanced_chunks(K kernel, size_t smem, int64_t rt, int64_t v, int64_t min_cols,
                               int64_t max_chunks) {
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t slots = static_cast<int64_t>(per_sm) * num_sms();
  const int64_t hi = std::max<int64_t>(1, std::min<int64_t>(max_chunks, ceil_div(v, min_cols)));
  int64_t best = 1;
  double best_cost = 1e300;
  for (int64_t P = 1; P <= hi; ++P) {
    const double cost = static_cast<double>(ceil_div(rt * P, slots)) / static_cast<double>(P);
    if (cost < best_cost * (1.0 - 1e-9)) {
      best_cost = cost;
      best = P;
    }
  }
  return best;
}

template <class T>
int simt_cce_forward(const T* X, const T* E, const int64_t* targets, int64_t n, int D,
                     int64_t v, int64_t v_offset, Partial<T>** part_out, int* P_out,
                     Scratch& ws, cudaStream_t st) {
  const size_t smem = fwd_smem<T>(D);
  if (smem > 227 * 1024) return fail(LF_EUNSUPPORTED, "simt forward: d too large");
  LF_CUDA(cudaFuncSetAttribute(cce_simt_fwd<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  const int64_t rt = ceil_div(n, Lay<T>::FR);
  const int64_t chunks = balanced_chunks(cce_simt_fwd<T>, smem, rt, v, 256, 64);
  const int64_t chunk = ceil_div(ceil_div(v, chunks), Lay<T>::FC) * Lay<T>::FC;
  const int64_t P = ceil_div(v, chunk);
  int rc = ws.alloc(sizeof(Partial<T>) * P * n, st);
  if (rc) return rc;
  ProfScope prof(LF_K_CCE_SIMT, st);
  cce_simt_fwd<T><<<dim3(rt, P), kThreads, smem, st>>>(X, E, targets, n, D, v, v_offset, chunk,
                                                      ws.as<Partial<T>>());
  LF_LAUNCHED();
  *part_out = ws.as<Partial<T>>();
  *P_out = static_cast<int>(P);
  return LF_OK;
}

template <class T>
int simt_cce_forward_full(const T* X, const T* E, const int64_t* targets, int64_t n, int D,
                          int64_t v, double* lse, double* pos, double* loss, cudaStream_t st) {
  Scratch ws;
  Partial<T>* part;
  int P;
  int rc = simt_cce_forward<T>(X, E, targets, n, D, v, 0, &part, &P, ws, st);
  if (rc) return rc;
  combine_partials<T, false><<<ceil_div(n, 256), 256, 0, st>>>(part, P, n, lse, pos);
  LF_LAUNCHED();
  if (loss) {
    mean_loss<<<1, 1024, 0, st>>>(lse, pos, n, loss);
    LF_LAUNCHED();
  }
  return LF_OK;
}

template <class T>
int simt_cce_forward_partial_log2(const T* X, const T* E, const int64_t* targets, int64_t n,
                                  int D, int64_t v, int64_t v_offset, float* out,
                                  cudaStream_t st);

template <class T>
__global__ void partial_to_log2(const Partial<T>* __restrict__ part, int P, int64_t n,
                                float4* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double M = -INFINITY;
  for (int p = 0; p < P; ++p) M = fmax(M, static_cast<double>(part[p * n + i].m));
  double S = 0.0, t = 0.0, h = 0.0;
  for (int p = 0; p < P; ++p) {
    const Partial<T> q = part[p * n + i];
    if (q.m != -INFINITY) S += static_cast<double>(q.s) * exp(static_cast<double>(q.m) - M);
    if (q.has != T(0)) { t = static_cast<double>(q.t); h = 1.0; }
  }
  out[i] = make_float4(static_cast<float>(M * 1.4426950408889634), static_cast<float>(S),
                       static_cast<float>(t), static_cast<float>(h));
}

template <class T>
int simt_cce_forward_partial_log2(const T* X, const T* E, const int64_t* targets, int64_t n,
                                  int D, int64_t v, int64_t v_offset, float* out,
                                  cudaStream_t st) {
  Scratch ws;
  Partial<T>* part;
  int P;
  int rc = simt_cce_forward<T>(X, E, targets, n, D, v, v_offset, &part, &P, ws, st);
  if (rc) return rc;
  partial_to_log2<T><<<ceil_div(n, 256), 256, 0, st>>>(part, P, n, reinterpret_cast<float4*>(out));
  LF_LAUNCHED();
  return LF_OK;
}

// The dE pass: one block per 32 items over all rows — fp32 splits the rows
// into Q slices when that fills the SMs' last wave better (partial dE per
// slice, then a fixed-order sum); fp64 keeps one slice (reference order).
template <class T, int NQ>
static int launch_de(const T* X, const T* E, const int64_t* targets, const double* lse, int64_t n, int D,
                     int64_t v, int64_t v_offset, T scale, T eps, T* dE, size_t sde, const double* omp,
                     cudaStream_t st) {
  constexpr int R = Lay<T>::ER;
  const int64_t blocks = ceil_div(v, Lay<T>::EC);
  int64_t Q = 1;
  if (sizeof(T) == 4 && sizeof(T) * 4 * v * D <= (int64_t(256) << 20))
    Q = balanced_chunks(cce_simt_bwd_de<T, NQ>, sde, blocks, n, R, 4);
  const int64_t rows_per = ceil_div(ceil_div(n, R), Q) * R;
  Q = ceil_div(n, rows_per);
  Scratch part;
  T* out = dE;
  if (Q > 1) {
    const int rc = part.alloc(sizeof(T) * Q * v * D, st);
    if (rc) return rc;
    out = part.as<T>();
  }
  cce_simt_bwd_de<T, NQ><<<dim3(blocks, Q), kThreads, sde, st>>>(X, E, targets, lse, n, D, v, v_offset, scale,
                                                                  eps, out, rows_per, omp);
  LF_LAUNCHED();
  if (Q > 1) {
    reduce_chunks<T, T><<<std::min<int64_t>(ceil_div(v * D, 256), 4 * num_sms()), 256, 0, st>>>(
        out, static_cast<int>(Q), v * D, dE);
    LF_LAUNCHED();
  }
  return LF_OK;
}

template <class T, int NQ>
static int simt_backward_nq(const T* X, const T* E, const int64_t* targets, const double* lse, double scale,
                            double eps, int64_t n, int D, int64_t v, int64_t v_offset, T* dX, T* dE,
                            unsigned long long* skip_counter, size_t sdx, size_t sde, cudaStream_t st) {
  LF_CUDA(cudaFuncSetAttribute(cce_simt_bwd_dx<T, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(sdx)));
  LF_CUDA(cudaFuncSetAttribute(cce_simt_bwd_de<T, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(sde)));
  const int64_t rt = ceil_div(n, Lay<T>::XR);
  // dX partials: P x n x D of scratch, so at most 16 chunks (8 past 64 MB)
  const int64_t max_p = sizeof(T) * 16 * n * D <= (int64_t(64) << 20) ? 16 : 8;
  const int64_t chunks = balanced_chunks(cce_simt_bwd_dx<T, NQ>, sdx, rt, v, 1024, max_p);
  const int64_t chunk = ceil_div(ceil_div(v, chunks), Lay<T>::XC) * Lay<T>::XC;
  const int64_t P = ceil_div(v, chunk);
  Scratch ws;
  T* part = dX;
  if (P > 1) {
    int rc = ws.alloc(sizeof(T) * P * n * D, st);
    if (rc) return rc;
    part = ws.as<T>();
  }
  ProfScope prof(LF_K_CCE_SIMT, st);
  cce_simt_bwd_dx<T, NQ><<<dim3(rt, P), kThreads, sdx, st>>>(X, E, targets, lse, n, D, v, v_offset,
                                                        chunk, T(scale), T(eps), part,
                                                        skip_counter);
  LF_LAUNCHED();
  if (P > 1) {
    reduce_chunks<T, T><<<std::min<int64_t>(ceil_div(n * D, 256), 4 * num_sms()), 256, 0, st>>>(
        part, static_cast<int>(P), n * D, dX);
    LF_LAUNCHED();
  }
  return launch_de<T, NQ>(X, E, targets, lse, n, D, v, v_offset, T(scale), T(eps), dE, sde, nullptr, st);
}


template <class T>
int simt_cce_backward(const T* X, const T* E, const int64_t* targets, const double* lse, double scale,
                      double eps, int64_t n, int D, int64_t v, int64_t v_offset, T* dX, T* dE,
                      unsigned long long* skip_counter, cudaStream_t st) {
  const size_t sdx = dx_smem<T>(D), sde = de_smem<T>(D);
  if (sdx > 227 * 1024 || sde > 227 * 1024) return fail(LF_EUNSUPPORTED, "simt backward: d too large");
  if (D > 256) return fail(LF_EUNSUPPORTED, "simt backward: d > 256");
  const int nq = (D + 31) / 32;
  return nq <= 1 ? simt_backward_nq<T, 1>(X, E, targets, lse, scale, eps, n, D, v, v_offset, dX, dE,
                                           skip_counter, sdx, sde, st)
       : nq <= 2 ? simt_backward_nq<T, 2>(X, E, targets, lse, scale, eps, n, D, v, v_offset, dX, dE,
                                           skip_counter, sdx, sde, st)
       : nq <= 4 ? simt_backward_nq<T, 4>(X, E, targets, lse, scale, eps, n, D, v, v_offset, dX, dE,
                                           skip_counter, sdx, sde, st)
                 : simt_backward_nq<T, 8>(X, E, targets, lse, scale, eps, n, D, v, v_offset, dX, dE,
                                           skip_counter, sdx, sde, st);
}

template <int NQ>
static int simt_fused_nq(const float* X, const float* E, const int64_t* targets, int64_t n, int D, int64_t v,
                         double scale, double eps, double* lse, double* pos, double* loss, float* dX, float* dE,
                         cudaStream_t st) {
  const size_t sfx = dx_smem<float>(D), sde = de_smem<float>(D);
  LF_CUDA(cudaFuncSetAttribute(cce_simt_fwdx<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(sfx)));
  LF_CUDA(cudaFuncSetAttribute(cce_simt_bwd_de<float, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(sde)));
  const int64_t rt = ceil_div(n, Lay<float>::XR);
  // O partials: P x n x D floats, so at most 16 chunks (8 past 64 MB)
  const int64_t max_p = sizeof(float) * 16 * n * D <= (int64_t(64) << 20) ? 16 : 8;
  const int64_t chunks = balanced_chunks(cce_simt_fwdx<NQ>, sfx, rt, v, 1024, max_p);
  const int64_t chunk = ceil_div(ceil_div(v, chunks), Lay<float>::XC) * Lay<float>::XC;
  const int64_t P = ceil_div(v, chunk);
  Scratch omp;
  int rc = omp.alloc(sizeof(double) * n, st);
  if (rc) return rc;
  {
    Scratch part, sxpart, opart;
    rc = part.alloc(sizeof(Partial<float>) * P * n, st);
    if (!rc) rc = sxpart.alloc(sizeof(float) * P * n, st);
    if (!rc) rc = opart.alloc(sizeof(float) * P * n * D, st);
    if (rc) return rc;
    ProfScope prof(LF_K_CCE_SIMT, st);
    cce_simt_fwdx<NQ><<<dim3(rt, P), kThreads, sfx, st>>>(X, E, targets, n, D, v, chunk,
                                                         part.as<Partial<float>>(), sxpart.as<float>(),
                                                         opart.as<float>());
    LF_LAUNCHED();
    simt_fwdx_combine<<<ceil_div(n, 8), 256, 0, st>>>(part.as<Partial<float>>(), sxpart.as<float>(),
                                                      opart.as<float>(), static_cast<int>(P), n, D, E,
                                                      targets, scale, lse, pos, omp.as<double>(), dX);
    LF_LAUNCHED();
    if (loss) {
      rc = launch_mean_loss(lse, pos, n, loss, st);
      if (rc) return rc;
    }
  }  // the O partials go back to the pool before the dE pass
  ProfScope prof(LF_K_CCE_SIMT, st);
  return launch_de<float, NQ>(X, E, targets, lse, n, D, v, 0, static_cast<float>(scale), static_cast<float>(eps),
                              dE, sde, omp.as<double>(), st);
}

int simt_cce_fused_f32(const float* X, const float* E, const int64_t* targets, int64_t n, int D, int64_t v,
                       double scale, double eps, double* lse, double* pos, double* loss, float* dX, float* dE,
                       cudaStream_t st) {
  const size_t sfx = dx_smem<float>(D), sde = de_smem<float>(D);
  if (D > 256 || sfx > 227 * 1024 || sde > 227 * 1024) return fail(LF_EUNSUPPORTED, "simt fused: d too large");
  const int nq = (D + 31) / 32;
  return nq <= 1 ? simt_fused_nq<1>(X, E, targets, n, D, v, scale, eps, lse, pos, loss, dX, dE, st)
       : nq <= 2 ? simt_fused_nq<2>(X, E, targets, n, D, v, scale, eps, lse, pos, loss, dX, dE, st)
       : nq <= 4 ? simt_fused_nq<4>(X, E, targets, n, D, v, scale, eps, lse, pos, loss, dX, dE, st)
                 : simt_fused_nq<8>(X, E, targets, n, D, v, scale, eps, lse, pos, loss, dX, dE, st);
}

// ---------------------------------------------------------------------------
// Full-catalog ranking, fp32 / fp64 (metrics.cpp:46-78).  Block = 32 rows x
// one V chunk; the 32 x 64 score tile is staged in shared memory and each
// warp walks 4 rows: lanes count the items ranked ahead of the target (score
// higher, or equal with a smaller item index) and the row's top-K (K <= 32)
// lives across the warp's lanes, lane e holding entry e (descending score,
// ties to the smaller index).  Scores use the k-ascending operand order of
// the reference (exact in fp64), and st is computed by eval_target_scores in
// the same order, so a score compares equal to st exactly when it would in
// the reference.
// ---------------------------------------------------------------------------
template <class T>
__global__ void eval_target_scores(const T* __restrict__ X, const T* __restrict__ Et, int64_t n,
                                   int D, T* __restrict__ st) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T acc = T(0);
  for (int k = 0; k < D; ++k) acc = fma_acc(acc, X[i * D + k], Et[i * D + k]);
  st[i] = acc;
}

template <class T>
__global__ void __launch_bounds__(kThreads) eval_simt(const T* __restrict__ X,
                                                      const T* __restrict__ E,
                                                      const T* __restrict__ st_in,
                                                      const int32_t* __restrict__ tl, int64_t n,
                                                      int D, int64_t v, int64_t chunk, int K,
                                                      uint32_t* __restrict__ cnt_out,
                                                      T* __restrict__ val_out,
                                                      int32_t* __restrict__ idx_out) {
  constexpr int R = 32, C = 64, RW = 4;  // rows per warp
  using M = TileMap<T, R, C>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Xs = reinterpret_cast<T*>(smem_raw);
  T* Es = Xs + D * (R + 1);
  T* Ss = Es + D * (C + 1);  // [R][C + 1]
  const unsigned full = 0xffffffffu;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * R;
  const int64_t c_begin = static_cast<int64_t>(blockIdx.y) * chunk;
  const int64_t c_end = min(v, c_begin + chunk);
  stage_T<T, R>(Xs, X, r0, n, D);
  T stv[RW], kv[RW];
  int64_t tlv[RW];
  int ki[RW];
  uint32_t cnt[RW];
#pragma unroll
  for (int rr = 0; rr < RW; ++rr) {
    const int64_t row = r0 + warp * RW + rr;
    stv[rr] = row < n ? st_in[row] : T(0);
    tlv[rr] = row < n ? tl[row] : -1;
    kv[rr] = neg_inf<T>();
    ki[rr] = 0x7fffffff;
    cnt[rr] = 0;
  }
  for (int64_t c0 = c_begin; c0 < c_end; c0 += C) {
    __syncthreads();
    stage_T<T, C>(Es, E, c0, c_end, D);
    __syncthreads();
    {
      T o[M::RPT][M::CPT];
      M::logits(Xs, Es, D, o);
#pragma unroll
      for (int i = 0; i < M::RPT; ++i)
#pragma unroll
        for (int q = 0; q < M::CPT; ++q) Ss[M::row(i) * (C + 1) + M::col(q)] = o[i][q];
    }
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
      const int r = warp * RW + rr;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int cl = half * 32 + lane;
        const int64_t col = c0 + cl;
        const bool valid = col < c_end;
        const T val = Ss[r * (C + 1) + cl];
        if (valid) cnt[rr] += col < tlv[rr] ? (val >= stv[rr]) : (col > tlv[rr] ? (val > stv[rr]) : 0);
        // columns arrive in ascending order, so an equal score never displaces
        const T kth = __shfl_sync(full, kv[rr], K - 1);
        unsigned bm = __ballot_sync(full, valid && val > kth);
        while (bm) {
          const int src = __ffs(bm) - 1;
          bm &= bm - 1u;
          const T cv = __shfl_sync(full, val, src);
          const int ci = static_cast<int>(c0 + half * 32 + src);
          const bool ahead = lane < K && (kv[rr] > cv || (kv[rr] == cv && ki[rr] < ci));
          const int pos = __popc(__ballot_sync(full, ahead));
          const T upv = __shfl_up_sync(full, kv[rr], 1);
          const int upi = __shfl_up_sync(full, ki[rr], 1);
          if (lane == pos) {
            kv[rr] = cv;
            ki[rr] = ci;
          } else if (lane > pos && lane < K) {
            kv[rr] = upv;
            ki[rr] = upi;
          }
        }
      }
    }
  }
#pragma unroll
  for (int rr = 0; rr < RW; ++rr) {
    uint32_t c = cnt[rr];
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(full, c, off);
    const int64_t row = r0 + warp * RW + rr;
    if (row < n) {
      const int64_t rp = static_cast<int64_t>(blockIdx.y) * n + row;
      if (lane == 0) cnt_out[rp] = c;
      if (lane < K) {
        val_out[rp * K + lane] = kv[rr];
        idx_out[rp * K + lane] = ki[rr];
      }
    }
  }
}

template <class T>
int simt_eval_partials(const T* X, const T* E, const T* Et, const int32_t* tl, int64_t n, int D,
                       int64_t v, int K, Scratch& cnt, Scratch& val, Scratch& idx, int* P_out,
                       cudaStream_t st) {
  const size_t smem = sizeof(T) * (D * (32 + 1 + 64 + 1) + 32 * (64 + 1));
  if (smem > 227 * 1024) return fail(LF_EUNSUPPORTED, "simt eval: d too large");
  LF_CUDA(cudaFuncSetAttribute(eval_simt<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  const int64_t rt = ceil_div(n, 32);
  const int64_t chunks = pick_chunks(rt, v, 256);
  const int64_t chunk = ceil_div(ceil_div(v, chunks), 64) * 64;
  const int64_t P = ceil_div(v, chunk);
  Scratch stv;
  int rc = stv.alloc(sizeof(T) * n, st);
  if (!rc) rc = cnt.alloc(sizeof(uint32_t) * P * n, st);
  if (!rc) rc = val.alloc(sizeof(T) * P * n * K, st);
  if (!rc) rc = idx.alloc(sizeof(int32_t) * P * n * K, st);
  if (rc) return rc;
  ProfScope prof(LF_K_EVAL, st);
  eval_target_scores<T><<<ceil_div(n, 128), 128, 0, st>>>(X, Et, n, D, stv.as<T>());
  LF_LAUNCHED();
  eval_simt<T><<<dim3(rt, P), kThreads, smem, st>>>(X, E, stv.as<T>(), tl, n, D, v, chunk, K,
                                                    cnt.as<uint32_t>(), val.as<T>(),
                                                    idx.as<int32_t>());
  LF_LAUNCHED();
  *P_out = static_cast<int>(P);
  return LF_OK;
}

template int simt_eval_partials<float>(const float*, const float*, const float*, const int32_t*,
                                       int64_t, int, int64_t, int, Scratch&, Scratch&, Scratch&,
                                       int*, cudaStream_t);
template int simt_eval_partials<double>(const double*, const double*, const double*,
                                        const int32_t*, int64_t, int, int64_t, int, Scratch&,
                                        Scratch&, Scratch&, int*, cudaStream_t);

template int simt_cce_forward_full<float>(const float*, const float*, const int64_t*, int64_t, int,
                                          int64_t, double*, double*, double*, cudaStream_t);
template int simt_cce_forward_full<double>(const double*, const double*, const int64_t*, int64_t,
                                           int, int64_t, double*, double*, double*, cudaStream_t);
template int simt_cce_forward_partial_log2<float>(const float*, const float*, const int64_t*,
                                                  int64_t, int, int64_t, int64_t, float*,
                                                  cudaStream_t);
template int simt_cce_forward_partial_log2<double>(const double*, const double*, const int64_t*,
                                                   int64_t, int, int64_t, int64_t, float*,
                                                   cudaStream_t);
template int simt_cce_backward<float>(const float*, const float*, const int64_t*, const double*,
                                      double, double, int64_t, int, int64_t, int64_t, float*,
                                      float*, unsigned long long*, cudaStream_t);
template int simt_cce_backward<double>(const double*, const double*, const int64_t*,
                                       const double*, double, double, int64_t, int, int64_t,
                                       int64_t, double*, double*, unsigned long long*,
                                       cudaStream_t);

int launch_reduce_f32(const float* part, int P, int64_t count, float* out, cudaStream_t st) {
  reduce_chunks<float, float><<<std::min<int64_t>(ceil_div(count, 256), 4 * num_sms()), 256, 0, st>>>(
      part, P, count, out);
  LF_LAUNCHED();
  return LF_OK;
}

__global__ void fold_partials(const float4* __restrict__ part, int P, int64_t n,
                              float4* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float M = -INFINITY;
  for (int p = 0; p < P; ++p) M = fmaxf(M, part[p * n + i].x);
  float S = 0.f, t = 0.f, h = 0.f;
  for (int p = 0; p < P; ++p) {
    const float4 q = part[p * n + i];
    if (q.x != -INFINITY) S += q.y * exp2f(q.x - M);
    if (q.w != 0.f) { t = q.z; h = 1.f; }
  }
  out[i] = make_float4(M, S, t, h);
}

__global__ void negate_kernel(float* __restrict__ x, int64_t count) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = -x[i];
}

int launch_fold_partials(const float* part, int P, int64_t n, float* out, cudaStream_t st) {
  fold_partials<<<ceil_div(n, 256), 256, 0, st>>>(reinterpret_cast<const float4*>(part), P, n,
                                                  reinterpret_cast<float4*>(out));
  LF_LAUNCHED();
  return LF_OK;
}

int launch_negate(float* x, int64_t count, cudaStream_t st) {
  negate_kernel<<<std::min<int64_t>(ceil_div(count, 256), 8 * num_sms()), 256, 0, st>>>(x, count);
  LF_LAUNCHED();
  return LF_OK;
}

int launch_mean_loss(const double* lse, const double* pos, int64_t n, double* loss, cudaStream_t st) {
  mean_loss<<<1, 1024, 0, st>>>(lse, pos, n, loss);
  LF_LAUNCHED();
  return LF_OK;
}

}  // namespace lf
