// lf_encoder.cu — the toy sequence encoder on either side of the loss, on the
// device: encode_batch (proj/src/encoder.cpp:64-116) produces the hidden rows
// the CCE kernels consume, encoder_backward (encoder.cpp:118-173) consumes
// their dX.  With lf_adam_step this keeps the whole training step
// (trainer.cpp:209-227) on the GPU.
//
// Everything is computed in double in the reference's operand order (one
// rounding per operation, __dmul_rn / __dadd_rn): pooled means a are bitwise
// the reference's; h = tanh(z) uses CUDA's tanh (within an ulp of glibc's),
// so h and the gradients match the reference to ~1e-15 relative.  d_emb sums
// each item's suffix vectors serially in the reference's visiting order (rows
// grouped per item by a stable sort, then reduced in order); d_W / d_b sum the
// rows from last to first in 256-row chunks combined in a fixed order
// (encoder.cpp:136-154; re-associated, deterministic).
//
// Windows arrive as a device CSR (items, win_off[n_windows + 1]); rows are
// enumerated window by window, position t = 1 .. len-1 (encoder.cpp:88-112).
#include <cuda_bf16.h>

#include <algorithm>
#include <string>

#include "lf_internal.cuh"
#include "lf_kernels.cuh"

namespace lf {
namespace {

// row_off[w] = sum_{w' < w} (len_w' - 1); status[0] = first window with fewer
// than 2 items, status[1] = total rows.  One thread (n_windows is a batch).
__global__ void window_rows(const int64_t* __restrict__ win_off, int64_t n_windows,
                            int64_t* __restrict__ row_off, unsigned long long* __restrict__ status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t r = 0;
  for (int64_t w = 0; w < n_windows; ++w) {
    row_off[w] = r;
    const int64_t len = win_off[w + 1] - win_off[w];
    if (len < 2 && status[0] == ~0ull) status[0] = static_cast<unsigned long long>(w);
    r += len > 1 ? len - 1 : 0;
  }
  row_off[n_windows] = r;
  status[1] = static_cast<unsigned long long>(r);
}

// Warp per window (encoder.cpp:88-102): running sum of the prefix's item rows,
// a = sum * (1/t); the dense part runs per row (encode_rows).
__global__ void __launch_bounds__(256) encode_windows(
    const int64_t* __restrict__ items, const int64_t* __restrict__ win_off,
    const int64_t* __restrict__ row_off, int64_t n_windows, const float* __restrict__ emb,
    int64_t catalog, int D, double* __restrict__ a_out, int64_t* __restrict__ targets, int64_t* __restrict__ row_window, int64_t* __restrict__ row_pos,
    unsigned long long* __restrict__ bad_item) {
  extern __shared__ double sm[];  // per warp: sum[D]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (w >= n_windows) return;
  double* sum = sm + warp * D;
  const int64_t* win = items + win_off[w];
  const int64_t len = win_off[w + 1] - win_off[w];
  for (int k = lane; k < D; k += 32) sum[k] = 0.0;
  for (int64_t t = 1; t < len; ++t) {
    const int64_t prev = win[t - 1], cur = win[t];
    if (prev < 0 || prev >= catalog || cur < 0 || cur >= catalog) {  // check_item, encoder.cpp:11-16
      if (lane == 0) atomicMin(bad_item, static_cast<unsigned long long>(win_off[w] + (prev < 0 || prev >= catalog ? t - 1 : t)));
      return;
    }
    const int64_t r = row_off[w] + t - 1;
    const double inv = __ddiv_rn(1.0, static_cast<double>(t));
    for (int k = lane; k < D; k += 32) {
      sum[k] = __dadd_rn(sum[k], static_cast<double>(emb[prev * D + k]));
      a_out[r * D + k] = __dmul_rn(sum[k], inv);
    }
    if (lane == 0) {
      targets[r] = cur;
      row_window[r] = w;
      row_pos[r] = t;
    }
  }
}

// Warp per row (encoder.cpp:103-108): z_j = b_j + sum_k W[j][k] a_k (k
// ascending), h = tanh(z), e = float(h).
__global__ void __launch_bounds__(256) encode_rows(const double* __restrict__ a, const float* __restrict__ W,
                                                  const float* __restrict__ bias, int64_t rows, int D,
                                                  double* __restrict__ h_out, float* __restrict__ e_out) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (r >= rows) return;
  double* as = sm + warp * D;
  for (int k = lane; k < D; k += 32) as[k] = a[r * D + k];
  __syncwarp();
  for (int j = lane; j < D; j += 32) {
    double z = static_cast<double>(bias[j]);
    const float* wrow = W + static_cast<int64_t>(j) * D;
    for (int k = 0; k < D; ++k) z = __dadd_rn(z, __dmul_rn(static_cast<double>(wrow[k]), as[k]));
    const double hv = tanh(z);
    h_out[r * D + j] = hv;
    e_out[r * D + j] = static_cast<float>(hv);
  }
}

// Warp per row (encoder.cpp:145-160): g = (1 - h^2) dh, u_k = (sum_j W[j][k] g_j) / t.
template <class TD>
__global__ void __launch_bounds__(256) encoder_g_u(const double* __restrict__ h, const TD* __restrict__ dh,
                                                  const int64_t* __restrict__ row_pos,
                                                  const float* __restrict__ W, int64_t rows, int D,
                                                  double* __restrict__ g_out, double* __restrict__ u_out) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (r >= rows) return;
  double* gs = sm + warp * D;
  for (int j = lane; j < D; j += 32) {
    const double hv = h[r * D + j];
    const double gv = __dmul_rn(__dadd_rn(1.0, -__dmul_rn(hv, hv)), static_cast<double>(dh[r * D + j]));
    gs[j] = gv;
    g_out[r * D + j] = gv;
  }
  __syncwarp();
  const double inv = __ddiv_rn(1.0, static_cast<double>(row_pos[r]));
  for (int k = lane; k < D; k += 32) {
    double acc = 0.0;
    for (int j = 0; j < D; ++j) acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(W[j * D + k]), gs[j]));
    u_out[r * D + k] = __dmul_rn(acc, inv);
  }
}

// d_W (D x D) and d_b (D), rows from last to first as the reference visits
// them (encoder.cpp:136-154), in two fixed-order levels: block (o, c) sums
// chunk c's rows (descending) for 256 outputs, then encoder_reduce_chunks
// adds the chunk partials from the last chunk to the first.  Deterministic;
// differs from the single serial sum only by re-association (~1e-16 rel).
constexpr int kRowChunk = 256;
__global__ void __launch_bounds__(256) encoder_dw_db(const double* __restrict__ g, const double* __restrict__ a,
                                                    int64_t rows, int D, double* __restrict__ part) {
  const int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t DD = static_cast<int64_t>(D) * D, nout = DD + D;
  if (o >= nout) return;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kRowChunk;
  const int64_t r1 = min(rows, r0 + kRowChunk);
  double acc = 0.0;
  if (o < DD) {
    const int j = static_cast<int>(o / D), k = static_cast<int>(o % D);
    for (int64_t r = r1 - 1; r >= r0; --r) acc = __dadd_rn(acc, __dmul_rn(g[r * D + j], a[r * D + k]));
  } else {
    const int j = static_cast<int>(o - DD);
    for (int64_t r = r1 - 1; r >= r0; --r) acc = __dadd_rn(acc, g[r * D + j]);
  }
  part[static_cast<int64_t>(blockIdx.y) * nout + o] = acc;
}

__global__ void encoder_reduce_chunks(const double* __restrict__ part, int64_t chunks, int D,
                                      double* __restrict__ dW, double* __restrict__ db) {
  const int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t DD = static_cast<int64_t>(D) * D, nout = DD + D;
  if (o >= nout) return;
  double acc = 0.0;
  for (int64_t c = chunks - 1; c >= 0; --c) acc = __dadd_rn(acc, part[c * nout + o]);
  if (o < DD) dW[o] = acc;
  else db[o - DD] = acc;
}

// Warp per window, rows last to first: suffix += u_t; the suffix is owed to the
// item entering at position t-1 (encoder.cpp:162-167).  Also the per-entry
// item keys for the grouping: entry e = rows-1-r (the reference's visiting order).
__global__ void __launch_bounds__(256) encoder_suffix(const double* __restrict__ u, const int64_t* __restrict__ items,
                                                     const int64_t* __restrict__ win_off,
                                                     const int64_t* __restrict__ row_off, int64_t n_windows,
                                                     int64_t rows, int D, double* __restrict__ contrib,
                                                     int64_t* __restrict__ keys) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (w >= n_windows) return;
  const int64_t rb = row_off[w], re = row_off[w + 1];
  double s[8];  // D <= 256
#pragma unroll
  for (int q = 0; q < 8; ++q) s[q] = 0.0;
  for (int64_t r = re - 1; r >= rb; --r) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = lane + 32 * q;
      if (k < D) {
        s[q] = __dadd_rn(s[q], u[r * D + k]);
        contrib[r * D + k] = s[q];
      }
    }
    if (lane == 0) keys[rows - 1 - r] = items[win_off[w] + (r - rb)];  // win[t-1], t = r - rb + 1
  }
}

// Warp per item: d_emb[item] = sum of its entries' suffix vectors in entry order.
__global__ void __launch_bounds__(256) encoder_demb(const double* __restrict__ contrib,
                                                   const uint32_t* __restrict__ sorted,
                                                   const uint32_t* __restrict__ item_off, int64_t catalog,
                                                   int64_t rows, int D, double* __restrict__ d_emb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (item >= catalog) return;
  const uint32_t b = item_off[item], e = item_off[item + 1];
  for (int k = lane; k < D; k += 32) {
    double acc = 0.0;
    for (uint32_t x = b; x < e; ++x) {
      const int64_t r = rows - 1 - static_cast<int64_t>(sorted[x]);
      acc = __dadd_rn(acc, contrib[r * D + k]);
    }
    d_emb[item * D + k] = acc;
  }
}

}  // namespace

int encode_batch(const int64_t* items, const int64_t* win_off, int64_t n_windows, const float* emb,
                 const float* W, const float* bias, int64_t catalog, int D, int64_t rows, int x_dtype,
                 void* X, double* a, double* h, int64_t* targets, int64_t* row_window,
                 int64_t* row_pos, cudaStream_t st) {
  if (catalog < 1 || D < 1) return fail(LF_EINVAL, "encoder: catalog and hidden must be >= 1");
  if (D > 256) return fail(LF_EUNSUPPORTED, "encoder: hidden > 256");
  if (n_windows < 0 || rows < 0) return fail(LF_EINVAL, "encoder: negative extent");
  Scratch row_off, status, e;
  int rc = row_off.alloc(sizeof(int64_t) * (n_windows + 1), st);
  if (!rc) rc = status.alloc(3 * sizeof(unsigned long long), st);
  if (!rc) rc = e.alloc(sizeof(float) * std::max<int64_t>(rows, 1) * D, st);
  if (rc) return rc;
  LF_CUDA(cudaMemsetAsync(status.ptr, 0xff, 3 * sizeof(unsigned long long), st));
  window_rows<<<1, 32, 0, st>>>(win_off, n_windows, row_off.as<int64_t>(), status.as<unsigned long long>());
  LF_LAUNCHED();
  unsigned long long hs[2];
  LF_CUDA(cudaMemcpyAsync(hs, status.ptr, sizeof(hs), cudaMemcpyDeviceToHost, st));
  LF_CUDA(cudaStreamSynchronize(st));
  if (hs[0] != ~0ull)  // encoder.cpp:75-77
    return fail(LF_EINVAL, "encode_batch: every window needs at least 2 items");
  if (hs[1] == 0) return fail(LF_EINVAL, "encode_batch: batch is empty");  // encoder.cpp:80-82
  if (static_cast<int64_t>(hs[1]) != rows)
    return fail(LF_EINVAL, "encode_batch: rows = " + std::to_string(rows) + " but the windows hold " +
                               std::to_string(hs[1]));
  const size_t smem = sizeof(double) * D * 8;
  encode_windows<<<static_cast<unsigned>(ceil_div(n_windows, 8)), 256, smem, st>>>(
      items, win_off, row_off.as<int64_t>(), n_windows, emb, catalog, D, a, targets, row_window, row_pos,
      status.as<unsigned long long>() + 2);
  LF_LAUNCHED();
  encode_rows<<<static_cast<unsigned>(ceil_div(rows, 8)), 256, smem, st>>>(a, W, bias, rows, D, h, e.as<float>());
  LF_LAUNCHED();
  unsigned long long bad = 0;
  LF_CUDA(cudaMemcpyAsync(&bad, status.as<unsigned long long>() + 2, sizeof(bad), cudaMemcpyDeviceToHost, st));
  LF_CUDA(cudaStreamSynchronize(st));
  if (bad != ~0ull) {
    int64_t item = 0;
    LF_CUDA(cudaMemcpy(&item, items + bad, sizeof(item), cudaMemcpyDeviceToHost));
    return fail(LF_EINVAL, "encode_batch: item id " + std::to_string(item) + " outside catalog of size " +
                               std::to_string(catalog));
  }
  // X = e (float, EncodedBatch::e) in the loss's dtype
  return layout_convert_rows(e.as<float>(), rows * D, x_dtype, X, st);
}

int encoder_backward(const int64_t* items, const int64_t* win_off, int64_t n_windows, const float* W,
                     int64_t catalog, int D, const double* a, const double* h, const int64_t* row_pos,
                     int64_t rows, const void* dh, int dh_dtype, double* d_emb, double* dW, double* db,
                     cudaStream_t st) {
  if (catalog < 1 || D < 1) return fail(LF_EINVAL, "encoder: catalog and hidden must be >= 1");
  if (D > 256) return fail(LF_EUNSUPPORTED, "encoder: hidden > 256");
  if (dh_dtype != LF_F32 && dh_dtype != LF_F64) return fail(LF_EINVAL, "encoder_backward: d_h must be f32 or f64");
  LF_CUDA(cudaMemsetAsync(d_emb, 0, sizeof(double) * catalog * D, st));
  if (rows == 0) {
    LF_CUDA(cudaMemsetAsync(dW, 0, sizeof(double) * D * D, st));
    LF_CUDA(cudaMemsetAsync(db, 0, sizeof(double) * D, st));
    return LF_OK;
  }
  Scratch g, u, contrib, keys, row_off, status, sorted, item_off;
  int rc = g.alloc(sizeof(double) * rows * D, st);
  if (!rc) rc = u.alloc(sizeof(double) * rows * D, st);
  if (!rc) rc = contrib.alloc(sizeof(double) * rows * D, st);
  if (!rc) rc = keys.alloc(sizeof(int64_t) * rows, st);
  if (!rc) rc = row_off.alloc(sizeof(int64_t) * (n_windows + 1), st);
  if (!rc) rc = status.alloc(2 * sizeof(unsigned long long), st);
  if (rc) return rc;
  LF_CUDA(cudaMemsetAsync(status.ptr, 0xff, 2 * sizeof(unsigned long long), st));
  window_rows<<<1, 32, 0, st>>>(win_off, n_windows, row_off.as<int64_t>(), status.as<unsigned long long>());
  LF_LAUNCHED();
  const unsigned row_blocks = static_cast<unsigned>(ceil_div(rows, 8));
  if (dh_dtype == LF_F64)
    encoder_g_u<double><<<row_blocks, 256, sizeof(double) * 8 * D, st>>>(
        h, static_cast<const double*>(dh), row_pos, W, rows, D, g.as<double>(), u.as<double>());
  else
    encoder_g_u<float><<<row_blocks, 256, sizeof(double) * 8 * D, st>>>(
        h, static_cast<const float*>(dh), row_pos, W, rows, D, g.as<double>(), u.as<double>());
  LF_LAUNCHED();
  {
    const int64_t nout = static_cast<int64_t>(D) * D + D, chunks = ceil_div(rows, kRowChunk);
    Scratch part;
    rc = part.alloc(sizeof(double) * nout * chunks, st);
    if (rc) return rc;
    encoder_dw_db<<<dim3(static_cast<unsigned>(ceil_div(nout, 256)), static_cast<unsigned>(chunks)), 256, 0, st>>>(
        g.as<double>(), a, rows, D, part.as<double>());
    LF_LAUNCHED();
    encoder_reduce_chunks<<<static_cast<unsigned>(ceil_div(nout, 256)), 256, 0, st>>>(part.as<double>(), chunks,
                                                                                      D, dW, db);
    LF_LAUNCHED();
  }
  encoder_suffix<<<static_cast<unsigned>(ceil_div(n_windows, 8)), 256, 0, st>>>(
      u.as<double>(), items, win_off, row_off.as<int64_t>(), n_windows, rows, D, contrib.as<double>(),
      keys.as<int64_t>());
  LF_LAUNCHED();
  rc = sort_by_item(keys.as<int64_t>(), rows, catalog, sorted, item_off, st);
  if (rc) return rc;
  encoder_demb<<<static_cast<unsigned>(ceil_div(catalog, 8)), 256, 0, st>>>(
      contrib.as<double>(), sorted.as<uint32_t>(), item_off.as<uint32_t>(), catalog, rows, D, d_emb);
  LF_LAUNCHED();
  return LF_OK;
}

}  // namespace lf
