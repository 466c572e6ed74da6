// lseforge_shim.cpp — the C++ drop-in for the reference's loss hot path.
//
// Defines, with the reference's exact signatures, the functions a maintainer
// would otherwise get from proj/src/cce.cpp and proj/src/ccem.cpp:
//
//   lseforge::cce_forward          cce.hpp:36-38   (reference cce.cpp:65-145)
//   lseforge::cce_backward         cce.hpp:51-54   (reference cce.cpp:147-272)
//   lseforge::ccem_forward         ccem.hpp:19-20  (reference ccem.cpp:48-105)
//   lseforge::ccem_backward        ccem.hpp:27-29  (reference ccem.cpp:196-205)
//   lseforge::ccem_backward_rows   ccem.hpp:34-36  (reference ccem.cpp:107-194)
//   lseforge::estimate_flops       ccem.hpp:48-49  (reference ccem.cpp:207-235)
//   lseforge::evaluate             metrics.hpp:18-24 (reference metrics.cpp:13-103)
//   lseforge::sample_uniform,      sampler.hpp:26-40 (reference sampler.cpp:30-127,
//     sample_popularity,           index for index — popularity: for exponent 1
//     PopularityTable::FromCounts  (exact integer sums); other exponents agree to
//                                  the device pow's last ulp; FromCounts is
//                                  restated on the host)
//
// It is compiled against the reference's own headers (-I proj/include) and
// linked in place of cce.cpp + ccem.cpp + metrics.cpp + sampler.cpp; everything else in liblseforge
// (losses.cpp validation and oracles, neg_index.cpp, accountant.cpp, the
// trainer) is unchanged.  Each call: validate on the host with the
// reference's own functions and messages -> upload the host matrices ->
// convert layouts on the device (ref-C D x V float -> E V x D) -> run the
// B200 kernels through the C-ABI (include/lseforge_b200.h) -> convert the
// gradients back (dE -> d_classifier D x V double) -> download.  Synchronous
// and blocking, like the reference.  No CPU fallback: a missing GPU or a
// kernel error throws.
//
// Element type of the device computation: environment LSEFORGE_B200_DTYPE =
//   f64  (default) exact mode — fp64 kernels in the reference's operand order,
//        pos_logits bitwise equal to the reference's double results;
//   f32  fp32 FFMA kernels;
//   bf16 tcgen05 tensor-core kernels (inputs rounded to bf16, d % 64 == 0).
// CceConfig::row_block / col_block / workers are CPU tiling knobs: validated
// exactly as the reference does, otherwise ignored (the device results never
// depend on them, which is the reference's own worker-invariance contract,
// README.md:149-153).
//
// Memory accounting: the "retained/..." tags are charged exactly as the
// reference charges them (cce.cpp:79-84, ccem.cpp:64-69, ccem.cpp:132-137);
// the "scratch/..." tags are charged with the library's real device scratch
// high-water mark for the call, in 4-byte scalars, and released before
// returning.  The reference's CPU tile-scratch closed form
// (memory_model.cpp:46-60) does not describe the GPU and is not imitated.
#include <cuda_runtime.h>
#include <malloc.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <limits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "lseforge/accountant.hpp"
#include "lseforge/backend.hpp"
#include "lseforge/cce.hpp"
#include "lseforge/ccem.hpp"
#include "lseforge/losses.hpp"
#include "lseforge/encoder.hpp"
#include "lseforge/matrix.hpp"
#include "lseforge/metrics.hpp"
#include "lseforge/neg_index.hpp"
#include "lseforge/sampler.hpp"
#include "lseforge/split.hpp"
#include "lseforge/threads.hpp"
#include "lseforge_b200.h"

namespace lseforge {

namespace {

// LSEFORGE_B200_HOST_HEAP=keep: serve large host blocks from the heap and
// keep them there after free (glibc mallopt), so the d x v double gradient
// the reference signature returns every step (512 MB at cfg2) reuses
// already-mapped pages instead of faulting in fresh ones (~170 ms per step
// on the B200 box).  Process-wide, hence opt-in; off by default.
const bool g_host_heap = [] {
  const char* s = std::getenv("LSEFORGE_B200_HOST_HEAP");
  if (!s || std::strcmp(s, "keep") != 0) return false;
  mallopt(M_MMAP_THRESHOLD, 1 << 30);
  mallopt(M_TRIM_THRESHOLD, std::numeric_limits<int>::max());
  return true;
}();

[[noreturn]] void throw_status(int rc, const char* what) {
  const std::string msg = lf_last_error();
  if (rc == LF_EINVAL) throw std::invalid_argument(msg);
  if (rc == LF_ERUNTIME) throw std::runtime_error(msg);  // the reference's own text (e.g. sampler.cpp:22-27)
  throw std::runtime_error(std::string(what) + ": " + msg);
}

void check(int rc, const char* what) {
  if (rc != LF_OK) throw_status(rc, what);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("lseforge_b200 shim: ") + what + ": " + cudaGetErrorString(e));
}

int device_dtype() {
  const char* s = std::getenv("LSEFORGE_B200_DTYPE");
  if (!s || !*s || std::strcmp(s, "f64") == 0) return LF_F64;
  if (std::strcmp(s, "f32") == 0) return LF_F32;
  if (std::strcmp(s, "bf16") == 0) return LF_BF16;
  throw std::invalid_argument(std::string("LSEFORGE_B200_DTYPE must be f64, f32 or bf16, got ") + s);
}

std::size_t elem_bytes(int dtype) { return dtype == LF_F64 ? 8 : (dtype == LF_F32 ? 4 : 2); }
std::size_t grad_bytes(int dtype) { return dtype == LF_F64 ? 8 : 4; }

// Device buffer owned for the duration of one call, from the device's
// stream-ordered pool on the legacy stream every call here uses (the library
// keeps that pool resident, so repeated calls do not pay cudaMalloc again).
struct Dev {
  void* p = nullptr;
  explicit Dev(std::size_t bytes) {
    if (bytes) cuda_check(cudaMallocAsync(&p, bytes, nullptr), "cudaMallocAsync");
  }
  ~Dev() {
    if (p) cudaFreeAsync(p, nullptr);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// Host copies split over a few persistent threads (the pageable side of a
// transfer is host-memory bound; one thread cannot keep PCIe busy).
class CopyPool {
 public:
  explicit CopyPool(int parts) : parts_(parts) {
    for (int k = 1; k < parts_; ++k) workers_.emplace_back([this, k] { loop(k); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void copy(void* dst, const void* src, std::size_t len) {
    if (parts_ == 1 || len < (1u << 20)) {
      std::memcpy(dst, src, len);
      return;
    }
    {
      std::lock_guard<std::mutex> g(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      len_ = len;
      pending_ = parts_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    piece(0);
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [this] { return pending_ == 0; });
  }

 private:
  void piece(int k) {
    const std::size_t a = len_ * k / parts_, b = len_ * (k + 1) / parts_;
    std::memcpy(dst_ + a, src_ + a, b - a);
  }
  void loop(int k) {
    std::size_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      piece(k);
      {
        std::lock_guard<std::mutex> g(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  int parts_;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  std::size_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  std::size_t len_ = 0;
};

// Per-thread transfer engine: two pinned chunks; large copies are pipelined
// (the host fills / drains one chunk while the DMA engine moves the other),
// on the legacy stream the library calls of this file are ordered on.
class Xfer {
 public:
  static Xfer& get() {
    thread_local Xfer x;
    return x;
  }
  void h2d(void* dst, const void* src, std::size_t bytes) {
    if (bytes < kSmall) {
      cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "upload");
      return;
    }
    ready();
    int i = 0;
    for (std::size_t off = 0; off < bytes; off += kChunk, ++i) {
      const std::size_t len = std::min(kChunk, bytes - off);
      const int b = i & 1;
      cuda_check(cudaEventSynchronize(ev_[b]), "upload chunk reuse");
      pool_.copy(pin_[b], static_cast<const char*>(src) + off, len);
      cuda_check(cudaMemcpyAsync(static_cast<char*>(dst) + off, pin_[b], len, cudaMemcpyHostToDevice, nullptr),
                 "upload");
      cuda_check(cudaEventRecord(ev_[b], nullptr), "upload event");
    }
  }
  void d2h(void* dst, const void* src, std::size_t bytes) {
    if (bytes < kSmall) {
      cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "download");
      return;
    }
    ready();
    const std::size_t chunks = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](std::size_t i) {
      const std::size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
      cuda_check(cudaMemcpyAsync(pin_[i & 1], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost,
                                 nullptr),
                 "download");
      cuda_check(cudaEventRecord(ev_[i & 1], nullptr), "download event");
    };
    issue(0);
    for (std::size_t i = 0; i < chunks; ++i) {
      if (i + 1 < chunks) issue(i + 1);
      cuda_check(cudaEventSynchronize(ev_[i & 1]), "download chunk");
      const std::size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
      pool_.copy(static_cast<char*>(dst) + off, pin_[i & 1], len);
    }
  }
  ~Xfer() {
    if (pin_[0]) {
      cudaFreeHost(pin_[0]);
      cudaFreeHost(pin_[1]);
      cudaEventDestroy(ev_[0]);
      cudaEventDestroy(ev_[1]);
    }
  }

 private:
  static constexpr std::size_t kChunk = std::size_t(16) << 20;
  static constexpr std::size_t kSmall = std::size_t(1) << 20;
  Xfer() : pool_(std::max(1, std::min(8, static_cast<int>(std::thread::hardware_concurrency()) / 2))) {}
  void ready() {
    if (pin_[0]) return;
    for (int b = 0; b < 2; ++b) {
      cuda_check(cudaHostAlloc(&pin_[b], kChunk, cudaHostAllocDefault), "cudaHostAlloc");
      cuda_check(cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming), "cudaEventCreate");
      cuda_check(cudaEventRecord(ev_[b], nullptr), "cudaEventRecord");
    }
  }
  CopyPool pool_;
  void* pin_[2] = {nullptr, nullptr};
  cudaEvent_t ev_[2] = {};
};

void upload(void* dst, const void* src, std::size_t bytes) {
  if (bytes) Xfer::get().h2d(dst, src, bytes);
}
// synchronous on return, like the reference's host results
void download(void* dst, const void* src, std::size_t bytes) {
  if (bytes) Xfer::get().d2h(dst, src, bytes);
}

// The inputs of one loss call, resident on the device in kernel layout.
struct DeviceInputs {
  int dtype;
  std::size_t n, d, v;
  Dev X, E;
  DeviceInputs(const DenseMatrix& Eh, const DenseMatrix& Ch, int dt)
      : dtype(dt), n(Eh.rows()), d(Eh.cols()), v(Ch.cols()),
        X(n * d * elem_bytes(dt)), E(v * d * elem_bytes(dt)) {
    Dev stage(std::max(n * d, d * v) * sizeof(float));
    upload(stage.p, Eh.data().data(), n * d * sizeof(float));
    check(lf_convert_rows(stage.as<float>(), static_cast<int64_t>(n * d), dtype, X.p, nullptr),
          "lf_convert_rows");
    upload(stage.p, Ch.data().data(), d * v * sizeof(float));
    check(lf_classifier_to_items(stage.as<float>(), static_cast<int64_t>(d), static_cast<int64_t>(v),
                                 dtype, E.p, nullptr),
          "lf_classifier_to_items");
  }
};

lf_cce_config make_cfg(const CceConfig& cfg, int dtype) {
  lf_cce_config c{};
  c.filter_eps = cfg.filter_eps;
  c.dtype = dtype;
  c.flags = LF_FLAG_NONE;
  return c;
}

// cce.cpp:17-27 (same messages).
void validate_config(const CceConfig& cfg) {
  if (cfg.row_block < 1 || cfg.col_block < 1) {
    throw std::invalid_argument("CceConfig: block sizes must be >= 1 (row_block=" +
                                std::to_string(cfg.row_block) + ", col_block=" +
                                std::to_string(cfg.col_block) + ")");
  }
  if (!(cfg.filter_eps >= 0.0)) {
    throw std::invalid_argument("CceConfig: filter_eps must be >= 0, got " +
                                std::to_string(cfg.filter_eps));
  }
}

// ccem.cpp:16-31 (same messages); index checks by NegIndexMatrix::validate.
void validate_sampled_inputs(const DenseMatrix& E, const DenseMatrix& C,
                             const NegIndexMatrix& inds) {
  if (inds.rows() != E.rows()) {
    throw std::invalid_argument("fused sampled loss: " + std::to_string(inds.rows()) +
                                " candidate rows for " + std::to_string(E.rows()) +
                                " embedding rows");
  }
  if (E.rows() == 0) {
    throw std::invalid_argument("fused sampled loss: zero rows; the mean loss is undefined");
  }
  if (E.cols() != C.rows()) {
    throw std::invalid_argument("fused sampled loss: embedding width " + std::to_string(E.cols()) +
                                " does not match classifier height " + std::to_string(C.rows()));
  }
  inds.validate(C.cols());
}

// Charges the library's device scratch high-water of the enclosed calls.
struct ScratchCharge {
  MemAccountant* acct;
  const char* tag;
  uint64_t base = 0;
  ScratchCharge(MemAccountant* a, const char* t) : acct(a), tag(t) {
    if (!acct) return;
    lf_workspace_reset_peak();
    uint64_t cur = 0;
    lf_workspace_stats(&cur, &base);
  }
  void settle() {
    if (!acct) return;
    uint64_t cur = 0, peak = 0;
    lf_workspace_stats(&cur, &peak);
    const std::size_t scalars = static_cast<std::size_t>((peak - base + 3) / 4);
    if (scalars) {
      acct->record_alloc(tag, scalars);
      acct->record_free(tag, scalars);
    }
  }
};

LossOutput download_loss(const Dev& lse, const Dev& pos, const Dev& loss, std::size_t n) {
  LossOutput out;
  out.lse.resize(n);
  out.pos_logits.resize(n);
  download(out.lse.data(), lse.p, n * sizeof(double));
  download(out.pos_logits.data(), pos.p, n * sizeof(double));
  download(&out.loss, loss.p, sizeof(double));
  return out;
}

GradPair download_grads(const Dev& dX, const Dev& dE, int dtype, std::size_t n, std::size_t d,
                        std::size_t v) {
  GradPair g{DenseMatrixD(n, d), DenseMatrixD(d, v)};
  Dev wide(std::max(n * d, d * v) * sizeof(double));
  check(lf_widen_grad(dX.p, dtype, static_cast<int64_t>(n * d), wide.as<double>(), nullptr),
        "lf_widen_grad");
  download(g.d_embeddings.data().data(), wide.p, n * d * sizeof(double));
  check(lf_items_grad_to_classifier(dE.p, dtype, static_cast<int64_t>(v), static_cast<int64_t>(d),
                                    wide.as<double>(), nullptr),
        "lf_items_grad_to_classifier");
  download(g.d_classifier.data().data(), wide.p, d * v * sizeof(double));
  return g;
}

}  // namespace

LossOutput cce_forward(const DenseMatrix& E, const DenseMatrix& C, std::span<const std::int64_t> x,
                       const CceConfig& cfg, MemAccountant* acct) {
  validate_loss_inputs(E, C, x);
  validate_config(cfg);
  const std::size_t n = E.rows();
  if (acct) {
    acct->record_ensure("retained/cce/pos_logits", n);
    acct->record_ensure("retained/cce/lse", n);
  }
  ScratchCharge sc(acct, "scratch/cce/forward");
  const int dt = device_dtype();
  DeviceInputs in(E, C, dt);
  Dev tg(n * sizeof(int64_t)), lse(n * sizeof(double)), pos(n * sizeof(double)), loss(sizeof(double));
  upload(tg.p, x.data(), n * sizeof(int64_t));
  const lf_cce_config c = make_cfg(cfg, dt);
  check(lf_cce_forward(in.X.p, in.E.p, tg.as<int64_t>(), static_cast<int64_t>(n),
                       static_cast<int64_t>(in.d), static_cast<int64_t>(in.v), &c, lse.as<double>(),
                       pos.as<double>(), loss.as<double>(), nullptr),
        "lf_cce_forward");
  LossOutput out = download_loss(lse, pos, loss, n);
  sc.settle();
  return out;
}

CceBackwardResult cce_backward(const DenseMatrix& E, const DenseMatrix& C,
                               std::span<const std::int64_t> x, std::span<const double> lse,
                               double upstream, const CceConfig& cfg, MemAccountant* acct) {
  validate_loss_inputs(E, C, x);
  validate_config(cfg);
  if (lse.size() != E.rows()) {
    throw std::invalid_argument("cce_backward: LSE vector has " + std::to_string(lse.size()) +
                                " entries for " + std::to_string(E.rows()) + " rows");
  }
  const std::size_t n = E.rows(), d = E.cols(), v = C.cols();
  if (acct) acct->record_ensure("retained/cce/lse", n);
  ScratchCharge sc(acct, "scratch/cce/backward");
  const int dt = device_dtype();
  DeviceInputs in(E, C, dt);
  Dev tg(n * sizeof(int64_t)), dl(n * sizeof(double));
  Dev dX(n * d * grad_bytes(dt)), dE(v * d * grad_bytes(dt));
  upload(tg.p, x.data(), n * sizeof(int64_t));
  upload(dl.p, lse.data(), n * sizeof(double));
  const lf_cce_config c = make_cfg(cfg, dt);
  lf_cce_stats st{};
  check(lf_cce_backward(in.X.p, in.E.p, tg.as<int64_t>(), dl.as<double>(), upstream,
                        static_cast<int64_t>(n), static_cast<int64_t>(d), static_cast<int64_t>(v),
                        &c, dX.p, dE.p, &st, nullptr),
        "lf_cce_backward");
  CceBackwardResult out{download_grads(dX, dE, dt, n, d, v), st.skipped_fraction};
  sc.settle();
  return out;
}

LossOutput ccem_forward(const DenseMatrix& E, const DenseMatrix& C, const NegIndexMatrix& inds,
                        const CceConfig& cfg, MemAccountant* acct) {
  validate_sampled_inputs(E, C, inds);
  if (cfg.row_block < 1) throw std::invalid_argument("CceConfig: row_block must be >= 1");
  const std::size_t n = E.rows(), w = inds.width();
  if (acct) {
    acct->record_ensure("retained/ccem/pos_logits", n);
    acct->record_ensure("retained/ccem/lse", n);
    acct->record_ensure("retained/ccem/inds", n * w, ScalarKind::kIndex);
  }
  ScratchCharge sc(acct, "scratch/ccem/forward");
  const int dt = device_dtype();
  DeviceInputs in(E, C, dt);
  Dev ind(n * w * sizeof(int64_t)), lse(n * sizeof(double)), pos(n * sizeof(double)),
      loss(sizeof(double));
  upload(ind.p, inds.data().data(), n * w * sizeof(int64_t));
  const lf_cce_config c = make_cfg(cfg, dt);
  check(lf_ccem_forward(in.X.p, in.E.p, ind.as<int64_t>(), static_cast<int64_t>(n),
                        static_cast<int64_t>(in.d), static_cast<int64_t>(in.v),
                        static_cast<int64_t>(w), &c, lse.as<double>(), pos.as<double>(),
                        loss.as<double>(), nullptr),
        "lf_ccem_forward");
  LossOutput out = download_loss(lse, pos, loss, n);
  sc.settle();
  return out;
}

GradPair ccem_backward_rows(const DenseMatrix& E, const DenseMatrix& C, const NegIndexMatrix& inds,
                            std::span<const double> lse, std::span<const double> row_upstream,
                            const CceConfig& cfg, MemAccountant* acct) {
  validate_sampled_inputs(E, C, inds);
  if (cfg.row_block < 1) throw std::invalid_argument("CceConfig: row_block must be >= 1");
  const std::size_t n = E.rows(), d = E.cols(), v = C.cols(), w = inds.width();
  if (lse.size() != n) {
    throw std::invalid_argument("ccem_backward: LSE vector has " + std::to_string(lse.size()) +
                                " entries for " + std::to_string(n) + " rows");
  }
  if (row_upstream.size() != n) {
    throw std::invalid_argument("ccem_backward: upstream vector has " +
                                std::to_string(row_upstream.size()) + " entries for " +
                                std::to_string(n) + " rows");
  }
  if (acct) {
    acct->record_ensure("retained/ccem/lse", n);
    acct->record_ensure("retained/ccem/inds", n * w, ScalarKind::kIndex);
  }
  ScratchCharge sc(acct, "scratch/ccem/backward");
  const int dt = device_dtype();
  DeviceInputs in(E, C, dt);
  Dev ind(n * w * sizeof(int64_t)), dl(n * sizeof(double)), up(n * sizeof(double));
  Dev dX(n * d * grad_bytes(dt)), dE(v * d * grad_bytes(dt));
  upload(ind.p, inds.data().data(), n * w * sizeof(int64_t));
  upload(dl.p, lse.data(), n * sizeof(double));
  upload(up.p, row_upstream.data(), n * sizeof(double));
  const lf_cce_config c = make_cfg(cfg, dt);
  check(lf_ccem_backward(in.X.p, in.E.p, ind.as<int64_t>(), dl.as<double>(), up.as<double>(), 0.0,
                         static_cast<int64_t>(n), static_cast<int64_t>(d), static_cast<int64_t>(v),
                         static_cast<int64_t>(w), &c, dX.p, dE.p, nullptr),
        "lf_ccem_backward");
  GradPair g = download_grads(dX, dE, dt, n, d, v);
  sc.settle();
  return g;
}

GradPair ccem_backward(const DenseMatrix& E, const DenseMatrix& C, const NegIndexMatrix& inds,
                       std::span<const double> lse, double upstream, const CceConfig& cfg,
                       MemAccountant* acct) {
  const std::size_t n = E.rows();
  if (n == 0) {
    throw std::invalid_argument("fused sampled loss: zero rows; the mean loss is undefined");
  }
  // ccem.cpp:203: the scalar form is the per-row form with upstream / N.
  std::vector<double> row_upstream(n, upstream / static_cast<double>(n));
  return ccem_backward_rows(E, C, inds, lse, row_upstream, cfg, acct);
}

FlopEstimate estimate_flops(std::size_t n, std::size_t d, std::size_t v, std::size_t ns,
                            Backend backend) {
  FlopEstimate f;
  const int rc = lf_estimate_flops(static_cast<int64_t>(n), static_cast<int64_t>(d),
                                   static_cast<int64_t>(v), static_cast<int64_t>(ns),
                                   static_cast<int32_t>(backend), &f.forward, &f.backward);
  if (rc != LF_OK) throw_status(rc, "lf_estimate_flops");
  return f;
}

PopularityTable PopularityTable::FromCounts(std::vector<std::int64_t> counts) {
  // sampler.cpp:30-42: reject negative counts, keep the total
  PopularityTable t;
  for (std::size_t v = 0; v < counts.size(); ++v) {
    if (counts[v] < 0)
      throw std::invalid_argument("PopularityTable: item " + std::to_string(v) + " has negative count " +
                                  std::to_string(counts[v]));
    t.total += counts[v];
  }
  t.counts = std::move(counts);
  return t;
}

namespace {
NegIndexMatrix download_inds(const Dev& d, std::size_t n, std::size_t w) {
  std::vector<int64_t> h(n * w);
  download(h.data(), d.p, sizeof(int64_t) * n * w);
  NegIndexMatrix m(n, w);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t s = 0; s < w; ++s) m(i, s) = h[i * w + s];
  return m;
}
}  // namespace

NegIndexMatrix sample_uniform(std::span<const std::int64_t> positives, std::size_t ns, std::size_t catalog,
                              const SplitMix64& rng, const SamplerConfig& cfg) {
  // rows draw from rng.derived(i), which depends only on the construction seed
  const std::size_t n = positives.size();
  Dev pos(n * 8), out(n * (1 + ns) * 8);
  upload(pos.p, positives.data(), n * 8);
  check(lf_sample_uniform(pos.as<int64_t>(), static_cast<int64_t>(n), static_cast<int64_t>(ns),
                          static_cast<int64_t>(catalog), rng.seed(), cfg.retry_cap, out.as<int64_t>(), nullptr),
        "lf_sample_uniform");
  return download_inds(out, n, 1 + ns);
}

NegIndexMatrix sample_popularity(std::span<const std::int64_t> positives, std::size_t ns,
                                 const PopularityTable& pop, const SplitMix64& rng, const SamplerConfig& cfg) {
  const std::size_t n = positives.size(), catalog = pop.counts.size();
  if (catalog == 0) throw std::invalid_argument("sample_popularity: empty popularity table");
  Dev pos(n * 8), counts(catalog * 8), out(n * (1 + ns) * 8);
  upload(pos.p, positives.data(), n * 8);
  upload(counts.p, pop.counts.data(), catalog * 8);
  check(lf_sample_popularity(pos.as<int64_t>(), static_cast<int64_t>(n), static_cast<int64_t>(ns),
                             counts.as<int64_t>(), static_cast<int64_t>(catalog), cfg.popularity_exponent,
                             rng.seed(), cfg.retry_cap, out.as<int64_t>(), nullptr),
        "lf_sample_popularity");
  return download_inds(out, n, 1 + ns);
}

EvalSummary evaluate(const ToyEncoderParams& params, std::span<const EvalPair> pairs, std::size_t k,
                     const std::vector<std::int64_t>& popularity_counts, int workers) {
  // argument checks in the reference's order (metrics.cpp:16-25); the
  // popularity-table checks (metrics.cpp:26-33) run on the device with the
  // same messages
  if (pairs.empty()) throw std::invalid_argument("evaluate: no eval pairs");
  if (k == 0) throw std::invalid_argument("evaluate: k must be >= 1");
  const std::size_t v = params.catalog();
  if (popularity_counts.size() != v)
    throw std::invalid_argument("evaluate: popularity table size does not match the catalog");
  const std::size_t n = pairs.size(), d = params.hidden();
  // the encoder stays on the host (metrics.cpp:46): h for every pair
  std::vector<double> H(n * d);
  parallel_blocks(n, resolve_worker_count(workers), [&](std::size_t, std::size_t i) {
    const std::vector<double> h = encode(params, pairs[i].prefix);
    std::memcpy(H.data() + i * d, h.data(), sizeof(double) * d);
  });
  std::vector<std::int64_t> targets(n);
  for (std::size_t i = 0; i < n; ++i) targets[i] = pairs[i].target;

  const int dtype = device_dtype();
  Dev X(n * d * elem_bytes(dtype)), E(v * d * elem_bytes(dtype)), tg(n * 8), pop(v * 8);
  if (dtype == LF_F64) {
    upload(X.p, H.data(), n * d * sizeof(double));  // exact: the reference scores in double
  } else {
    std::vector<float> Hf(H.begin(), H.end());
    Dev stage(n * d * sizeof(float));
    upload(stage.p, Hf.data(), n * d * sizeof(float));
    check(lf_convert_rows(stage.as<float>(), static_cast<int64_t>(n * d), dtype, X.p, nullptr),
          "lf_convert_rows");
  }
  {
    Dev stage(d * v * sizeof(float));
    upload(stage.p, params.c.data().data(), d * v * sizeof(float));
    check(lf_classifier_to_items(stage.as<float>(), static_cast<int64_t>(d), static_cast<int64_t>(v),
                                 dtype, E.p, nullptr),
          "lf_classifier_to_items");
  }
  upload(tg.p, targets.data(), n * 8);
  upload(pop.p, popularity_counts.data(), v * 8);
  double out3[3];
  check(lf_evaluate(X.p, E.p, tg.as<int64_t>(), static_cast<int64_t>(n), static_cast<int64_t>(d),
                    static_cast<int64_t>(v), static_cast<int32_t>(std::min<std::size_t>(k, 1u << 30)),
                    dtype, pop.as<int64_t>(), out3, nullptr),
        "lf_evaluate");
  EvalSummary out;
  out.ndcg = out3[0];
  out.coverage = out3[1];
  out.surprisal = out3[2];
  return out;
}

}  // namespace lseforge
