// test_sharded.cpp — catalog sharding from C++ through the C-ABI, no PyTorch
// (TEST INFRASTRUCTURE; run by tests/test_sharded_cpp_gpu.py).
//
//   test_sharded peer W   fork W ranks that share GPU 0 (CUDA IPC between
//                         processes on one device is the same mapped-pointer
//                         path as across NVLink peers), exchange the peer
//                         communicator's handles through files, and shard
//                         the catalog W ways
//   test_sharded nccl1    one rank with a size-1 NCCL communicator
//                         (lf_comm_nccl on the real libnccl; two NCCL ranks
//                         cannot share one GPU)
//
// Every rank also runs the unsharded call on the full catalog and checks the
// sharded results against it: pos bitwise (the target logit comes from the
// same MMA inputs), lse / loss to fp32 rounding of the partial sums, dX and
// the shard's dE rows normwise, the skip statistics summed over ranks.
// Reference caller being replaced: run_loss_layer (proj/src/trainer.cpp:71-77).
#include <cuda_runtime.h>
#include <nccl.h>
#include <sys/stat.h>
#include <sys/wait.h>
#include <unistd.h>

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "lseforge_b200.h"

namespace {

int g_fail = 0;
#define CHECK(cond, ...)                       \
  do {                                         \
    if (!(cond)) {                             \
      std::printf("  FAIL: " __VA_ARGS__);     \
      std::printf("\n");                       \
      ++g_fail;                                \
    }                                          \
  } while (0)
#define LF(call)                                                                       \
  do {                                                                                 \
    int _rc = (call);                                                                  \
    if (_rc) {                                                                         \
      std::printf("  lf error %d in %s: %s\n", _rc, #call, lf_last_error());           \
      std::exit(3);                                                                    \
    }                                                                                  \
  } while (0)
#define CU(call)                                                                       \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess) {                                                           \
      std::printf("  cuda error in %s: %s\n", #call, cudaGetErrorString(_e));          \
      std::exit(3);                                                                    \
    }                                                                                  \
  } while (0)

struct SplitMix {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

uint16_t bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

struct Problem {
  int64_t n, d, v;
  int dtype;  // LF_BF16 or LF_F32
  double eps;
  std::vector<uint16_t> Xb, Eb;  // bf16
  std::vector<float> Xf, Ef;     // f32
  std::vector<int64_t> t;
};

Problem make_problem(uint64_t seed, int64_t n, int64_t d, int64_t v, int dtype, double eps) {
  Problem p{n, d, v, dtype, eps, {}, {}, {}, {}, {}};
  SplitMix r{seed};
  auto fill = [&](std::vector<uint16_t>& b, std::vector<float>& f, int64_t cnt) {
    b.resize(cnt);
    f.resize(cnt);
    for (int64_t i = 0; i < cnt; ++i) {
      const float x = static_cast<float>(2.0 * r.uniform() - 1.0);
      b[i] = bf16_rne(x);
      f[i] = x;
    }
  };
  fill(p.Xb, p.Xf, n * d);
  fill(p.Eb, p.Ef, v * d);
  p.t.resize(n);
  for (int64_t i = 0; i < n; ++i) p.t[i] = static_cast<int64_t>(r.next() % static_cast<uint64_t>(v));
  return p;
}

struct Out {
  std::vector<double> lse, pos;
  double loss = 0;
  std::vector<float> dX, dE;
};

struct Dev {
  void* X = nullptr;
  void* E = nullptr;
  int64_t* t = nullptr;
  double *lse = nullptr, *pos = nullptr, *loss = nullptr;
  float *dX = nullptr, *dE = nullptr;
};

size_t esize(int dtype) { return dtype == LF_BF16 ? 2 : 4; }

Dev upload(const Problem& p, int64_t v0, int64_t vs) {
  Dev g;
  const size_t es = esize(p.dtype);
  CU(cudaMalloc(&g.X, p.n * p.d * es));
  CU(cudaMalloc(&g.E, vs * p.d * es));
  CU(cudaMalloc(&g.t, p.n * 8));
  CU(cudaMalloc(&g.lse, p.n * 8));
  CU(cudaMalloc(&g.pos, p.n * 8));
  CU(cudaMalloc(&g.loss, 8));
  CU(cudaMalloc(&g.dX, p.n * p.d * 4));
  CU(cudaMalloc(&g.dE, vs * p.d * 4));
  const void* xs = p.dtype == LF_BF16 ? static_cast<const void*>(p.Xb.data()) : p.Xf.data();
  const unsigned char* es0 = p.dtype == LF_BF16 ? reinterpret_cast<const unsigned char*>(p.Eb.data())
                                                 : reinterpret_cast<const unsigned char*>(p.Ef.data());
  CU(cudaMemcpy(g.X, xs, p.n * p.d * es, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(g.E, es0 + v0 * p.d * es, vs * p.d * es, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(g.t, p.t.data(), p.n * 8, cudaMemcpyHostToDevice));
  return g;
}

Out download(const Problem& p, const Dev& g, int64_t vs) {
  Out o;
  o.lse.resize(p.n);
  o.pos.resize(p.n);
  o.dX.resize(p.n * p.d);
  o.dE.resize(vs * p.d);
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(o.lse.data(), g.lse, p.n * 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(o.pos.data(), g.pos, p.n * 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(&o.loss, g.loss, 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(o.dX.data(), g.dX, p.n * p.d * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(o.dE.data(), g.dE, vs * p.d * 4, cudaMemcpyDeviceToHost));
  return o;
}

void release(Dev& g) {
  for (void* q : {g.X, g.E, static_cast<void*>(g.t), static_cast<void*>(g.lse), static_cast<void*>(g.pos),
                  static_cast<void*>(g.loss), static_cast<void*>(g.dX), static_cast<void*>(g.dE)})
    cudaFree(q);
}

double normwise(const float* a, const float* b, int64_t cnt) {
  double num = 0, den = 0;
  for (int64_t i = 0; i < cnt; ++i) {
    num += (double(a[i]) - b[i]) * (double(a[i]) - b[i]);
    den += double(b[i]) * b[i];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

// One configuration: unsharded reference, then this rank's shard.
void run_case(const char* name, const Problem& p, const lf_comm& comm, bool fused_api) {
  const int W = comm.world, R = comm.rank;
  const int64_t v0 = p.v * R / W, v1 = p.v * (R + 1) / W, vs = v1 - v0;
  lf_cce_config cfg{p.eps, p.dtype, 0};
  // unsharded reference on the full catalog
  Dev full = upload(p, 0, p.v);
  lf_cce_stats fst{};
  LF(lf_cce_forward_backward(full.X, full.E, full.t, p.n, p.d, p.v, 1.0, &cfg, full.lse, full.pos, full.loss,
                             full.dX, full.dE, &fst, nullptr));
  Out ref = download(p, full, p.v);
  release(full);
  // this rank's shard
  Dev sh = upload(p, v0, vs);
  lf_cce_stats sst{};
  if (fused_api) {
    LF(lf_cce_forward_backward_sharded(sh.X, sh.E, sh.t, p.n, p.d, vs, v0, p.v, 1.0, &cfg, &comm, sh.lse, sh.pos,
                                       sh.loss, sh.dX, sh.dE, &sst, nullptr));
  } else {
    LF(lf_cce_forward_sharded(sh.X, sh.E, sh.t, p.n, p.d, vs, v0, &cfg, &comm, sh.lse, sh.pos, sh.loss, nullptr));
    LF(lf_cce_backward_sharded(sh.X, sh.E, sh.t, sh.lse, 1.0, p.n, p.d, vs, v0, p.v, &cfg, &comm, sh.dX, sh.dE,
                               &sst, nullptr));
  }
  Out got = download(p, sh, vs);
  release(sh);
  LF(lf_peer_comm_status());
  double lse_err = 0;
  bool pos_eq = true;
  for (int64_t i = 0; i < p.n; ++i) {
    lse_err = std::fmax(lse_err, std::fabs(got.lse[i] - ref.lse[i]) / std::fmax(1.0, std::fabs(ref.lse[i])));
    pos_eq &= got.pos[i] == ref.pos[i];
  }
  const double loss_err = std::fabs(got.loss - ref.loss) / std::fmax(1.0, std::fabs(ref.loss));
  const double dx_err = normwise(got.dX.data(), ref.dX.data(), p.n * p.d);
  const double de_err = normwise(got.dE.data(), ref.dE.data() + v0 * p.d, vs * p.d);
  const double sfrac = sst.skipped_fraction, ffrac = fst.skipped_fraction;
  std::printf("[rank %d/%d] %-26s lse %.2e loss %.2e pos %s dX %.2e dE %.2e skip %.6f/%.6f\n", R, W, name,
              lse_err, loss_err, pos_eq ? "bitwise" : "DIFF", dx_err, de_err, sfrac, ffrac);
  const bool bf = p.dtype == LF_BF16;
  CHECK(lse_err < 1e-5, "%s lse %.3e", name, lse_err);
  CHECK(loss_err < 1e-5, "%s loss %.3e", name, loss_err);
  CHECK(pos_eq, "%s pos not bitwise", name);
  CHECK(dx_err < (bf ? 5e-3 : 1e-5), "%s dX %.3e", name, dx_err);
  CHECK(de_err < (bf ? 5e-3 : 1e-5), "%s dE %.3e", name, de_err);
  CHECK(std::fabs(sfrac - ffrac) <= 1e-4, "%s skipped_fraction %.6f vs %.6f", name, sfrac, ffrac);
}

void run_all(const lf_comm& comm) {
  run_case("bf16 fused eps=0", make_problem(11, 1000, 64, 20000, LF_BF16, 0.0), comm, true);
  run_case("bf16 fused eps=6e-8", make_problem(12, 777, 64, 30011, LF_BF16, 6e-8), comm, true);
  run_case("bf16 fused d=128", make_problem(13, 300, 128, 9000, LF_BF16, 0.0), comm, true);
  run_case("bf16 eps=2^-8 (3-pass)", make_problem(14, 500, 64, 12000, LF_BF16, 0x1p-8), comm, true);
  run_case("f32 fwd+bwd phases", make_problem(15, 200, 64, 3001, LF_F32, 1e-6), comm, false);
}

int peer_rank(int W, int R, const std::string& dir) {
  CU(cudaSetDevice(0));
  const uint64_t slot = 1000ull * 128 * 4;  // the largest dX exchanged (n x d floats)
  lf_peer_comm* pc = nullptr;
  const uint64_t hb = lf_peer_comm_handle_bytes();
  std::vector<unsigned char> mine(hb), all(hb * W);
  LF(lf_peer_comm_create(slot, W, R, &pc, mine.data()));
  {
    const std::string tmp = dir + "/h" + std::to_string(R) + ".tmp", fin = dir + "/h" + std::to_string(R);
    std::ofstream(tmp, std::ios::binary).write(reinterpret_cast<const char*>(mine.data()), hb);
    std::rename(tmp.c_str(), fin.c_str());
  }
  for (int r = 0; r < W; ++r) {
    const std::string fin = dir + "/h" + std::to_string(r);
    for (int tries = 0;; ++tries) {
      std::ifstream f(fin, std::ios::binary);
      if (f && f.read(reinterpret_cast<char*>(all.data() + r * hb), hb)) break;
      if (tries > 6000) {
        std::printf("rank %d: no handle from rank %d\n", R, r);
        return 4;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(10));
    }
  }
  lf_comm comm{};
  LF(lf_peer_comm_open(pc, all.data(), &comm));
  run_all(comm);
  LF(lf_peer_comm_destroy(pc));
  return g_fail ? 1 : 0;
}

}  // namespace

int main(int argc, char** argv) {
  std::setvbuf(stdout, nullptr, _IOLBF, 0);  // the ranks' lines interleave whole
  const std::string mode = argc > 1 ? argv[1] : "peer";
  if (mode == "nccl1") {
    CU(cudaSetDevice(0));
    ncclComm_t nc;
    int dev = 0;
    if (ncclCommInitAll(&nc, 1, &dev) != ncclSuccess) {
      std::printf("ncclCommInitAll failed\n");
      return 3;
    }
    lf_comm comm{};
    LF(lf_comm_nccl(nc, 1, 0, &comm));
    run_all(comm);
    ncclCommDestroy(nc);
    std::printf("%s\n", g_fail ? "FAILED" : "OK");
    return g_fail ? 1 : 0;
  }
  const int W = argc > 2 ? std::atoi(argv[2]) : 2;
  char tmpl[] = "/tmp/lf_sharded_XXXXXX";
  const char* dir = mkdtemp(tmpl);
  if (!dir) return 3;
  std::vector<pid_t> kids;
  for (int r = 0; r < W; ++r) {  // no CUDA call in the parent before fork
    const pid_t pid = fork();
    if (pid == 0) {
      const int code = peer_rank(W, r, dir);
      std::fflush(stdout);
      std::_Exit(code);
    }
    kids.push_back(pid);
  }
  int worst = 0;
  for (pid_t k : kids) {
    int status = 0;
    waitpid(k, &status, 0);
    const int code = WIFEXITED(status) ? WEXITSTATUS(status) : 128;
    worst = code > worst ? code : worst;
  }
  std::printf("%s\n", worst ? "FAILED" : "OK");
  return worst;
}
