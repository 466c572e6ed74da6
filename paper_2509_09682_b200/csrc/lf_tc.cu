// lf_tc.cu — tcgen05 / TMEM / TMA kernels for the bf16 CCE path (sm_100a).
//
// One warp-specialized persistent kernel, three modes:
//   FWD       owner = 128 rows of X, stream = BN-item tiles of E.
//             S = X_o E_t^T in TMEM; epilogue does the online LSE (log2
//             domain) and the target-logit capture in registers; writes one
//             float4 partial {m, s, t, has} per (V-chunk, row)
//             (reference: cce_forward, cce.cpp:99-137).
//   BWD_ROWS  owner = rows, stream = items: S -> G = softmax*scale (-scale at
//             the target, 0 below the filter threshold) -> bf16 into TMEM ->
//             TS-MMA dX_o += G E_t (E_t reused from smem as an MN-major B
//             operand).  Pass 1 of cce_backward (cce.cpp:210-233).
//   BWD_ITEMS owner = items, stream = rows: S^T -> G^T -> dE_o += G^T X_t.
//             Pass 2 of cce_backward (cce.cpp:240-262).  No atomics: every
//             output row has one owner CTA.
//   EVAL      full-catalog ranking (metrics.cpp:46-78): owner = rows, stream =
//             items; each unit first multiplies the owner rows by their own
//             target items' rows (gathered) to get the target scores on the
//             same MMA datapath, then counts per row the items ranked ahead
//             of the target and keeps a per-row top-16 in registers.
//
// Roles: warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer (one
// elected lane), then NWG epilogue warpgroups that take stream tiles round
// robin, so the MUFU-bound epilogue of one tile overlaps the MMAs of the
// next ones.  Tile width BN and NWG are per mode (Geo below); the MMA warp
// runs NWG tiles ahead of the G read-back (lookahead), which needs
// NWG + 1 S buffers in TMEM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "lf_internal.cuh"
#include "lf_kernels.cuh"
#include "lf_ptx.cuh"

#ifndef LF_POLY_FWD
#define LF_POLY_FWD 0
#endif
#ifndef LF_COMMIT_ALWAYS
#define LF_COMMIT_ALWAYS 1  // backward: release a tile's stage / S buffer by tcgen05.commit even when every G MMA was filtered away
#endif
#ifndef LF_POLY_BWD
#define LF_POLY_BWD 4  // backward (fast filter domain): exps per 32 on the FMA pipe (packed), even
#endif
#ifndef LF_NOSCALE
#define LF_NOSCALE 1
#endif
#ifndef LF_NWG_FWD
#define LF_NWG_FWD 3
#endif
#ifndef LF_BN_FWD
#define LF_BN_FWD 128
#endif
#ifndef LF_SL_FWD
#define LF_SL_FWD 64  // forward epilogue slab (columns held in registers at once)
#endif
#ifndef LF_FWD_LD64
#define LF_FWD_LD64 1  // forward / EVAL: one 32x32b.x64 TMEM load per 64-column slab
#endif
#ifndef LF_FWD_MAXCHUNKS
#define LF_FWD_MAXCHUNKS 64  // forward: most V chunks pick_chunks may choose
#endif
#ifndef LF_EVAL_PIPE
#define LF_EVAL_PIPE 0  // EVAL: 1 = double-buffered 32-column TMEM loads, gate per 32 columns (measured 19.2 vs 13.9 ms at cfg2, k = 10)
#endif
#ifndef LF_EVAL_CONTIG
#define LF_EVAL_CONTIG 1  // EVAL: 1 CTA-contiguous owner-tile-major units, 2 phase-aligned rounds of owner tiles (see Units; E read ~once per round from HBM, measured slower), 0 chunk-major round robin
#endif
#ifndef LF_NWG_EVAL
#define LF_NWG_EVAL 2
#endif
#ifndef LF_BN_EVAL
#define LF_BN_EVAL 128  // EVAL stream tile (64: eight S buffers; the target-rows tile then spans two tiles)
#endif
#ifndef LF_BWD_LD64
#define LF_BWD_LD64 0  // backward: 64-column TMEM loads (two chunks), no prefetch
#endif
#ifndef LF_BWD_PREFETCH
#define LF_BWD_PREFETCH 1  // backward epilogue: double-buffered 32-column TMEM loads
#endif
#ifndef LF_NWG_BWD
#define LF_NWG_BWD 2
#endif
#ifndef LF_BN_BWD
#define LF_BN_BWD 128
#endif
#ifndef LF_NWG_FWDX
#define LF_NWG_FWDX 2
#endif
#ifndef LF_BN_FWDX
#define LF_BN_FWDX 128
#endif
#ifndef LF_FWDX_X2
#define LF_FWDX_X2 1  // FWDX: packed FFMA2 exponent arguments and an FADD2 tree for the row sum
#endif

namespace lf {

namespace {

constexpr int BM = 128;  // owner tile (TMEM lanes)

enum Mode : int { FWD = 0, BWD_ROWS = 1, BWD_ITEMS = 2, EVAL = 3, FWDX = 4 };
constexpr int kEvalK = 16;  // largest per-row top-K the EVAL epilogue keeps
// "no published k-th score yet" (the 0x80 byte-fill; below the key of any
// score above -3.4e38)
constexpr int kFloorNone = static_cast<int>(0x80808080u);
// EVAL list length by FLAGS (a shorter list for small k rises faster, so
// fewer slabs reach the insertion path): 0 -> 16, 1 -> 12, 2 -> 8, 3 -> 4
template <int MODE, int FLAGS>
constexpr int kEvalKOf = MODE != EVAL ? kEvalK : (FLAGS == 1 ? 12 : (FLAGS == 2 ? 8 : (FLAGS == 3 ? 4 : 16)));
// Backward variants: kFilt = filter_eps > 0 (flush below eps, sub-tile skip);
// kCount = also count skipped elements / sub-tiles (only when stats are read).
// kTgtIn = handle each row's own target inside the tile loop (exact for any
// eps, needed for the skip statistics); without it the target column is an
// ordinary softmax entry and the "-1" of softmax - onehot is applied at the
// accumulator read-out (dX_i -= scale E_{x_i}; dE_v -= scale sum_{x_i = v} X_i),
// which keeps the tile loop free of per-row branches.  The two differ only
// when the target's own softmax is below eps (then < eps relative), so the
// read-out form is used for eps < 2^-12 without stats.
constexpr int kFilt = 1, kCount = 2, kTgtIn = 4;

struct TcParams {
  int64_t n_owner;       // owner rows (n or v_shard)
  int64_t n_stream;      // stream rows (v_shard or n)
  int64_t owner_tiles;
  int64_t chunk;         // stream rows per unit (multiple of BN)
  int64_t n_chunks;
  int64_t c_first;       // EVAL: this launch's first chunk (the seeding pass took the ones before)
  int64_t units;
  const int32_t* tgt;    // FWD/BWD_ROWS: per owner row (local item or -1); BWD_ITEMS: per stream row
  const float* lse2;     // lse*log2e - log2|scale| per row (padded; +inf pad); FWDX: logit bound
  float abs_scale;       // |upstream / n| in the kernel's (possibly rescaled) G domain
  float out_scale;       // multiplies the dX / dE accumulators on read-out
  const __nv_bfloat16* fix_rows;  // !kTgtIn read-out: BWD_ROWS E, BWD_ITEMS X (bf16)
  float fix_scale;               // scale = upstream / n (signed, real units)
  const uint32_t* fix_off;       // BWD_ITEMS: [v + 2] offsets into fix_list per local item
  const uint32_t* fix_list;      // BWD_ITEMS: rows sorted by local target
  const float* tw;               // !kTgtIn: 1 - p_t per row (its target's softmax, full precision)
  const uint32_t* hit_off;       // BWD_ITEMS !kTgtIn: [item tiles + 1] offsets into hit_list
  const uint64_t* hit_list;      // rows grouped by their target's item tile, ascending
  float4* part;          // FWD: [n_chunks][n_owner]
  float* out;            // BWD_ROWS: [n_chunks][n_owner][D]; BWD_ITEMS: [n_owner][D]
  unsigned long long* counters;  // [0] skipped elems, [1] skipped tiles, [2] total tiles
  // EVAL (tgt = the target's local index clamped to [-1, n_stream]: -1 = before
  // the shard, n_stream = after it)
  uint32_t* ev_count;    // [n_chunks][n_owner] items of the chunk ranked ahead of the target
  float* ev_val;         // [n_chunks][n_owner][K] top scores, descending (K = kEvalKOf)
  int32_t* ev_idx;       // same, local item index (INT32_MAX = empty)
  int32_t* ev_floor;     // [owner rows] order-preserving bits of the best known k-th score
                         // (kFloorNone = none): runs of the same rows share it
};

// Position + phase in an N-slot mbarrier ring.
template <int N>
struct Ring {
  uint32_t i = 0, ph = 0;
  __device__ __forceinline__ void next() {
    if (++i == N) {
      i = 0;
      ph ^= 1;
    }
  }
};

// The dE pass's stream tile (rows) at width D: at D = 256 its accumulator
// takes half of TMEM, and 64-column S tiles leave four S buffers instead of
// two (measured: dE pass 19.4 -> 12.4 ms at the cfg5 shard shape; 64 columns
// are slower at D <= 128).
constexpr int bn_items(int D) { return D >= 256 ? 64 : LF_BN_BWD; }
// The fused forward + dX at D = 256: one epilogue warpgroup (its 256-column O
// accumulator is half of TMEM) on 64-column S tiles (four S buffers).  At
// D = 256 the tile's MMA work is four times D = 64's per logit, so one
// warpgroup's exps keep pace with the tensor pipe.
#ifndef LF_FWDX256_BN
#define LF_FWDX256_BN 64
#endif
#ifndef LF_FWDX128_NWG
#define LF_FWDX128_NWG LF_NWG_FWDX
#endif
constexpr int nwg_fwdx(int D) { return D >= 256 ? 1 : (D >= 128 ? LF_FWDX128_NWG : LF_NWG_FWDX); }
#ifndef LF_FWDX128_BN
#define LF_FWDX128_BN LF_BN_FWDX
#endif
constexpr int bn_fwdx(int D) { return D >= 256 ? LF_FWDX256_BN : (D >= 128 ? LF_FWDX128_BN : LF_BN_FWDX); }

template <int MODE, int D = 64>
struct Geo {
  static constexpr int BN = MODE == FWD    ? LF_BN_FWD
                            : MODE == FWDX ? bn_fwdx(D)
                            : MODE == EVAL ? LF_BN_EVAL
                            : MODE == BWD_ITEMS ? bn_items(D)
                                                : LF_BN_BWD;  // stream tile
  static constexpr int NWG = MODE == FWD    ? LF_NWG_FWD
                             : MODE == EVAL ? LF_NWG_EVAL
                             : MODE == FWDX ? nwg_fwdx(D)
                                            : LF_NWG_BWD;  // epilogue WGs
  // control warps: TMA producer, S-MMA issuer (+ the G-MMA issuer in the
  // backward and the fused forward)
  static constexpr int kCtrlWarps = MODE == FWD || MODE == EVAL ? 2 : 3;
  static constexpr int kThreads = 32 * kCtrlWarps + 128 * NWG;
  static constexpr int kEpiThreads = 128 * NWG;
  static constexpr int NQ = BN / 32;  // 32-column chunks per tile and thread
  static_assert(BN % 32 == 0 && BN >= 64 && (BN <= 128 || (MODE == FWD && BN == 256)), "BN");
};

template <int D, int MODE>
struct Cfg {
  using G = Geo<MODE, D>;
  static constexpr int BN = G::BN;
  static constexpr int kAtoms = D / 64;               // 128-byte K atoms per row
  static constexpr int kOwnerBytes = BM * D * 2;
  static constexpr int kTileBytes = BN * D * 2;
  // BWD_ITEMS stage extra: the stream rows' bias columns (BN rows x 16 bf16
  // = 32 B, SWIZZLE_32B) that fold -lse2 into the S MMA as a fifth K=16 step.
  static constexpr int kBiasOff = kTileBytes;
  static constexpr int kBiasBytes = BN * 32;
  static constexpr int kExtraBytes = MODE == BWD_ITEMS ? kBiasBytes : 0;
  static constexpr int kStageBytes = kTileBytes + kExtraBytes;
  static constexpr int kOnesBytes = MODE == BWD_ITEMS ? BM * 32 : 0;  // constant A bias columns
  // EVAL: per-row merge records {count, K values, K indices} (stride 2K + 1
  // words: conflict-free) of the other warpgroups + the shared target scores
  static constexpr int kEvalStride = 2 * kEvalK + 1;
  static constexpr int kEvalMerge = MODE == EVAL ? ((G::NWG - 1) * BM * kEvalStride + 2 * BM) * 4 : 0;
  static constexpr int kStagesFit = (200 * 1024 - kOwnerBytes - kOnesBytes - kEvalMerge) / kStageBytes;
  static constexpr int kStages = kStagesFit > 12 ? 12 : kStagesFit;
  // S buffers in TMEM; the rest holds the accumulators (one D-column O per
  // epilogue warpgroup in FWDX, one dX / dE tile in the backward)
  static constexpr int kNBMax =
      (MODE == FWD || MODE == EVAL ? 512 : (MODE == FWDX ? 512 - G::NWG * D : 512 - D)) / BN;
  static constexpr int kNB = kNBMax > 8 ? 8 : kNBMax;
  static_assert(MODE == FWD || MODE == EVAL || kNB >= 2, "not enough TMEM for the backward pipeline");
  // every epilogue warpgroup holds one S buffer while it works on a tile
  // (BN = 256 forward tiles with 3 warpgroups leave 2 buffers: measured to hang)
  static_assert(kNB >= G::NWG, "fewer TMEM S buffers than epilogue warpgroups");
  static constexpr int kAccCol = kNB * BN;
  static constexpr int kSmem = 1024 /*align slack*/ + kOwnerBytes + kOnesBytes + kStages * kStageBytes +
                               1024 /*barriers*/ +
                               (MODE == FWD ? (G::NWG - 1) * BM * 16 : (MODE == FWDX ? G::NWG * BM * 16 : 0)) +
                               kEvalMerge;
};
__device__ __forceinline__ float fma_log2(float v, float sub) { return fmaf(v, kLog2e, -sub); }

// Exp offload: of every 32 columns, the last POLY take 2^x on the FMA pipe
// (ex2_fma) and the rest on MUFU.  The clamp keeps ex2_fma in range; an
// argument above 127 still yields a huge value, so the forward's overflow
// rebase check fires exactly as with MUFU's +inf.
constexpr int kPolyFwd = LF_POLY_FWD;
// G domain of the filtered kernels.  Fast path (no kTgtIn): survivors of the
// ftz flush are >= 2^-126 and stay as they are (the tensor cores keep the
// tiny products exact enough: dX/dE errors are unchanged vs. the scaled
// domain, tools/filter_accuracy.py); the target's -1 is applied at read-out
// in real units.  kTgtIn puts (softmax - 1) x 2^-126 / eps into G, which for
// coarse eps is subnormal, so those kernels scale survivors by 2^64.
template <int FLAGS>
constexpr bool kNoScale = LF_NOSCALE != 0 && !(FLAGS & kTgtIn);
constexpr int kPolyBwd = LF_POLY_BWD;
#ifndef LF_POLY_FWDX
#define LF_POLY_FWDX 8  // fused forward: exps per 32 taken on the FMA pipe (packed), even
#endif
constexpr int kPolyFwdx = LF_POLY_FWDX;
template <int POLY>
__device__ __forceinline__ float ex2_mix(int c, float a) {
  if ((c & 31) >= 32 - POLY) return ex2_fma(fminf(fmaxf(a, -125.f), 127.f));
  return ex2_approx(a);
}

// Backward filter domain: the exp argument a = S log2e - lse2 is offset so
// that a < kThr (= -126) exactly when softmax < eps; ex2.approx.ftz flushes
// those results; the kTgtIn kernels then scale the survivors by 2^64 (kNoScale).
template <int FLAGS>
constexpr float kThr = -126.f;

// Backward coefficient of a row's own target column (never filtered).
template <int FLAGS>
__device__ __forceinline__ float target_g(float e, uint32_t raw, float l, float t_scale) {
  if (FLAGS & kFilt)
    return ex2_approx(fmaf(__uint_as_float(raw), kLog2e, -l) + (kNoScale<FLAGS> ? 0.f : 64.f)) - t_scale;
  return e - t_scale;
}

// Tree max of 32 registers, depth 4 with 3-input max (FMNMX3).
__device__ __forceinline__ float max32(const float (&e)[32]) {
  float a[11];
#pragma unroll
  for (int i = 0; i < 10; ++i) a[i] = fmaxf(e[3 * i], fmaxf(e[3 * i + 1], e[3 * i + 2]));
  a[10] = fmaxf(e[30], e[31]);
  float b[4];
#pragma unroll
  for (int i = 0; i < 3; ++i) b[i] = fmaxf(a[3 * i], fmaxf(a[3 * i + 1], a[3 * i + 2]));
  b[3] = fmaxf(a[9], a[10]);
  return fmaxf(fmaxf(b[0], b[1]), fmaxf(b[2], b[3]));
}

// Max of the first nv (<= 32) entries of 32 raw fp32 registers (-inf if none).
__device__ __forceinline__ float max32_valid(const uint32_t (&r)[32], int nv) {
  float e[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) e[c] = c < nv ? __uint_as_float(r[c]) : -INFINITY;
  return max32(e);
}

// Select r[idx] from a register array without dynamic indexing.
template <int N>
__device__ __forceinline__ float select_reg(const float (&r)[N], int idx) {
  float out = 0.f;
#pragma unroll
  for (int j = 0; j < N; ++j) out = (j == idx) ? r[j] : out;
  return out;
}
template <int N>
__device__ __forceinline__ uint32_t select_reg(const uint32_t (&r)[N], int idx) {
  uint32_t out = 0u;
#pragma unroll
  for (int j = 0; j < N; ++j) out = (j == idx) ? r[j] : out;
  return out;
}

// Rare path of the FWDX epilogue (a running-max rebase): multiply this
// warp's 32 TMEM lanes over `ncols` fp32 columns (the O accumulator) or
// `nwords` packed-bf16x2 columns (the tile's P already written) by each
// lane's own factor f.  Warp-collective (tcgen05.ld/st are .sync.aligned).
__device__ __noinline__ void tmem_scale_f32(uint32_t taddr, int ncols, float f) {
  for (int c0 = 0; c0 < ncols; c0 += 16) {
    uint32_t r[16];
    LF_TMEM_LD16(taddr + c0, r);
    tmem_ld_wait();
#pragma unroll
    for (int c = 0; c < 16; ++c) r[c] = __float_as_uint(__uint_as_float(r[c]) * f);
    LF_TMEM_ST16(taddr + c0, r);
  }
  tmem_st_wait();
}
__device__ __noinline__ void tmem_scale_bf16(uint32_t taddr, int nwords, float f) {
  for (int c0 = 0; c0 < nwords; c0 += 16) {
    uint32_t r[16];
    LF_TMEM_LD16(taddr + c0, r);
    tmem_ld_wait();
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const float lo = __uint_as_float(r[c] << 16), hi = __uint_as_float(r[c] & 0xffff0000u);
      r[c] = pack_bf16x2(lo * f, hi * f);
    }
    LF_TMEM_ST16(taddr + c0, r);
  }
  tmem_st_wait();
}

// Out-of-line paths of the FWDX epilogue (warp-collective; tcgen05.ld/st are
// .sync.aligned, so every lane of the warp calls them).  ta = the tile's S
// buffer at this warp's lanes, o_addr = this warpgroup's O accumulator.

// Rebase chunk q (valid columns nv) of the tile: lanes with `over` move their
// reference to the chunk's max; P chunk q is recomputed from S (still intact
// in TMEM), stored, and O and the P chunks already written are rescaled by
// f = 2^(m - m_new).  Returns {m_new, f, sum of the chunk's P}.
__device__ __noinline__ float4 fwdx_rebase(uint32_t ta, uint32_t o_addr, int D, int q, int nv, float m,
                                           bool over, int jt) {
  uint32_t r[32];
  LF_TMEM_LD32(ta + q * 32, r);
  tmem_ld_wait();
  float f = 1.f, nm = m;
  if (over) {
    nm = fmaxf(m, max32_valid(r, nv) * kLog2e);
    f = m == -INFINITY ? 0.f : ex2_approx(m - nm);
  }
  const float mr = nm == -INFINITY ? 0.f : nm;
  float x[32], a = 0.f;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    x[c] = c < nv ? ex2_approx(fma_log2(__uint_as_float(r[c]), mr)) : 0.f;
    a += x[c];
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) x[c] = c == jt ? 0.f : x[c];  // the target leaves O (see fwdx_dx)
  uint32_t g[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) g[c] = pack_bf16x2(x[2 * c], x[2 * c + 1]);
  LF_TMEM_ST16(ta + q * 16, g);
  tmem_st_wait();
  tmem_scale_f32(o_addr, D, f);
  if (q > 0) tmem_scale_bf16(ta, 16 * q, f);
  return make_float4(nm, f, a, 0.f);
}

// The target logit of rows whose target lies in this 128-column tile (read
// before P overwrites the S columns).
__device__ __noinline__ float2 fwdx_capture(uint32_t ta, int nq, int lc, float tv, float has) {
#pragma unroll 1
  for (int q = 0; q < nq; ++q) {
    const bool here = static_cast<unsigned>(lc - q * 32) < 32u;
    if (!__any_sync(0xffffffffu, here)) continue;
    uint32_t r[32];
    LF_TMEM_LD32(ta + q * 32, r);
    tmem_ld_wait();
    if (here) {
      tv = __uint_as_float(select_reg(r, lc - q * 32));
      has = 1.f;
    }
  }
  return make_float2(tv, has);
}

// The catalog's last, partial tile (nvalid < 128 columns): capture, masked
// max / P, rebase by max, store.  Returns the new {m, s, t, has}.
__device__ __noinline__ float4 fwdx_tile_tail(uint32_t ta, uint32_t o_addr, int D, int nq, int nvalid,
                                              int lc, float m, float s, float tv, float has) {
  const float2 t2 = fwdx_capture(ta, nq, lc, tv, has);
#pragma unroll 1
  for (int q = 0; q < nq; ++q) {
    const int nv = nvalid - q * 32;
    uint32_t r[32];
    LF_TMEM_LD32(ta + q * 32, r);
    tmem_ld_wait();
    const float mm = max32_valid(r, nv) * kLog2e;
    const bool over = mm > (m == -INFINITY ? -INFINITY : m + 64.f);
    const float4 o = fwdx_rebase(ta, o_addr, D, q, nv, m, over, lc - q * 32);
    m = o.x;
    s = fmaf(s, o.y, o.z);
  }
  return make_float4(m, s, t2.x, t2.y);
}

// Work units (chunk, owner tile).  FWD / backward: round robin over the
// grid, chunk-major.  EVAL: each CTA takes a contiguous range of units in
// owner-tile-major order, so consecutive units usually share the owner rows
// and the per-row top-k state carries over (see the EVAL epilogue).
//
// EVAL, phase-aligned (LF_EVAL_CONTIG = 2, when there are at least as many
// owner tiles as CTAs): u is a position in this CTA's own sequence.  Rounds
// of whole owner tiles first — CTA c takes owner r*grid + c through chunks
// 0..P-1 in order, so all CTAs stream the same region of E at the same time
// and E comes from HBM about once per round.  Then the remaining owner
// tiles' (owner, chunk) cells, split owner-major into one contiguous range
// per CTA (at most two runs: the tail of one owner tile, the head of the
// next) — each run carries its rows' state — processed head run first, so
// that at step t every CTA is at chunk t or t + (P - range): the CTAs stay
// within a window of E that fits L2.
template <int MODE>
struct Units {
  int64_t begin, end, step, P, OT;
  // EVAL phase-aligned: phase-A units, owner tiles in phase A, the phase-B
  // range's first owner / first chunk, its last owner, and the head run length
  int64_t A = 0, R0 = 0, bo = 0, bj = 0, lo = 0, hl = 0;
  int64_t cf = 0;  // EVAL: chunk offset of this launch (TcParams::c_first)
  bool aligned = false;
  __device__ Units(const TcParams& p) : P(p.n_chunks), OT(p.owner_tiles) {
    if (MODE == EVAL) {
      cf = p.c_first;
      P -= cf;
    }
    const int64_t G = gridDim.x, c = blockIdx.x;
    if (MODE == EVAL && LF_EVAL_CONTIG == 2 && OT >= G) {
      aligned = true;
      R0 = (OT / G) * G;
      A = (OT / G) * P;
      const int64_t cells = (OT - R0) * P;
      const int64_t b0 = c * cells / G, b1 = (c + 1) * cells / G;
      begin = 0;
      end = A + (b1 - b0);
      step = 1;
      if (b1 > b0) {
        bo = b0 / P;
        bj = b0 % P;
        lo = (b1 - 1) / P;  // == bo or bo + 1 (the range is shorter than one owner tile)
        hl = lo == bo ? 0 : (b1 - 1) % P + 1;
      }
    } else if (MODE == EVAL && LF_EVAL_CONTIG) {
      begin = c * p.units / G;
      end = (c + 1) * p.units / G;
      step = 1;
    } else {
      begin = c;
      end = p.units;
      step = G;
    }
  }
  __device__ int64_t chunk(int64_t u) const {
    if (MODE == EVAL && aligned) {
      if (u < A) return cf + u % P;
      const int64_t t = u - A;
      return cf + (t < hl ? t : bj + (t - hl));
    }
    return MODE == EVAL ? cf + (LF_EVAL_CONTIG ? u % P : u / OT) : u / OT;
  }
  __device__ int64_t owner(int64_t u) const {
    if (MODE == EVAL && aligned) {
      if (u < A) return (u / P) * gridDim.x + blockIdx.x;
      return R0 + (u - A < hl ? lo : bo);
    }
    return MODE == EVAL && LF_EVAL_CONTIG ? u / P : u % OT;
  }
};

// Largest float below x (finite x): "score >= x" == "score > next_down(x)".
__device__ __forceinline__ float next_down(float x) {
  if (x == 0.f) return __int_as_float(0x80000001);
  const int b = __float_as_int(x);
  return __int_as_float(x > 0.f ? b - 1 : b + 1);
}

// Insert (cv, ci) into a descending top-K list, ties to the smaller index
// (metrics.cpp:64-71 order); a no-op when it ranks below the K-th entry.
template <int K>
__device__ __forceinline__ void topk_insert(float (&kv)[K], int (&ki)[K], float cv, int ci) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool bt = cv > kv[k] || (cv == kv[k] && ci < ki[k]);
    const float t = kv[k];
    const int u = ki[k];
    kv[k] = bt ? cv : t;
    ki[k] = bt ? ci : u;
    cv = bt ? t : cv;
    ci = bt ? u : ci;
  }
}

template <int D, int MODE, int FLAGS>
__global__ void __launch_bounds__(Geo<MODE, D>::kThreads, 1)
    cce_tc_kernel(const __grid_constant__ CUtensorMap map_owner,
                  const __grid_constant__ CUtensorMap map_stream,
                  const __grid_constant__ CUtensorMap map_lsex,
                  const __grid_constant__ CUtensorMap map_ones, const TcParams p) {
  using C = Cfg<D, MODE>;
  using G = Geo<MODE, D>;
  constexpr int BN = G::BN;
  constexpr int NWG = G::NWG;
  constexpr int NQ = G::NQ;
  constexpr int KK = kEvalKOf<MODE, FLAGS>;  // EVAL: per-row list length
  constexpr int RS = 2 * KK + 1;             // EVAL: merge record stride (words)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1 KB alignment by plain pointer arithmetic on the __shared__ array, so
  // every pointer derived from `base` stays in the shared address space
  // (ordinary loads through it compile to LDS, not generic LD).
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* owner_smem = base;
  unsigned char* ones_smem = base + C::kOwnerBytes;  // BWD_ITEMS: [1,1,1,0..] per owner row
  unsigned char* stage_smem = base + C::kOwnerBytes + C::kOnesBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage_smem + C::kStages * C::kStageBytes);
  uint64_t* full = bars;                      // [kStages]
  uint64_t* empty = full + C::kStages;        // [kStages]
  uint64_t* s_full = empty + C::kStages;      // [kNB]
  uint64_t* s_empty = s_full + C::kNB;        // [kNB]
  uint64_t* g_ready = s_empty + C::kNB;       // [kNB]
  uint64_t* owner_full = g_ready + C::kNB;
  uint64_t* owner_empty = owner_full + 1;
  uint64_t* acc_full = owner_empty + 1;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* o_done = acc_empty + 1;           // [4] FWDX: a warpgroup's O MMAs completed (per tile)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_done + 4);
  // backward: per S buffer and epilogue warp, the 32-column chunks of G it did
  // NOT skip (bit q); warp 2 leaves out the G MMA K steps no warp needs
  uint32_t* live_mask = tmem_holder + 1;      // [kNB][4]
  float4* merge = reinterpret_cast<float4*>(reinterpret_cast<unsigned char*>(bars) + 1024);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < C::kNB; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], MODE == FWD || MODE == EVAL ? 4 : 1);  // one arrive per epilogue warp
      mbar_init(&g_ready[i], 4);
    }
    mbar_init(owner_full, 1);
    mbar_init(owner_empty, 1);
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4 * NWG);
    for (int i = 0; i < 4; ++i) mbar_init(&o_done[i], 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_owner);
    tma_prefetch_desc(&map_stream);
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      const uint64_t pol = policy_evict_normal();
      Ring<C::kStages> rs;
      uint32_t j = 0;
      const Units<MODE> U(p);
      for (int64_t u = U.begin; u < U.end; u += U.step, ++j) {
        const int64_t chunk = U.chunk(u), ot = U.owner(u);
        const int64_t s_begin = chunk * p.chunk;
        const int64_t s_end = min(p.n_stream, s_begin + p.chunk);
        mbar_wait(owner_empty, (j & 1) ^ 1);
        mbar_arrive_expect_tx(owner_full, C::kOwnerBytes + C::kOnesBytes);
#pragma unroll
        for (int a = 0; a < C::kAtoms; ++a)
          tma_load_2d(owner_smem + a * BM * 128, &map_owner, owner_full, a * 64,
                      static_cast<int32_t>(ot * BM), pol);
        if (MODE == BWD_ITEMS) tma_load_2d(ones_smem, &map_ones, owner_full, 0, 0, pol);
        if (MODE == EVAL) {
          // the owner rows' own target items (gathered, row-aligned with the
          // owner tile), BN rows per tile: BM / BN tiles
          for (int h = 0; h < BM / BN; ++h) {
            unsigned char* stg = stage_smem + rs.i * C::kStageBytes;
            mbar_wait(&empty[rs.i], rs.ph ^ 1);
            mbar_arrive_expect_tx(&full[rs.i], C::kTileBytes);
#pragma unroll
            for (int a = 0; a < C::kAtoms; ++a)
              tma_load_2d(stg + a * BN * 128, &map_lsex, &full[rs.i], a * 64,
                          static_cast<int32_t>(ot * BM + h * BN), pol);
            rs.next();
          }
        }
        for (int64_t s0 = s_begin; s0 < s_end; s0 += BN, rs.next()) {
          unsigned char* stg = stage_smem + rs.i * C::kStageBytes;
          mbar_wait(&empty[rs.i], rs.ph ^ 1);
          // BWD_ITEMS also stages the stream rows' bias columns.
          mbar_arrive_expect_tx(&full[rs.i], C::kTileBytes + (MODE == BWD_ITEMS ? C::kBiasBytes : 0));
#pragma unroll
          for (int a = 0; a < C::kAtoms; ++a)
            tma_load_2d(stg + a * BN * 128, &map_stream, &full[rs.i], a * 64,
                        static_cast<int32_t>(s0), pol);
          if (MODE == BWD_ITEMS)
            tma_load_2d(stg + C::kBiasOff, &map_lsex, &full[rs.i], 0, static_cast<int32_t>(s0), pol);
        }
      }
    }
  } else if (warp == 1) {
    // =========================== MMA issuer: S ===========================
    // S(t) = owner . stream(t)^T into S buffer b1.  Kept lean (ring cursors,
    // split descriptors): this warp shares its SM sub-partition with
    // epilogue warps.  In the backward the G.stream MMAs are issued by a
    // second warp, so the commit that frees an S buffer never tracks the S
    // MMA just issued here, and consecutive S MMAs never wait on each other.
    constexpr uint32_t idesc1 = idesc_bf16(BM, BN, 0, 0);
    constexpr uint32_t hi = umma_desc_hi_sw128(1024);
    const uint32_t a_lo = umma_desc_lo(smem_u32(owner_smem), 16);
    const uint32_t b_lo = umma_desc_lo(smem_u32(stage_smem), 16);
    // SWIZZLE_32B K-major operands of the bias step: rows of 32 B, 8-row
    // groups 256 B apart
    constexpr uint32_t hi32 = umma_desc_hi_sw32(256);
    const uint32_t ones_lo = umma_desc_lo(smem_u32(ones_smem), 16);
    Ring<C::kStages> s1;
    Ring<C::kNB> b1;
    uint32_t j = 0;
    unsigned long long tiles_seen = 0;
    const Units<MODE> U(p);
    for (int64_t u = U.begin; u < U.end; u += U.step, ++j) {
      const int64_t chunk = U.chunk(u);
      const int64_t s_begin = chunk * p.chunk;
      const int64_t s_end = min(p.n_stream, s_begin + p.chunk);
      const int ntile = static_cast<int>(ceil_div(s_end - s_begin, BN)) + (MODE == EVAL ? BM / BN : 0);
      mbar_wait(owner_full, j & 1);
      tc_fence_after();
      for (int i = 0; i < ntile; ++i, s1.next(), b1.next()) {
        mbar_wait(&full[s1.i], s1.ph);
        mbar_wait(&s_empty[b1.i], b1.ph ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t lo = b_lo + s1.i * (C::kStageBytes >> 4);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t koff = (kk >> 2) * (BM * 128) + (kk & 3) * 32;
            const uint32_t koffb = (kk >> 2) * (BN * 128) + (kk & 3) * 32;
            mma_ss(tmem + b1.i * BN, umma_desc(a_lo + (koff >> 4), hi),
                   umma_desc(lo + (koffb >> 4), hi), idesc1, kk > 0 ? 1u : 0u);
          }
          if (MODE == BWD_ITEMS) {
            // fifth K = 16 step: [1, 1, 1, 0..] (owner) x [c1, c2, c3, 0..] (stream
            // row), c1 + c2 + c3 = -lse2 ln 2 in three bf16 parts: S' = S - lse2 ln 2
            mma_ss(tmem + b1.i * BN, umma_desc(ones_lo, hi32), umma_desc(lo + (C::kBiasOff >> 4), hi32),
                   idesc1, 1u);
          }
          mma_commit(&s_full[b1.i]);
          if (MODE == FWD || MODE == EVAL) mma_commit(&empty[s1.i]);
        }
        __syncwarp();
        ++tiles_seen;
      }
      if (lane == 0) mma_commit(owner_empty);
      __syncwarp();
    }
    // 4 * NQ sub-tiles (4 warps x NQ column chunks) per 128 x BN tile
    if (lane == 0 && (MODE == BWD_ROWS || MODE == BWD_ITEMS) && (FLAGS & kCount))
      atomicAdd(&p.counters[2], 4ull * NQ * tiles_seen);
  } else if (G::kCtrlWarps == 3 && warp == 2) {
    // ============ MMA issuer: G . stream (backward) / P . stream (FWDX) ============
    // acc (dX_o or dE_o) += G(t) . stream(t): G is bf16 in S buffer b2, K step
    // kk (stream rows 16kk..16kk+15) at columns 8kk; B = the stream tile viewed
    // K(stream rows) x N(D), MN-major SW128: 16 rows = 2048 B per K step, 64-col
    // D atoms BN*128 B apart.  Its commits free the stage and the S buffer.
    // FWDX: every epilogue warpgroup has its own accumulator O_w (its own
    // running max), tile t goes to O_(t mod NWG), and one commit per tile tells
    // that warpgroup its O MMAs so far have completed (o_done, for rebases).
    constexpr uint32_t idesc2 = idesc_bf16(BM, D, 0, 1);
    constexpr uint32_t hi = umma_desc_hi_sw128(1024);
    const uint32_t b2_lo = umma_desc_lo(smem_u32(stage_smem), BN * 128);
    Ring<C::kStages> s2;
    Ring<C::kNB> b2;
    uint32_t j = 0;
    int tw2 = 0;  // FWDX: the tile's warpgroup, continuing across units like the epilogue's
    const Units<MODE> U(p);
    for (int64_t u = U.begin; u < U.end; u += U.step, ++j) {
      const int64_t chunk = U.chunk(u);
      const int64_t s_begin = chunk * p.chunk;
      const int64_t s_end = min(p.n_stream, s_begin + p.chunk);
      const int ntile = static_cast<int>(ceil_div(s_end - s_begin, BN));
      mbar_wait(acc_empty, (j & 1) ^ 1);
      uint32_t fresh = (1u << NWG) - 1u;  // accumulators not yet written in this unit
      for (int i = 0; i < ntile; ++i, s2.next(), b2.next()) {
        const int aw = MODE == FWDX ? tw2 : 0;
        mbar_wait(&g_ready[b2.i], b2.ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t lo = b2_lo + s2.i * (C::kStageBytes >> 4);
          // saturated-gradient filtering: a K step (16 stream rows) whose G
          // columns every epilogue warp skipped is all zeros — leave its MMA
          // out once the accumulator has been initialised
          uint32_t live = ~0u;
          if ((MODE == BWD_ROWS || MODE == BWD_ITEMS) && (FLAGS & kFilt)) {
            const uint32_t* lm = live_mask + b2.i * 4;
            live = lm[0] | lm[1] | lm[2] | lm[3];
          }
          bool init = !((fresh >> aw) & 1u);
          bool issued = false;
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            if (init && !((live >> (kk >> 1)) & 1u)) continue;
#ifndef LF_DIAG_NOMMA2
            mma_ts(tmem + C::kAccCol + aw * D, tmem + b2.i * BN + kk * 8, umma_desc(lo + kk * 128, hi),
                   idesc2, init ? 1u : 0u);
#endif
            init = true;
            issued = true;
          }
          if (issued || LF_COMMIT_ALWAYS) {
            // the stage and the S buffer are free once this tile's MMAs complete
            mma_commit(&empty[s2.i]);
            mma_commit(&s_empty[b2.i]);
          } else {
            // every K step filtered away: nothing reads them any more (the
            // epilogue's reads are ordered before g_ready) — release now
            mbar_arrive(&empty[s2.i]);
            mbar_arrive(&s_empty[b2.i]);
          }
          if (MODE == FWDX) mma_commit(&o_done[aw]);
        }
        fresh &= ~(1u << aw);
        if (MODE == FWDX) tw2 = tw2 + 1 == NWG ? 0 : tw2 + 1;
        __syncwarp();
      }
      if (lane == 0) mma_commit(acc_full);
      __syncwarp();
    }
  } else {
    // ============================== epilogue ==============================
    const int wg = (warp - G::kCtrlWarps) >> 2;  // takes tiles with t % NWG == wg
    const int quad = warp & 3;          // TMEM lane quadrant this warp may access
    const int lrow = quad * 32 + lane;  // owner row within the tile
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    unsigned long long skipped = 0, skipped_sub = 0;
    bool skip_on = true;  // backward: run the skipping variant on the next tile (warp-uniform)
    // This CTA's stream tiles before the current unit: tile T (counted over
    // the CTA's units) sits in S buffer T mod kNB (phase (T / kNB) & 1) and
    // belongs to epilogue warpgroup T mod NWG,
    // so a warpgroup steps straight from one of its tiles to the next.
    uint32_t T0 = 0;
    uint32_t k_tiles = 0;    // FWDX: tiles this warpgroup has handed to the O MMAs
    uint32_t j = 0;
    const Units<MODE> U(p);
    // EVAL state, carried across the consecutive units of one owner tile:
    // items ranked ahead of the target, running top-k
    uint32_t ecnt = 0;
    float kv[KK];
    int ki[KK];
    for (int64_t u = U.begin; u < U.end; u += U.step, ++j) {
      const int64_t chunk = U.chunk(u), ot = U.owner(u);
      const bool run_first = u == U.begin || U.owner(u - U.step) != ot;
      const bool run_last = u + U.step >= U.end || U.owner(u + U.step) != ot;
      const int64_t s_begin = chunk * p.chunk;
      const int64_t s_end = min(p.n_stream, s_begin + p.chunk);
      const int64_t ntile = ceil_div(s_end - s_begin, BN);
      const int64_t orow = ot * BM + lrow;
      const int o0 = static_cast<int>(ot * BM);
      int tgt = -1;
      float lse2 = 0.f;
      if (MODE != BWD_ITEMS) {
        tgt = p.tgt[orow];  // padded to owner_tiles*BM
        if (MODE == BWD_ROWS) lse2 = p.lse2[orow];
      }
      float m = -INFINITY, s = 0.f, tv = 0.f, has = 0.f;
      bool fast = false;  // FWDX: this warp's rows cannot overflow (set with m)
      // BWD_ITEMS read-out form: the rows whose target lies in this owner tile,
      // ascending, packed row << 7 | local target; hnext / hnext2 = the next
      // two (~0 when none is left), loaded a tile-walk ahead of their use;
      // hti = hnext's stream tile (the per-tile test is one 32-bit compare)
      uint32_t hptr = 0, hend = 0;
      uint64_t hnext = ~0ull, hnext2 = ~0ull;
      int hti = INT_MAX;
      auto hit_tile = [&](uint64_t h) {
        return h == ~0ull ? INT_MAX : static_cast<int>((static_cast<int64_t>(h >> 7) - s_begin) / BN);
      };
      if (MODE == BWD_ITEMS && !(FLAGS & kTgtIn)) {
        hptr = p.hit_off[ot];
        hend = p.hit_off[ot + 1];
        if (hptr < hend) hnext = p.hit_list[hptr];
        if (hptr + 1 < hend) hnext2 = p.hit_list[hptr + 1];
        hti = hit_tile(hnext);
      }
      float st = 0.f, st_dn = 0.f;  // EVAL: the row's target score
      bool cnt_fma = false;         // EVAL: rank count on the FMA pipe (see below)
      if (MODE == EVAL && run_first) {
        // Seed the list with placeholders just below the k-th score another
        // run of these rows has already published: at least k real items
        // score >= it, so nothing below it can make the final list, while
        // ties with it still enter (v > next_down(floor) == v >= floor).
        ecnt = 0;
        float seed = -INFINITY;
        if (orow < p.n_owner) {
          const int fk = __ldcg(p.ev_floor + orow);
          if (fk != kFloorNone) seed = next_down(__int_as_float(fk >= 0 ? fk : fk ^ 0x7fffffff));
        }
#pragma unroll
        for (int k = 0; k < KK; ++k) {
          kv[k] = seed;
          ki[k] = 0x7fffffff;
        }
      }
      constexpr int kPre = MODE == EVAL ? BM / BN : 0;  // EVAL: the target-rows tile(s) come first
      const int64_t i_first =
          MODE == EVAL ? 0 : static_cast<int64_t>((static_cast<uint32_t>(wg) + NWG - T0 % NWG) % NWG);
      // The loop's end test doubles as the BWD_ITEMS hit test: lim = the end
      // or the next hit's tile, whichever comes first, so a tile without a
      // hit pays nothing for it (a separate per-tile test measured +2 % of
      // the dE pass).
      int64_t lim = ntile + kPre;
      if (MODE == BWD_ITEMS && !(FLAGS & kTgtIn) && hti < lim) lim = hti;
      for (int64_t i = i_first;; i += (MODE == EVAL ? 1 : NWG)) {
        // BWD_ITEMS read-out form: tm[q] = this lane's target columns of
        // chunk q (its owner item is the target of those stream rows)
        bool tgt_tile = false;
        uint32_t tm[NQ];
        if (i >= lim) {
          if (i >= ntile + kPre) break;
          if (MODE == BWD_ITEMS && !(FLAGS & kTgtIn)) {
            const int ti = static_cast<int>(i - kPre);
#pragma unroll
            for (int q = 0; q < NQ; ++q) tm[q] = 0u;
            const int64_t col0 = s_begin + static_cast<int64_t>(ti) * BN;
            // hits in the other warpgroup's tiles (hti < ti) are passed over
            while (hti <= ti) {
              if (hti == ti) {
                const int c = static_cast<int>(static_cast<int64_t>(hnext >> 7) - col0);
                const uint32_t bit = lrow == static_cast<int>(hnext & 127u) ? 1u << (c & 31) : 0u;
#pragma unroll
                for (int q = 0; q < NQ; ++q) tm[q] |= q == (c >> 5) ? bit : 0u;
                tgt_tile = true;
              }
              ++hptr;
              hnext = hnext2;
              hnext2 = hptr + 1 < hend ? p.hit_list[hptr + 1] : ~0ull;
              hti = hit_tile(hnext);
            }
            lim = hti < ntile + kPre ? hti : ntile + kPre;
#ifdef LF_DIAG_NOMASK  // timing diagnostic only (wrong results): no target masking
            tgt_tile = false;
#endif
          }
        }
        const uint32_t T = T0 + static_cast<uint32_t>(i);
        const int tw = static_cast<int>(T % NWG);
        const uint32_t rbi = T % C::kNB, rbph = (T / C::kNB) & 1u;
        if (MODE == EVAL && kPre > 1 && i < kPre) {
          // BN < BM: target columns i BN .. i BN + BN - 1 in tile i; the warps
          // whose rows lie there read their diagonal, every warp of the owner
          // releases the buffer, and after the last such tile all epilogue
          // threads meet once (same double buffering by unit parity).
          float* st_sh = reinterpret_cast<float*>(merge) + (NWG - 1) * BM * C::kEvalStride + (j & 1) * BM;
          if (tw == wg) {
            const int b = static_cast<int>(rbi);
            mbar_wait(&s_full[b], rbph);
            tc_fence_after();
            const int c = quad * 32 - static_cast<int>(i) * BN;  // this warp's diagonal column
            if (c >= 0 && c < BN) {
              float d[32];
              LF_TMEM_LD32(tmem + lane_base + b * BN + c, reinterpret_cast<uint32_t*>(d));
              tmem_ld_wait();
              st_sh[lrow] = select_reg(d, lane);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[b]);
          }
          if (i + 1 == kPre) {
            named_bar_sync(2, G::kEpiThreads);
            st = st_sh[lrow];
            st_dn = next_down(st);
            cnt_fma = __all_sync(0xffffffffu, fabsf(st) >= 0x1p-60f && fabsf(st) < 0x1p27f);
          }
          continue;
        }
        if (MODE == EVAL && i == 0) {
          // S = owner rows x their target rows: the diagonal is each row's
          // target score, from the same MMA as the scores it is compared with.
          // The warpgroup that owns this tile publishes it to the others
          // (double-buffered by unit parity: a buffer is rewritten only after
          // every warpgroup has passed the next unit's handoff).
          float* st_sh = reinterpret_cast<float*>(merge) + (NWG - 1) * BM * C::kEvalStride + (j & 1) * BM;
          if (tw == wg) {
            const int b = static_cast<int>(rbi);
            mbar_wait(&s_full[b], rbph);
            tc_fence_after();
            float d[32];
            LF_TMEM_LD32(tmem + lane_base + b * BN + quad * 32, reinterpret_cast<uint32_t*>(d));
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[b]);
            st = select_reg(d, lane);
            st_sh[lrow] = st;
            named_bar_arrive(2, G::kEpiThreads);
          } else {
            named_bar_sync(2, G::kEpiThreads);
            st = st_sh[lrow];
          }
          st_dn = next_down(st);
          // the rank count's FMA-pipe form needs 2^-60 <= |st| < 2^27 in every
          // row of the warp (always, in practice); otherwise exact FSET compares
          cnt_fma = __all_sync(0xffffffffu, fabsf(st) >= 0x1p-60f && fabsf(st) < 0x1p27f);
          continue;
        }
        if (tw != wg) continue;
        const int b = static_cast<int>(rbi);
        const int64_t col0 = s_begin + (i - kPre) * BN;
        const int nvalid = static_cast<int>((s_end - col0 < BN ? s_end - col0 : BN));
        // BWD_ITEMS with in-loop targets: the stream rows' local targets (read
        // from global, in flight while this warp waits for the tile's S)
        int tpre[NQ];
        if (MODE == BWD_ITEMS && (FLAGS & kTgtIn)) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) tpre[q] = __ldg(p.tgt + col0 + q * 32 + lane);
        }
        mbar_wait(&s_full[b], rbph);
        tc_fence_after();
        const uint32_t ta = tmem + lane_base + b * BN;
        if (MODE == FWD) {
          // The tile in 128-column slabs, each entirely in registers (one
          // wait per slab); S goes back once the last slab is loaded.
          constexpr int SL = BN < LF_SL_FWD ? BN : LF_SL_FWD;
          const int lc = tgt - static_cast<int>(col0);
#pragma unroll
          for (int h = 0; h < BN / SL; ++h) {
          float v[SL];
          {
            uint32_t* r = reinterpret_cast<uint32_t*>(v);
#if LF_FWD_LD64
            if constexpr (SL % 64 == 0) {
#pragma unroll
              for (int q = 0; q < SL / 64; ++q) LF_TMEM_LD64(ta + h * SL + q * 64, (r + q * 64));
            } else
#endif
            {
#pragma unroll
              for (int q = 0; q < SL / 32; ++q) LF_TMEM_LD32(ta + h * SL + q * 32, (r + q * 32));
            }
            tmem_ld_wait();
          }
          if (h + 1 == BN / SL) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[b]);
          }
          if (nvalid < BN) {
#pragma unroll
            for (int c = 0; c < SL; ++c)
              if (h * SL + c >= nvalid) v[c] = -INFINITY;
          }
          if (static_cast<unsigned>(lc - h * SL) < static_cast<unsigned>(SL)) {
            tv = select_reg(v, lc - h * SL);
            has = 1.f;
          }
          if (m == -INFINITY) {
            float mx = v[0];
#pragma unroll
            for (int c = 1; c < SL; ++c) mx = fmaxf(mx, v[c]);
            if (mx == -INFINITY) continue;  // slab entirely past the catalog end
            m = mx * kLog2e;
          }
          float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
          for (int c = 0; c < SL; c += 2) {
            acc0 += ex2_mix<kPolyFwd>(c, fma_log2(v[c], m));
            acc1 += ex2_mix<kPolyFwd>(c + 1, fma_log2(v[c + 1], m));
          }
          float sum = acc0 + acc1;
          if (!(sum <= 1.8446744e19f)) {  // > 2^64 or NaN: rebase on the true max
            float mx = v[0];
#pragma unroll
            for (int c = 1; c < SL; ++c) mx = fmaxf(mx, v[c]);
            const float nm = fmaxf(m, mx * kLog2e);
            s *= ex2_approx(m - nm);
            m = nm;
            acc0 = 0.f;
            acc1 = 0.f;
#pragma unroll
            for (int c = 0; c < SL; c += 2) {
              acc0 += ex2_approx(fma_log2(v[c], m));
              acc1 += ex2_approx(fma_log2(v[c + 1], m));
            }
            sum = acc0 + acc1;
          }
          s += sum;
          }
        } else if (MODE == FWDX) {
          // ---- fused forward + dX.  P = 2^(S log2e - m) against this
          // warpgroup's running reference m: s += sum P is the forward's
          // online LSE (cce.cpp:111-126) and P, rounded to bf16 into the
          // already-read S columns (chunk q -> columns 16q..16q+15), feeds
          // the TS-MMA O_wg += P E_t that warp 2 issues — the softmax-weighted
          // item sum of dX, normalised by the combine once lse is known.  m is
          // the first chunk's max and only moves when a chunk's sum would pass
          // 2^64 (a logit ~44 nats above it): then s, the P chunks already
          // written and O_wg (after its MMAs so far complete) are rescaled.
          const int lc = tgt - static_cast<int>(col0);
          bool waited = k_tiles == 0;  // o_done of this warpgroup's previous tile consumed
          const uint32_t o_addr = tmem + lane_base + C::kAccCol + wg * D;
          if (nvalid < BN) {
            // the catalog's last, partial tile: out of line (masking)
            if (!waited) {
              mbar_wait(&o_done[wg], (k_tiles - 1) & 1);
              waited = true;
            }
            tc_fence_after();
            const float4 r = fwdx_tile_tail(ta, o_addr, D, NQ, nvalid, lc, m, s, tv, has);
            m = r.x;
            s = r.y;
            tv = r.z;
            has = r.w;
          } else {
            // a tile holding some row's target: capture the logit, and run the
            // CHECK body, which leaves the target entry out of P (the rare path)
            const bool tgt_tile = __any_sync(0xffffffffu, static_cast<unsigned>(lc) < static_cast<unsigned>(BN));
            if (tgt_tile) {
              const float2 r = fwdx_capture(ta, NQ, lc, tv, has);  // before P overwrites S
              tv = r.x;
              has = r.y;
            }
            uint32_t ra[32], rc2[32];
            LF_TMEM_LD32(ta, ra);
            tmem_ld_wait();
            if (m == -INFINITY) {  // this warpgroup's first tile of the unit
              float e[32];
#pragma unroll
              for (int c = 0; c < 32; ++c) e[c] = __uint_as_float(ra[c]);
              m = max32(e) * kLog2e;
              // no logit exceeds the Cauchy-Schwarz bound |x_i| max_j |e_j|, so
              // with m at most 64 below it no chunk sum can pass 2^64: such
              // warps run the tile body without the per-chunk overflow check.
              // The reference is raised toward bound - 64 by up to 60: the
              // row's max is >= the first chunk's, so nothing within 2^-66 of
              // it can fall under the ftz flush (m - 126), and rows whose
              // first chunk sits up to 124 below their bound (trained-like
              // rows: a dominant target) still take the fast body.
              m = fmaxf(m, fminf(p.lse2[orow] - 64.f, m + 60.f));
              fast = __all_sync(0xffffffffu, !(m < p.lse2[orow] - 64.f));
            }
            // CHECK: per-chunk overflow vote (rebase out of line); !CHECK:
            // straight-line code, chunk q's pack / store overlaps chunk q+1's exps
            auto body = [&](auto check_tag) {
              constexpr bool CHECK = decltype(check_tag)::value;
#pragma unroll
              for (int q = 0; q < NQ; ++q) {
                uint32_t(&cur)[32] = (q & 1) ? rc2 : ra;
                uint32_t(&nxt)[32] = (q & 1) ? ra : rc2;
                if (q + 1 < NQ) LF_TMEM_LD32(ta + (q + 1) * 32, nxt);
                float x[32];
#if LF_FWDX_X2
#pragma unroll
                for (int c = 0; c < 32; c += 2)
                  ffma2(x[c], x[c + 1], __uint_as_float(cur[c]), __uint_as_float(cur[c + 1]), kLog2e, kLog2e,
                        -m, -m);
#pragma unroll
                for (int c = 0; c < 32 - (CHECK ? 0 : kPolyFwdx); ++c) x[c] = ex2_approx(x[c]);
                if (!CHECK) {  // (branch-free body) the FMA-pipe share of the exps
#pragma unroll
                  for (int c = 32 - kPolyFwdx; c < 32; c += 2) ex2_poly_x2<0>(x[c], x[c + 1], x[c], x[c + 1]);
                }
                const float sum = sum32_x2(x);
#else
#pragma unroll
                for (int c = 0; c < 32; ++c) x[c] = ex2_approx(fma_log2(__uint_as_float(cur[c]), m));
                float a0 = 0.f, a1 = 0.f;
#pragma unroll
                for (int c = 0; c < 32; c += 2) {
                  a0 += x[c];
                  a1 += x[c + 1];
                }
                const float sum = a0 + a1;
#endif
                bool stored = false;
                if (CHECK) {
                  const bool over = !(sum <= 1.8446744e19f);  // > 2^64 or NaN
                  if (__any_sync(0xffffffffu, over)) {
                    // rare: move the reference; out of line, P chunk q stored there
                    if (q + 1 < NQ) tmem_ld_wait();
                    if (!waited) {
                      mbar_wait(&o_done[wg], (k_tiles - 1) & 1);
                      waited = true;
                    }
                    tc_fence_after();
                    const float4 r = fwdx_rebase(ta, o_addr, D, q, 32, m, over, lc - q * 32);
                    m = r.x;
                    s = fmaf(s, r.y, r.z);
                    stored = true;
                  }
                }
                if (CHECK && !stored) {
                  // the target entry leaves O (counted in s above; fwdx_dx adds
                  // -(1 - p_t) E_t back in full precision)
                  const int jt = lc - q * 32;
#pragma unroll
                  for (int c = 0; c < 32; ++c) x[c] = c == jt ? 0.f : x[c];
                }
                if (!stored) {
                  s += sum;
                  uint32_t g[16];
#pragma unroll
                  for (int c = 0; c < 16; ++c) g[c] = pack_bf16x2(x[2 * c], x[2 * c + 1]);
                  LF_TMEM_ST16(ta + q * 16, g);
                }
                if (q + 1 < NQ) tmem_ld_wait();
              }
            };
            if (fast && !tgt_tile) {
              body(std::false_type{});
            } else {
              body(std::true_type{});
              fast = __all_sync(0xffffffffu, !(m < p.lse2[orow] - 64.f));  // after a rebase
            }
          }
          tmem_st_wait();
#ifndef LF_DIAG_NO_ODONE  // timing diagnostic only (unsafe if a rebase happens)
          if (!waited) mbar_wait(&o_done[wg], (k_tiles - 1) & 1);
#endif
          ++k_tiles;
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&g_ready[b]);
        } else if (MODE == EVAL) {
          // ---- ranking (metrics.cpp:56-78).  An item ranks ahead of the
          // target if its score is higher, or equal with a smaller index: a
          // 64-column slab wholly before the target counts score >= st (as
          // > next_down(st)), one wholly after counts score > st, and the slab
          // holding the target compares per element.  The top-k list only
          // sees slabs whose max beats its k-th entry (rare after warm-up).
          // The slab loop stays rolled: the epilogue must fit the i-cache.
          const int lc = tgt - static_cast<int>(col0);
#if LF_EVAL_PIPE
          // 32-column chunks, double-buffered: chunk q+1's tcgen05.ld is in
          // flight while chunk q is counted and gated (the loop stays rolled,
          // two chunks per trip, for the i-cache).
          auto chunk32 = [&](float (&w)[32], int q) {
            if (nvalid - q * 32 < 32) {
#pragma unroll
              for (int c = 0; c < 32; ++c)
                if (q * 32 + c >= nvalid) w[c] = -INFINITY;
            }
            const int l = lc - q * 32;
            if (static_cast<unsigned>(l) < 32u) {
#pragma unroll
              for (int c = 0; c < 32; ++c) ecnt -= c < l ? set_ge(w[c], st) : (c > l ? set_gt(w[c], st) : 0u);
            } else {
              const float thr = l >= 32 ? st_dn : st;
              float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
              if (cnt_fma) {  // see the 64-column form below
                const float nk = -thr * 0x1p100f;
#pragma unroll
                for (int c = 0; c < 32; c += 8) {
#pragma unroll
                  for (int e = 0; e < 8; e += 2)
                    fadd2(f[e], f[e + 1], f[e], f[e + 1], fma_sat(w[c + e], 0x1p100f, nk),
                          fma_sat(w[c + e + 1], 0x1p100f, nk));
                }
              } else {
#pragma unroll
                for (int c = 0; c < 32; ++c) f[c & 7] += fset_gt(w[c], thr);
              }
              ecnt += static_cast<uint32_t>(((f[0] + f[1]) + (f[2] + f[3])) + ((f[4] + f[5]) + (f[6] + f[7])));
            }
#ifndef LF_DIAG_NOTOPK
            const float g = max32(w);
            if (g > kv[KK - 1]) {  // divergent, rare once the list has filled
              const float kth = kv[KK - 1];
              uint32_t msk = 0;
#pragma unroll
              for (int c = 0; c < 32; ++c) msk |= (w[c] > kth ? 1u : 0u) << c;
              const int base = static_cast<int>(col0) + q * 32;
              if ((msk & (msk - 1u)) == 0u) {  // the chunk max is the only candidate
                topk_insert(kv, ki, g, base + __ffs(static_cast<int>(msk)) - 1);
              } else {
                do {
                  const int c = __ffs(static_cast<int>(msk)) - 1;
                  msk &= msk - 1u;
                  const float cv = select_reg(w, c);
                  if (cv > kv[KK - 1]) topk_insert(kv, ki, cv, base + c);
                } while (msk);
              }
            }
#endif
          };
          float wa[32], wb[32];
          LF_TMEM_LD32(ta, reinterpret_cast<uint32_t*>(wa));
          tmem_ld_wait();
#pragma unroll 1
          for (int q = 0; q < BN / 32; q += 2) {
            LF_TMEM_LD32(ta + (q + 1) * 32, reinterpret_cast<uint32_t*>(wb));
            chunk32(wa, q);
            tmem_ld_wait();
            if (q + 2 < BN / 32) {
              LF_TMEM_LD32(ta + (q + 2) * 32, reinterpret_cast<uint32_t*>(wa));
            } else {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&s_empty[b]);
            }
            chunk32(wb, q + 1);
            if (q + 2 < BN / 32) tmem_ld_wait();
          }
#else
#pragma unroll 1
          for (int h = 0; h < BN / 64; ++h) {
            float w[2][32];
#if LF_FWD_LD64
            {
              uint32_t* r = reinterpret_cast<uint32_t*>(&w[0][0]);
              LF_TMEM_LD64(ta + h * 64, r);
            }
#else
            LF_TMEM_LD32(ta + h * 64, reinterpret_cast<uint32_t*>(w[0]));
            LF_TMEM_LD32(ta + h * 64 + 32, reinterpret_cast<uint32_t*>(w[1]));
#endif
            tmem_ld_wait();
            if (h + 1 == BN / 64) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&s_empty[b]);
            }
            if (nvalid - h * 64 < 64) {
#pragma unroll
              for (int g = 0; g < 2; ++g)
#pragma unroll
                for (int c = 0; c < 32; ++c)
                  if (h * 64 + g * 32 + c >= nvalid) w[g][c] = -INFINITY;
            }
            const int l = lc - h * 64;
            if (static_cast<unsigned>(l) < 64u) {
#pragma unroll
              for (int g = 0; g < 2; ++g)
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                  const int cc = g * 32 + c;
                  ecnt -= cc < l ? set_ge(w[g][c], st) : (cc > l ? set_gt(w[g][c], st) : 0u);
                }
            } else {
              const float thr = l >= 64 ? st_dn : st;
              if (cnt_fma) {
                // score > thr as sat(score 2^100 - thr 2^100) on the FMA pipe:
                // the exact difference of two distinct floats of which one
                // (thr) has 2^-60 <= |thr| < 2^27 is at least ulp(thr) >=
                // 2^-83, so the scaled difference is >= 2^17 (or +-inf) and
                // saturates to exactly 1.0; equal or lower scores give 0.0.
                // Summed in pairs with FADD2 — exact (<= 64).
                const float nk = -thr * 0x1p100f;
                // four independent FADD2 chains (8 deep per 64 columns)
                float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                  for (int c = 0; c < 32; c += 8) {
#pragma unroll
                    for (int e = 0; e < 8; e += 2)
                      fadd2(f[e], f[e + 1], f[e], f[e + 1], fma_sat(w[g][c + e], 0x1p100f, nk),
                            fma_sat(w[g][c + e + 1], 0x1p100f, nk));
                  }
                ecnt += static_cast<uint32_t>(((f[0] + f[1]) + (f[2] + f[3])) + ((f[4] + f[5]) + (f[6] + f[7])));
              } else {
                // 1.0f / 0.0f per compare (FSET.BF, ALU pipe) summed on the FMA
                // pipe: exact (<= 64), one ALU op per item
                float f[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                  for (int c = 0; c < 32; ++c) f[c & 3] += fset_gt(w[g][c], thr);
                ecnt += static_cast<uint32_t>((f[0] + f[1]) + (f[2] + f[3]));
              }
            }
#ifndef LF_DIAG_NOTOPK
            const float g0 = max32(w[0]), g1 = max32(w[1]);
            if (fmaxf(g0, g1) > kv[KK - 1]) {  // divergent, rare once the list has filled
              const float kth = kv[KK - 1];
              uint32_t m0 = 0, m1 = 0;
              if (g0 > kth) {
#pragma unroll
                for (int c = 0; c < 32; ++c) m0 |= (w[0][c] > kth ? 1u : 0u) << c;
              }
              if (g1 > kth) {
#pragma unroll
                for (int c = 0; c < 32; ++c) m1 |= (w[1][c] > kth ? 1u : 0u) << c;
              }
              unsigned long long msk = (static_cast<unsigned long long>(m1) << 32) | m0;
              const int base = static_cast<int>(col0) + h * 64;
              if ((msk & (msk - 1ull)) == 0ull) {  // the slab max is the only candidate
                topk_insert(kv, ki, fmaxf(g0, g1), base + __ffsll(static_cast<long long>(msk)) - 1);
              } else {
                do {
                  const int c = __ffsll(static_cast<long long>(msk)) - 1;
                  msk &= msk - 1ull;
                  const float cv = c < 32 ? select_reg(w[0], c) : select_reg(w[1], c - 32);
                  if (cv > kv[KK - 1]) topk_insert(kv, ki, cv, base + c);
                } while (msk);
              }
            }
#endif
          }
#endif
        } else {
          // ---- backward: G = softmax * |scale| (target: minus |scale|), bf16,
          // back into the same TMEM columns (chunk q -> columns 16q..16q+15,
          // already consumed by this warp).  Filtering (FILT): lse2 carries the
          // shift log2(eps) + 126, so a = S log2e - lse2 < -126 exactly when
          // softmax < eps and ex2.approx.ftz flushes those results to +0 — no
          // compare or select per element; (kTgtIn kernels) survivors are rescaled by 2^64 so
          // every bf16 G and every MMA product stays normal, and out_scale
          // undoes the factor on the accumulator.  A 32 x 32 sub-tile whose
          // largest a is below the threshold (and that holds no target) skips
          // its exps (warp vote).
#ifdef LF_DIAG_EPI
          {  // timing diagnostic only (wrong results): 1 = no TMEM traffic, 2 = ld + st only
            if (LF_DIAG_EPI == 2) {
              uint32_t r0[32];
#pragma unroll
              for (int q = 0; q < NQ; ++q) {
                LF_TMEM_LD32(ta + q * 32, r0);
                tmem_ld_wait();
                LF_TMEM_ST16(ta + q * 16, r0);
              }
              tmem_st_wait();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&g_ready[b]);
            continue;
          }
#endif
          const int lc_t = MODE == BWD_ROWS ? tgt - static_cast<int>(col0) : -1;
          // 32-column chunks, the next chunk's tcgen05.ld in flight while this
          // one is processed.  Two instantiations: TEST = false is straight-line
          // code across all chunks (no branch in front of the exps) and only
          // notes, off the critical path, whether some sub-tile was entirely
          // below the filter threshold; TEST = true also skips those sub-tiles'
          // exps (warp vote + branch).  The next tile uses TEST = true only
          // while skippable sub-tiles keep appearing (uniform logits — the
          // headline case — never have one).  Either way the result is exact:
          // the ftz flush zeroes every entry below eps.
          uint32_t live_bits = 0u;  // chunks of G this warp did not skip
          // The read-out form (!kTgtIn): each row's target entry leaves the
          // product (fwdx_dx / the read-out add -(1 - p_t) back in full
          // precision).  Tiles holding a target (~BN / tiles of the other side,
          // 1.6 % at cfg2) run the TEST body, which masks it in registers:
          // BWD_ROWS at column lc_t, BWD_ITEMS at the bits of tm[] (this lane's
          // owner item is the target of those stream rows, from the hit list).
#ifndef LF_DIAG_NOMASK
          if (MODE == BWD_ROWS && !(FLAGS & kTgtIn))
            tgt_tile = __any_sync(0xffffffffu, static_cast<unsigned>(lc_t) < static_cast<unsigned>(BN));
#endif
          auto process = [&](auto test_tag) -> bool {
          constexpr bool TEST = decltype(test_tag)::value;
          bool any_below = false;
#if LF_BWD_LD64
          uint32_t ra[64];  // two 32-column chunks per tcgen05.ld
          LF_TMEM_LD64(ta, ra);
#elif LF_BWD_PREFETCH
          uint32_t ra[32], rb[32];
          LF_TMEM_LD32(ta, ra);
#else
          uint32_t ra[32];
          LF_TMEM_LD32(ta, ra);
#endif
          tmem_ld_wait();
#ifdef LF_DIAG_EARLY  // timing diagnostic only (wrong results): hand G over before computing it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&g_ready[b]);
#endif
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
#if LF_BWD_LD64
            if (q > 0 && (q & 1) == 0) {
              LF_TMEM_LD64(ta + q * 32, ra);
              tmem_ld_wait();
            }
            uint32_t(&cur)[32] = *reinterpret_cast<uint32_t(*)[32]>(ra + (q & 1) * 32);
#elif LF_BWD_PREFETCH
            // the next chunk's tcgen05.ld in flight while this one is processed
            uint32_t(&cur)[32] = (q & 1) ? rb : ra;
            uint32_t(&nxt)[32] = (q & 1) ? ra : rb;
            if (q + 1 < NQ) LF_TMEM_LD32(ta + (q + 1) * 32, nxt);
#else
            uint32_t(&cur)[32] = ra;
            if (q > 0) {
              LF_TMEM_LD32(ta + q * 32, ra);
              tmem_ld_wait();
            }
#endif
            // exp arguments a = S log2e (BWD_ITEMS: S already carries -lse2 ln 2)
            // or S log2e - lse2 — monotone in S, so the chunk's largest a is
            // the transform of its largest S (the skip test needs no product)
            auto arg = [&](float v) { return MODE == BWD_ITEMS ? v * kLog2e : fmaf(v, kLog2e, -lse2); };
            float e[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) e[c] = __uint_as_float(cur[c]);

            // BWD_ITEMS: lane k checks stream row q*32+k; hm = rows of this chunk
            // whose target item lies in the owner tile (warp-uniform, rare).
            int tq = 0;
            unsigned hm = 0;
#ifndef LF_DIAG_NOTGT
            if (MODE == BWD_ITEMS && (FLAGS & kTgtIn)) {
              tq = tpre[q] - o0;  // the stream row's local target (p.tgt is padded to the tile grid)
              hm = __ballot_sync(0xffffffffu, static_cast<unsigned>(tq) < static_cast<unsigned>(BM));
            }
#endif
            const int jt = lc_t - q * 32;
#ifdef LF_DIAG_NOTGT  // timing diagnostic only (wrong results): no target handling
            const bool tgt_here = false;
            hm = 0;
#else
            const bool tgt_here = !(FLAGS & kTgtIn) ? false
                                  : MODE == BWD_ROWS ? static_cast<unsigned>(jt) < 32u : hm != 0u;
#endif
            bool skip = false;
            // (TEST = false samples only the first chunk of the tile)
            if ((FLAGS & kFilt) && (TEST || q == 0 || (FLAGS & kCount))) {
              const float mx = arg(max32(e));  // log-depth (FMNMX3 tree) on raw S
              const bool below = __all_sync(0xffffffffu, mx < kThr<FLAGS> && !tgt_here);
              any_below |= below;
              if (TEST) skip = below;
              if (FLAGS & kCount) {
#pragma unroll
                for (int c = 0; c < 32; ++c) e[c] = arg(e[c]);
              }
              if ((FLAGS & kCount) && MODE == BWD_ROWS) {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                  skipped += (e[c] < kThr<FLAGS> && q * 32 + c < nvalid && orow < p.n_owner) ? 1 : 0;
                // the target is never filtered (cce.cpp:193-195): undo its count
                if (tgt_here && select_reg(e, jt) < kThr<FLAGS> && orow < p.n_owner) --skipped;
                if (skip) ++skipped_sub;
              }
              if ((FLAGS & kCount) && MODE == BWD_ITEMS) {
                // the same statistic from the item side (the fused path has no
                // dX pass): stream columns are rows, each row's own target
                // entry (item = this lane's owner row) is never filtered
#pragma unroll
                for (int c = 0; c < 32; ++c)
                  skipped += (e[c] < kThr<FLAGS> && q * 32 + c < nvalid && orow < p.n_owner) ? 1 : 0;
                unsigned h = hm;
                while (h) {  // warp-uniform
                  const int jc = __ffs(h) - 1;
                  h &= h - 1u;
                  const int li = __shfl_sync(0xffffffffu, tq, jc);
                  if (li == lrow && select_reg(e, jc) < kThr<FLAGS> && orow < p.n_owner) --skipped;
                }
                if (skip) ++skipped_sub;
              }
            }
            if (skip) {
              // every G entry of the sub-tile is an exact zero
              uint32_t z[16];
#pragma unroll
              for (int c = 0; c < 16; ++c) z[c] = 0u;
              LF_TMEM_ST16(ta + q * 16, z);
            } else {
              live_bits |= 1u << q;
              if (!(FLAGS & kCount)) {
                // packed: two exp arguments per FFMA2 (bitwise the scalar
                // fmaf / multiply: one rounding each)
                const float bias = MODE == BWD_ITEMS ? 0.f : -lse2;
#pragma unroll
                for (int c = 0; c < 32; c += 2) ffma2(e[c], e[c + 1], e[c], e[c + 1], kLog2e, kLog2e, bias, bias);
              }
              float x[32];
              // FMA-pipe share of the exps (fast filter domain only)
              constexpr int kP = (FLAGS & kFilt) && kNoScale<FLAGS> ? kPolyBwd : 0;
#pragma unroll
              for (int c = 0; c < 32 - kP; ++c) {
#ifdef LF_DIAG_NOEXP
                x[c] = e[c];  // timing diagnostic only: wrong results
#else
                x[c] = ex2_approx(e[c]);
#endif
                if ((FLAGS & kFilt) && !kNoScale<FLAGS>) x[c] *= 18446744073709551616.f;  // 2^64
              }
#pragma unroll
              for (int c = 32 - kP; c < 32; c += 2) ex2_poly_ftz_x2(x[c], x[c + 1], e[c], e[c + 1]);
              // The target is never filtered: g = (s - 1) |scale| (cce.cpp:193-195).
              // Under FILT its softmax is recomputed unflushed from the raw
              // logit still in `cur`: s * 2^-62 / eps = 2^(a + 64).
              if (MODE == BWD_ROWS && (FLAGS & kTgtIn) && tgt_here) {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                  if (c == jt) x[c] = target_g<FLAGS>(x[c], cur[c], lse2, p.abs_scale);
              }
              if (MODE == BWD_ITEMS && (FLAGS & kTgtIn)) {
                while (hm) {  // warp-uniform loop over the hit columns
                  const int jc = __ffs(hm) - 1;
                  hm &= hm - 1u;
                  const int li = __shfl_sync(0xffffffffu, tq, jc);
                  if (li == lrow) {
                    const float lj = 0.f;  // S' already carries -lse2 ln 2
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                      if (c == jc) x[c] = target_g<FLAGS>(x[c], cur[c], lj, p.abs_scale);
                  }
                }
              }
              if (TEST && !(FLAGS & kTgtIn) && tgt_tile) {
                if (MODE == BWD_ROWS) {
                  if (__any_sync(0xffffffffu, static_cast<unsigned>(jt) < 32u)) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) x[c] = c == jt ? 0.f : x[c];
                  }
                } else {
                  const uint32_t mk = tm[q];
                  if (__any_sync(0xffffffffu, mk != 0u)) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) x[c] = (mk >> c) & 1u ? 0.f : x[c];
                  }
                }
              }
              uint32_t g[16];
#pragma unroll
              for (int c = 0; c < 16; ++c) g[c] = pack_bf16x2(x[2 * c], x[2 * c + 1]);
              LF_TMEM_ST16(ta + q * 16, g);
            }
#if LF_BWD_PREFETCH && !LF_BWD_LD64
            if (q + 1 < NQ) tmem_ld_wait();
#endif
          }
          return any_below;
          };
          skip_on = skip_on || tgt_tile ? process(std::true_type{}) : process(std::false_type{});
          tmem_st_wait();
          if ((FLAGS & kFilt) && lane == 0) live_mask[b * 4 + quad] = live_bits;
#ifndef LF_DIAG_EARLY
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&g_ready[b]);
#endif
        }
      }
      T0 += static_cast<uint32_t>(ntile + kPre);
      if (MODE == FWD) {
        // merge the warpgroups' running states for each row
        if (wg > 0) merge[(wg - 1) * BM + lrow] = make_float4(m, s, tv, has);
        named_bar_sync(1, G::kEpiThreads);
        if (wg == 0) {
#pragma unroll
          for (int k = 0; k < NWG - 1; ++k) {
            const float4 o = merge[k * BM + lrow];
            if (o.x != -INFINITY) {
              if (m == -INFINITY) {
                m = o.x;
                s = o.y;
              } else {
                const float nm = fmaxf(m, o.x);
                s = s * ex2_approx(m - nm) + o.y * ex2_approx(o.x - nm);
                m = nm;
              }
            }
            if (o.w != 0.f) {
              tv = o.z;
              has = 1.f;
            }
          }
          if (orow < p.n_owner) p.part[chunk * p.n_owner + orow] = make_float4(m, s, tv, has);
        }
        named_bar_sync(1, G::kEpiThreads);
      } else if (MODE == EVAL && !run_last) {
        // the owner rows continue in this CTA's next unit: keep the state, and
        // leave this chunk's slot empty (the run's totals go to its last slot)
        if (wg == 0 && orow < p.n_owner) {
          const int64_t rowp = chunk * p.n_owner + orow;
          p.ev_count[rowp] = 0;
          int4* di = reinterpret_cast<int4*>(p.ev_idx + rowp * KK);
#pragma unroll
          for (int k = 0; k < KK; k += 4) di[k / 4] = make_int4(0x7fffffff, 0x7fffffff, 0x7fffffff, 0x7fffffff);
        }
      } else if (MODE == EVAL) {
        // end of the run: merge the warpgroups' counts and top-k lists, one
        // record per row
        uint32_t* rec = reinterpret_cast<uint32_t*>(merge);
        if (wg > 0) {
          uint32_t* r = rec + ((wg - 1) * BM + lrow) * RS;
          r[0] = ecnt;
#pragma unroll
          for (int k = 0; k < KK; ++k) {
            r[1 + k] = __float_as_uint(kv[k]);
            r[1 + KK + k] = static_cast<uint32_t>(ki[k]);
          }
        }
        named_bar_sync(1, G::kEpiThreads);
        if (wg == 0) {
          for (int o = 0; o < NWG - 1; ++o) {
            const uint32_t* r = rec + (o * BM + lrow) * RS;
            ecnt += r[0];
            for (int k = 0; k < KK; ++k) {  // descending: stop at the first that does not fit
              const float cv = __uint_as_float(r[1 + k]);
              const int ci = static_cast<int>(r[1 + KK + k]);
              if (!(cv > kv[KK - 1] || (cv == kv[KK - 1] && ci < ki[KK - 1]))) break;
              topk_insert(kv, ki, cv, ci);
            }
          }
          if (orow < p.n_owner && ki[KK - 1] != 0x7fffffff) {  // publish a real k-th score
            const int b = __float_as_int(kv[KK - 1]);
            atomicMax(p.ev_floor + orow, b >= 0 ? b : b ^ 0x7fffffff);
          }
          if (orow < p.n_owner) {
            const int64_t rowp = chunk * p.n_owner + orow;
            p.ev_count[rowp] = ecnt;
            float4* dv = reinterpret_cast<float4*>(p.ev_val + rowp * KK);
            int4* di = reinterpret_cast<int4*>(p.ev_idx + rowp * KK);
#pragma unroll
            for (int k = 0; k < KK; k += 4) {
              dv[k / 4] = make_float4(kv[k], kv[k + 1], kv[k + 2], kv[k + 3]);
              di[k / 4] = make_int4(ki[k], ki[k + 1], ki[k + 2], ki[k + 3]);
            }
          }
        }
        named_bar_sync(1, G::kEpiThreads);
      } else if (MODE == FWDX) {
        // merge the warpgroups' (m, s, t) and their O accumulators per row:
        // M = max m_w, O = sum_w O_w 2^(m_w - M) (a warpgroup without a tile
        // in this unit has m_w = -inf and is left out), one fp32 partial row
        // of D columns per (chunk, row) plus the float4 {M, S, t, has}
        merge[wg * BM + lrow] = make_float4(m, s, tv, has);
        named_bar_sync(1, G::kEpiThreads);
        float mw[NWG], fw[NWG];
        float M = -INFINITY, S = 0.f;
#pragma unroll
        for (int w = 0; w < NWG; ++w) {
          const float4 o = merge[w * BM + lrow];
          mw[w] = o.x;
          M = fmaxf(M, o.x);
          if (o.w != 0.f) {
            tv = o.z;
            has = 1.f;
          }
        }
#pragma unroll
        for (int w = 0; w < NWG; ++w) {
          fw[w] = mw[w] == -INFINITY ? 0.f : ex2_approx(mw[w] - M);
          S = fmaf(merge[w * BM + lrow].y, fw[w], S);
        }
        mbar_wait(acc_full, j & 1);
        tc_fence_after();
        float* dst = p.out + (chunk * p.n_owner + orow) * D;
        for (int c0 = wg * 16; c0 < D; c0 += 16 * NWG) {
          float o[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) o[c] = 0.f;
#pragma unroll
          for (int w = 0; w < NWG; ++w) {
            uint32_t r16[16];
            LF_TMEM_LD16(tmem + lane_base + C::kAccCol + w * D + c0, r16);
            tmem_ld_wait();
            if (mw[w] != -INFINITY) {
#pragma unroll
              for (int c = 0; c < 16; ++c) o[c] = fmaf(__uint_as_float(r16[c]), fw[w], o[c]);
            }
          }
          if (orow < p.n_owner) {
#pragma unroll
            for (int c = 0; c < 16; c += 4)
              *reinterpret_cast<float4*>(dst + c0 + c) = make_float4(o[c], o[c + 1], o[c + 2], o[c + 3]);
          }
        }
        if (wg == 0 && orow < p.n_owner) p.part[chunk * p.n_owner + orow] = make_float4(M, S, tv, has);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
        named_bar_sync(1, G::kEpiThreads);  // the merge records are rewritten by the next unit
      } else {
        // accumulator read-out: 16-column groups round robin over warpgroups
        mbar_wait(acc_full, j & 1);
        tc_fence_after();
        float* dst = MODE == BWD_ROWS ? p.out + (chunk * p.n_owner + orow) * D
                                      : p.out + orow * D;
        const float os = p.out_scale;
        // !kTgtIn: the target entries of softmax - onehot, left out of the
        // product: -scale (1 - p_t) x (the target's item row | the rows
        // targeting this item, in sorted = row order)
        uint32_t fb = 0, fe = 0;
        const __nv_bfloat16* frow = nullptr;
        if (!(FLAGS & kTgtIn) && orow < p.n_owner) {
          if (MODE == BWD_ROWS) {
            if (tgt >= s_begin && tgt < s_end) {
              frow = p.fix_rows + static_cast<int64_t>(tgt) * D;
              fe = 1;
            }
          } else {
            fb = p.fix_off[orow];
            fe = p.fix_off[orow + 1];
          }
        }
        for (int c0 = wg * 16; c0 < D; c0 += 16 * NWG) {
          uint32_t r16[16];
          LF_TMEM_LD16(tmem + lane_base + C::kAccCol + c0, r16);
          tmem_ld_wait();
          if (orow < p.n_owner) {
            float o[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) o[c] = __uint_as_float(r16[c]) * os;
            if (!(FLAGS & kTgtIn)) {
              float fx[16];
#pragma unroll
              for (int c = 0; c < 16; ++c) fx[c] = 0.f;
              for (uint32_t k = fb; k < fe; ++k) {
                const int64_t rr = MODE == BWD_ROWS ? orow : static_cast<int64_t>(p.fix_list[k]);
                const __nv_bfloat16* xr = MODE == BWD_ROWS ? frow : p.fix_rows + rr * D;
#ifdef LF_DIAG_NOTW  // timing diagnostic only (wrong results)
                const float wk = 1.f;
#else
                const float wk = p.tw[rr];  // 1 - p_t of that row
#endif
#pragma unroll
                for (int c = 0; c < 16; ++c) fx[c] = fmaf(wk, __bfloat162float(xr[c0 + c]), fx[c]);
              }
#pragma unroll
              for (int c = 0; c < 16; ++c) o[c] = fmaf(-p.fix_scale, fx[c], o[c]);
            }
#pragma unroll
            for (int c = 0; c < 16; c += 4)
              *reinterpret_cast<float4*>(dst + c0 + c) = make_float4(o[c], o[c + 1], o[c + 2], o[c + 3]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
      }
    }
    if ((FLAGS & kCount) && (MODE == BWD_ROWS || MODE == BWD_ITEMS)) {
      for (int off = 16; off > 0; off >>= 1) skipped += __shfl_xor_sync(0xffffffffu, skipped, off);
      if (lane == 0 && skipped) atomicAdd(&p.counters[0], skipped);
      if (lane == 0 && skipped_sub) atomicAdd(&p.counters[1], skipped_sub);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// -------------------------------------------------------------- host side --
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// rows x D bf16 row-major, box = 64 cols x box_rows rows, 128-byte swizzle.
int make_map(CUtensorMap* map, const void* ptr, int64_t rows, int D, int box_rows) {
  auto enc = get_encode();
  if (!enc) return fail(LF_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0)
    return fail(LF_EINVAL, "bf16 path: X/E base pointers must be 16-byte aligned");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LF_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return LF_OK;
}

// rows x 16 bf16 (32 B rows), box = 16 x box_rows, SWIZZLE_32B: the bias
// columns of the BWD_ITEMS S MMA.
int make_map_k16(CUtensorMap* map, const void* ptr, int64_t rows, int box_rows) {
  auto enc = get_encode();
  if (!enc) return fail(LF_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {16, static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {32};
  cuuint32_t box[2] = {16, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LF_ECUDA, "cuTensorMapEncodeTiled (k16) failed: " + std::to_string(r));
  return LF_OK;
}

// Bias columns: stream row i -> [c1, c2, c3, 0 x 13] with c1 + c2 + c3 =
// -lse2_i ln 2 to ~2^-24 relative (three bf16 parts); rows past n carry a
// huge negative bias (their softmax is 0).  The owner side multiplies by the
// constant [1, 1, 1, 0 x 13] rows (`ones`, 128 rows).
__global__ void bias_columns(const double* __restrict__ lse, int64_t n, int64_t n_pad,
                             double lse_sub, __nv_bfloat16* __restrict__ bias,
                             __nv_bfloat16* __restrict__ ones) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < 128 && ones) {
#pragma unroll
    for (int k = 0; k < 16; ++k) ones[i * 16 + k] = __float2bfloat16_rn(k < 3 ? 1.f : 0.f);
  }
  if (i >= n_pad) return;
  float c[3] = {-1e30f, 0.f, 0.f};
  if (i < n) {
    const double lse2 = lse[i] * 1.4426950408889634 - lse_sub;
    double r = -lse2 * 0.6931471805599453;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const __nv_bfloat16 h = __double2bfloat16(r);
      c[k] = __bfloat162float(h);
      r -= static_cast<double>(c[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) bias[i * 16 + k] = __float2bfloat16_rn(k < 3 ? c[k] : 0.f);
}

// max_j |E_j|_2 over the catalog (non-negative floats order like their bits).
template <int D>
__global__ void max_row_norm(const __nv_bfloat16* __restrict__ E, int64_t v, unsigned* __restrict__ out) {
  float best = 0.f;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < v;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4* r = reinterpret_cast<const uint4*>(E + j * D);
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < D / 8; ++k) {
      const uint4 w = __ldg(r + k);
      const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float lo = __uint_as_float(u[h] << 16), hi = __uint_as_float(u[h] & 0xffff0000u);
        acc = fmaf(lo, lo, fmaf(hi, hi, acc));
      }
    }
    best = fmaxf(best, acc);
  }
  for (int o = 16; o > 0; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(sqrtf(best)));
}

// FWDX per-row overflow bound in log2 units: |x_i| max_j |e_j| log2e (plus a
// rounding margin) bounds every logit of the row; padding rows get -inf.
template <int D>
__global__ void row_bounds(const __nv_bfloat16* __restrict__ X, int64_t n, int64_t n_pad,
                           const unsigned* __restrict__ emax, float* __restrict__ bound) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  float b = -INFINITY;
  if (i < n) {
    float acc = 0.f;
    for (int k = 0; k < D; ++k) {
      const float x = __bfloat162float(X[i * D + k]);
      acc = fmaf(x, x, acc);
    }
    b = sqrtf(acc) * __uint_as_float(*emax) * kLog2e * (1.f + 0x1p-10f) + 1.f;
  }
  bound[i] = b;
}

__global__ void prep_rows(const int64_t* __restrict__ targets, const double* __restrict__ lse,
                          int64_t n, int64_t n_pad, int64_t v_shard, int64_t v_offset,
                          double lse_sub, int32_t* __restrict__ tgt,
                          float* __restrict__ lse2) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  int32_t t = -1;
  float l = INFINITY;
  if (i < n) {
    const int64_t x = targets[i] - v_offset;
    t = (x >= 0 && x < v_shard) ? static_cast<int32_t>(x) : -1;
    if (lse) l = static_cast<float>(lse[i] * 1.4426950408889634 - lse_sub);
  }
  tgt[i] = t;
  if (lse2) lse2[i] = l;
}

// Sort keys of the rows by local target item >> shift (out-of-shard targets
// -> `none`, the last bin).
__global__ void target_keys(const int32_t* __restrict__ tgt, int64_t n, int64_t none,
                            int64_t* __restrict__ keys, int shift) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = tgt[i] >= 0 ? (tgt[i] >> shift) : none;
}

// The dE pass's hit list: row << 7 | (target & 127) (the local item in its
// 128-item owner tile), so the epilogue needs no dependent load of tgt[row].
__global__ void pack_hits(const uint32_t* __restrict__ rows, const int32_t* __restrict__ tgt, int64_t n,
                          uint64_t* __restrict__ hits) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) hits[i] = static_cast<uint64_t>(rows[i]) << 7 | static_cast<uint32_t>(tgt[rows[i]] & 127);
}

// Read-out form of the backward: w_i = 1 - p_t,i = -expm1(t_i - lse_i) per
// row whose target is in the shard (0 otherwise), with the target logit t_i
// in double from the bf16 rows (warp per row) — full precision however close
// p_t is to 1.
__global__ void target_weight(const __nv_bfloat16* __restrict__ X, const __nv_bfloat16* __restrict__ E,
                              const int32_t* __restrict__ tgt, const double* __restrict__ lse, int64_t n,
                              int64_t n_pad, int D, float* __restrict__ tw) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n_pad) return;
  const int t = row < n ? tgt[row] : -1;
  double acc = 0.0;
  if (t >= 0)
    for (int k = lane; k < D; k += 32)
      acc += static_cast<double>(__bfloat162float(X[row * D + k])) *
             static_cast<double>(__bfloat162float(E[static_cast<int64_t>(t) * D + k]));
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) tw[row] = t >= 0 ? static_cast<float>(-expm1(acc - lse[row])) : 0.f;
}

template <int D, int MODE, int FLAGS>
int launch_mode(const CUtensorMap& mo, const CUtensorMap& ms, const CUtensorMap& mb,
                const CUtensorMap& m1, const TcParams& p, cudaStream_t st) {
  using C = Cfg<D, MODE>;
  auto kern = cce_tc_kernel<D, MODE, FLAGS>;
  LF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
  const int grid = static_cast<int>(std::min<int64_t>(p.units, num_sms()));
  ProfScope prof(MODE == FWD    ? LF_K_CCE_FWD
                 : MODE == EVAL ? LF_K_EVAL
                 : MODE == FWDX ? LF_K_CCE_FWD_DX
                 : (MODE == BWD_ROWS ? LF_K_CCE_BWD_DX : LF_K_CCE_BWD_DE),
                 st);
  kern<<<grid, Geo<MODE, D>::kThreads, C::kSmem, st>>>(mo, ms, mb, m1, p);
  LF_LAUNCHED();
  return LF_OK;
}

template <int D, int MODE>
int launch_flags(int flags, const CUtensorMap& mo, const CUtensorMap& ms, const CUtensorMap& mb,
                 const CUtensorMap& m1, const TcParams& p, cudaStream_t st) {
  if constexpr (MODE == FWD) {
    return launch_mode<D, MODE, 0>(mo, ms, mb, m1, p, st);
  } else if constexpr (MODE == EVAL) {  // flags = list-length class (kEvalKOf)
    if (flags == 3) return launch_mode<D, MODE, 3>(mo, ms, mb, m1, p, st);
    if (flags == 2) return launch_mode<D, MODE, 2>(mo, ms, mb, m1, p, st);
    if (flags == 1) return launch_mode<D, MODE, 1>(mo, ms, mb, m1, p, st);
    return launch_mode<D, MODE, 0>(mo, ms, mb, m1, p, st);
  } else {
    switch (flags) {
      case 0: return launch_mode<D, MODE, 0>(mo, ms, mb, m1, p, st);
      case kFilt: return launch_mode<D, MODE, kFilt>(mo, ms, mb, m1, p, st);
      case kFilt | kTgtIn: return launch_mode<D, MODE, kFilt | kTgtIn>(mo, ms, mb, m1, p, st);
      default: return launch_mode<D, MODE, kFilt | kCount | kTgtIn>(mo, ms, mb, m1, p, st);
    }
  }
}

template <int MODE>
int launch_d(int D, int flags, const CUtensorMap& mo, const CUtensorMap& ms, const CUtensorMap& mb,
             const CUtensorMap& m1, const TcParams& p, cudaStream_t st) {
  switch (D) {
    case 64: return launch_flags<64, MODE>(flags, mo, ms, mb, m1, p, st);
#ifndef LF_VARIANT_D64_ONLY
    case 128: return launch_flags<128, MODE>(flags, mo, ms, mb, m1, p, st);
    case 192: return launch_flags<192, MODE>(flags, mo, ms, mb, m1, p, st);
    case 256: return launch_flags<256, MODE>(flags, mo, ms, mb, m1, p, st);
#endif
    default: return fail(LF_EUNSUPPORTED, "tc: d must be 64/128/192/256");
  }
}

// Pick the number of stream chunks so the persistent CTAs get equal work:
// maximise units / (waves * SMs) — a 0.98 wave efficiency leaves 2 % of the
// SMs idle for the whole last unit — with a tiny penalty per extra chunk
// (each costs one more partial buffer and owner-tile reload).
int64_t pick_chunks(int64_t owner_tiles, int64_t stream_tiles, int64_t max_chunks) {
  const int64_t sms = num_sms();
  int64_t best = 1;
  double best_score = -1.0;
  for (int64_t c = 1; c <= std::min(max_chunks, stream_tiles); ++c) {
    const int64_t tiles_per = ceil_div(stream_tiles, c);
    const int64_t real_c = ceil_div(stream_tiles, tiles_per);
    const int64_t units = owner_tiles * real_c;
    const int64_t waves = ceil_div(units, sms);
    const double eff = static_cast<double>(units) / static_cast<double>(waves * sms);
    const double score = eff - 2e-4 * static_cast<double>(real_c);
    if (score > best_score + 1e-12) {
      best_score = score;
      best = c;
    }
  }
  return best;
}

// dX from the FWDX partials, one warp per row.  The row's log2-domain LSE
// comes from its own partials (lse_in == nullptr; also writes lse / pos with
// combine_partials' double arithmetic) or from the given global lse (catalog
// sharding: the local partials after the (m, s, t) exchange).  Then
// dX_i = scale (sum_p O_p,i 2^(m_p,i - lse2_i) - [x_i local] E_(x_i))
// (cce.cpp:189-231 with the target's -1 folded out of the tile loop).
template <int D>
__global__ void fwdx_dx(const float4* __restrict__ part, const float* __restrict__ opart, int P,
                        int64_t n, const double* __restrict__ lse_in,
                        const __nv_bfloat16* __restrict__ E, const int32_t* __restrict__ tgt,
                        float scale, double* __restrict__ lse_out, double* __restrict__ pos_out,
                        float* __restrict__ dX) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n) return;
  double lse2, t = 0.0;
  for (int p = 0; p < P; ++p) {
    const float4 q = part[p * n + row];
    if (q.w != 0.f) t = static_cast<double>(q.z);
  }
  if (lse_in) {
    lse2 = lse_in[row] * 1.4426950408889634;
  } else {
    double M = -INFINITY;
    for (int p = 0; p < P; ++p) M = fmax(M, static_cast<double>(part[p * n + row].x));
    double S = 0.0;
    for (int p = 0; p < P; ++p) {
      const float4 q = part[p * n + row];
      if (q.x != -INFINITY) S += static_cast<double>(q.y) * exp2(static_cast<double>(q.x) - M);
    }
    lse2 = M + log2(S);
    if (lane == 0) {
      lse_out[row] = lse2 * 0.6931471805599453;
      pos_out[row] = t;
    }
  }
  constexpr int CPL = D / 32;  // columns per lane
  float acc[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) acc[k] = 0.f;
  for (int p = 0; p < P; ++p) {
    const float mp = part[p * n + row].x;
    if (mp == -INFINITY) continue;
    const float w = static_cast<float>(exp2(static_cast<double>(mp) - lse2));
    const float* o = opart + (p * n + row) * D;
#pragma unroll
    for (int k = 0; k < CPL; ++k) acc[k] = fmaf(w, o[lane + 32 * k], acc[k]);
  }
  // the target entry was left out of O: its term p_t - 1 in full precision
  const int ti = tgt[row];
  const float wt = ti >= 0 ? static_cast<float>(-expm1(t - lse2 * 0.6931471805599453)) : 0.f;
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    const float et = ti >= 0 ? __bfloat162float(E[static_cast<int64_t>(ti) * D + lane + 32 * k]) : 0.f;
    dX[row * D + lane + 32 * k] = scale * fmaf(-wt, et, acc[k]);
  }
}

}  // namespace

int tc_fwdx_supported(int D) { return D == 64 || D == 128 || D == 256; }

// Fused forward + unnormalised dX over the local shard.  part: [P][n] float4
// {m, s, t, has} (log2 units, as tc_cce_forward_partials); opart: [P][n][D]
// fp32 O = sum over the chunk's items j of 2^(logit_ij log2e - m) E_j;
// tgt: [ceil(n/128)*128] local target index or -1.
int tc_cce_fwdx_partials(const void* X, const void* E, const int64_t* targets, int64_t n, int D,
                         int64_t v, int64_t v_offset, Scratch& part, Scratch& opart, Scratch& tgt,
                         int* P_out, cudaStream_t st) {
  if (!tc_fwdx_supported(D)) return fail(LF_EUNSUPPORTED, "fused forward/dX: d must be 64, 128 or 256");
  const int BN = bn_fwdx(D);  // = Geo<FWDX, D>::BN
  const int64_t owner_tiles = ceil_div(n, BM);
  const int64_t stream_tiles = ceil_div(v, BN);
#ifndef LF_FWDX_MAXCHUNKS
#define LF_FWDX_MAXCHUNKS 0  // 0: bounded by the O partials' memory (see below)
#endif
  // More V chunks balance the waves when there are few owner tiles (cfg5's
  // shard: 60), at the price of one n x D fp32 partial per chunk: the
  // partials may take max(64 MB, 1/8 of the shard's E + dE bytes) — cfg2
  // keeps 4 chunks, the cfg5 shard gets ~27 (13.4 -> 11.4 ms).
  const int64_t part_budget = std::max<int64_t>(int64_t(64) << 20, v * D * 6 / 8);
  const int64_t max_chunks =
      LF_FWDX_MAXCHUNKS > 0 ? LF_FWDX_MAXCHUNKS
                            : std::max<int64_t>(4, std::min<int64_t>(64, part_budget / (n * D * 4)));
  const int64_t chunks = pick_chunks(owner_tiles, stream_tiles, max_chunks);
  const int64_t tiles_per = ceil_div(stream_tiles, chunks);
  const int64_t P = ceil_div(stream_tiles, tiles_per);
  const int64_t n_pad = owner_tiles * BM;
  int rc = tgt.alloc(sizeof(int32_t) * n_pad, st);
  if (!rc) rc = part.alloc(sizeof(float4) * P * n, st);
  if (!rc) rc = opart.alloc(sizeof(float) * P * n * D, st);
  Scratch bound;  // [n_pad] floats, then the catalog's max item norm
  if (!rc) rc = bound.alloc(sizeof(float) * (n_pad + 1), st);
  if (rc) return rc;
  prep_rows<<<ceil_div(n_pad, 256), 256, 0, st>>>(targets, nullptr, n, n_pad, v, v_offset, 0.0,
                                                 tgt.as<int32_t>(), nullptr);
  LF_LAUNCHED();
  unsigned* emax = reinterpret_cast<unsigned*>(bound.as<float>() + n_pad);
  LF_CUDA(cudaMemsetAsync(emax, 0, sizeof(unsigned), st));
  {
    const auto* Eb = static_cast<const __nv_bfloat16*>(E);
    const auto* Xb = static_cast<const __nv_bfloat16*>(X);
    const int g = static_cast<int>(std::min<int64_t>(ceil_div(v, 256), 4 * num_sms()));
    if (D == 64) {
      max_row_norm<64><<<g, 256, 0, st>>>(Eb, v, emax);
      row_bounds<64><<<ceil_div(n_pad, 256), 256, 0, st>>>(Xb, n, n_pad, emax, bound.as<float>());
    } else if (D == 128) {
      max_row_norm<128><<<g, 256, 0, st>>>(Eb, v, emax);
      row_bounds<128><<<ceil_div(n_pad, 256), 256, 0, st>>>(Xb, n, n_pad, emax, bound.as<float>());
    } else {
      max_row_norm<256><<<g, 256, 0, st>>>(Eb, v, emax);
      row_bounds<256><<<ceil_div(n_pad, 256), 256, 0, st>>>(Xb, n, n_pad, emax, bound.as<float>());
    }
    LF_LAUNCHED();
  }
  CUtensorMap mo, ms;
  rc = make_map(&mo, X, n, D, BM);
  if (!rc) rc = make_map(&ms, E, v, D, BN);
  if (rc) return rc;
  TcParams p{};
  p.n_owner = n;
  p.n_stream = v;
  p.owner_tiles = owner_tiles;
  p.chunk = tiles_per * BN;
  p.n_chunks = P;
  p.units = owner_tiles * P;
  p.tgt = tgt.as<int32_t>();
  p.lse2 = bound.as<float>();  // FWDX: the per-row overflow bound
  p.part = part.as<float4>();
  p.out = opart.as<float>();
#ifdef LF_VARIANT_D64_ONLY
  rc = launch_mode<64, FWDX, 0>(mo, ms, mo, mo, p, st);
#else
  rc = D == 64    ? launch_mode<64, FWDX, 0>(mo, ms, mo, mo, p, st)
       : D == 128 ? launch_mode<128, FWDX, 0>(mo, ms, mo, mo, p, st)
                  : launch_mode<256, FWDX, 0>(mo, ms, mo, mo, p, st);
#endif
  if (rc) return rc;
  *P_out = static_cast<int>(P);
  return LF_OK;
}

int tc_fwdx_dx(const float* part, const float* opart, int P, int64_t n, int D, const double* lse_in,
               const void* E, const int32_t* tgt, double scale, double* lse_out, double* pos_out,
               float* dX, cudaStream_t st) {
  const int64_t blocks = ceil_div(n, 8);
  const float sc = static_cast<float>(scale);
  const auto* pp = reinterpret_cast<const float4*>(part);
  const auto* Eb = static_cast<const __nv_bfloat16*>(E);
  ProfScope prof(LF_K_AUX, st);
  if (D == 64)
    fwdx_dx<64><<<blocks, 256, 0, st>>>(pp, opart, P, n, lse_in, Eb, tgt, sc, lse_out, pos_out, dX);
  else if (D == 128)
    fwdx_dx<128><<<blocks, 256, 0, st>>>(pp, opart, P, n, lse_in, Eb, tgt, sc, lse_out, pos_out, dX);
  else if (D == 256)
    fwdx_dx<256><<<blocks, 256, 0, st>>>(pp, opart, P, n, lse_in, Eb, tgt, sc, lse_out, pos_out, dX);
  else
    return fail(LF_EUNSUPPORTED, "fused forward/dX: d must be 64, 128 or 256");
  LF_LAUNCHED();
  return LF_OK;
}

// Both fold the per-chunk partials and run the forward.
int tc_cce_forward_partials(const void* X, const void* E, const int64_t* targets, int64_t n,
                            int D, int64_t v, int64_t v_offset, Scratch& ws, float** part_out,
                            int* P_out, cudaStream_t st) {
  constexpr int BN = Geo<FWD>::BN;
  const int64_t owner_tiles = ceil_div(n, BM);
  const int64_t stream_tiles = ceil_div(v, BN);
  const int64_t chunks = pick_chunks(owner_tiles, stream_tiles, LF_FWD_MAXCHUNKS);
  const int64_t tiles_per = ceil_div(stream_tiles, chunks);
  const int64_t P = ceil_div(stream_tiles, tiles_per);
  const int64_t n_pad = owner_tiles * BM;
  Scratch tgt;
  int rc = tgt.alloc(sizeof(int32_t) * n_pad, st);
  if (!rc) rc = ws.alloc(sizeof(float4) * P * n, st);
  if (rc) return rc;
  prep_rows<<<ceil_div(n_pad, 256), 256, 0, st>>>(targets, nullptr, n, n_pad, v, v_offset, 0.0,
                                                 tgt.as<int32_t>(), nullptr);
  LF_LAUNCHED();
  CUtensorMap mo, ms;
  rc = make_map(&mo, X, n, D, BM);
  if (!rc) rc = make_map(&ms, E, v, D, BN);
  if (rc) return rc;
  TcParams p{};
  p.n_owner = n;
  p.n_stream = v;
  p.owner_tiles = owner_tiles;
  p.chunk = tiles_per * BN;
  p.n_chunks = P;
  p.units = owner_tiles * P;
  p.tgt = tgt.as<int32_t>();
  p.part = ws.as<float4>();
  rc = launch_d<FWD>(D, 0, mo, ms, mo, mo, p, st);
  if (rc) return rc;
  *part_out = ws.as<float>();
  *P_out = static_cast<int>(P);
  return LF_OK;
}

int tc_eval_partials(const void* X, const void* E, const void* Et, const int32_t* tl, int64_t n,
                     int D, int64_t v, int k, Scratch& cnt, Scratch& val, Scratch& idx, int* P_out,
                     int* K_out, cudaStream_t st) {
  Scratch floor;
  {
    const int rc0 = floor.alloc(sizeof(int32_t) * ceil_div(n, BM) * BM, st);
    if (rc0) return rc0;
    LF_CUDA(cudaMemsetAsync(floor.ptr, 0x80, sizeof(int32_t) * ceil_div(n, BM) * BM, st));  // below any key
  }
  const int kclass = k <= 4 ? 3 : (k <= 8 ? 2 : (k <= 12 ? 1 : 0));
  const int K = kclass == 3 ? 4 : (kclass == 2 ? 8 : (kclass == 1 ? 12 : 16));
  constexpr int BN = Geo<EVAL>::BN;
  const int64_t owner_tiles = ceil_div(n, BM);
  const int64_t stream_tiles = ceil_div(v, BN);
#ifndef LF_EVAL_CHUNKS
#define LF_EVAL_CHUNKS 64
#endif
  const int64_t chunks = pick_chunks(owner_tiles, stream_tiles, LF_EVAL_CHUNKS);
  const int64_t tiles_per = ceil_div(stream_tiles, chunks);
  const int64_t P = ceil_div(stream_tiles, tiles_per);
  int rc = cnt.alloc(sizeof(uint32_t) * P * n, st);
  if (!rc) rc = val.alloc(sizeof(float) * P * n * K, st);
  if (!rc) rc = idx.alloc(sizeof(int32_t) * P * n * K, st);
  if (rc) return rc;
  CUtensorMap mo, ms, mt;
  rc = make_map(&mo, X, n, D, BM);
  if (!rc) rc = make_map(&ms, E, v, D, BN);
  if (!rc) rc = make_map(&mt, Et, owner_tiles * BM, D, BN);
  if (rc) return rc;
  TcParams p{};
  p.n_owner = n;
  p.n_stream = v;
  p.owner_tiles = owner_tiles;
  p.chunk = tiles_per * BN;
  p.n_chunks = P;
  p.tgt = tl;
  p.ev_count = cnt.as<uint32_t>();
  p.ev_val = val.as<float>();
  p.ev_idx = idx.as<int32_t>();
  p.ev_floor = floor.as<int32_t>();
  // Seeding pass: the first S chunks for every row, as a launch of their own.
  // Each row's k-th score over that subset (published to ev_floor) is a lower
  // bound of its k-th over the catalog, so the main launch starts every list
  // from placeholders just below it instead of empty, so fewer slabs reach
  // the divergent insertion path.  The seeding pass's results are the first
  // S chunks' records — no work repeats.  Off by default: at cfg2 (k = 10)
  // S = 1 / 2 / 4 measured 14.3 / 14.4 / 14.1 ms against 13.9 ms without — the
  // CTA-contiguous order already lets each list see most of V, and the gate
  // (two max trees per slab) costs the same either way.  S = LSEFORGE_EVAL_SEED_CHUNKS.
  int64_t seed_chunks = 0;
  if (const char* e = std::getenv("LSEFORGE_EVAL_SEED_CHUNKS")) seed_chunks = std::atoll(e);
  const int64_t S = P > 1 ? std::max<int64_t>(0, std::min<int64_t>(seed_chunks, P - 1)) : 0;
  if (S > 0) {
    TcParams q = p;
    q.n_chunks = S;
    q.c_first = 0;
    q.units = owner_tiles * S;
    rc = launch_d<EVAL>(D, kclass, mo, ms, mt, mo, q, st);
    if (rc) return rc;
  }
  p.c_first = S;
  p.units = owner_tiles * (P - S);
  rc = launch_d<EVAL>(D, kclass, mo, ms, mt, mo, p, st);
  if (rc) return rc;
  *P_out = static_cast<int>(P);
  *K_out = K;
  return LF_OK;
}

int tc_cce_backward(const void* X, const void* E, const int64_t* targets, const double* lse,
                    double scale, double eps, int64_t n, int D, int64_t v, int64_t v_offset,
                    float* dX, float* dE, unsigned long long* counters, cudaStream_t st,
                    const PeerPush* push) {
  if (scale == 0.0) {
    if (dX) LF_CUDA(cudaMemsetAsync(dX, 0, sizeof(float) * n * D, st));
    LF_CUDA(cudaMemsetAsync(dE, 0, sizeof(float) * v * D, st));
    if (push) return peer_reduce_push(dX, 1, n * D, push->peers, push->world, push->rank, push->parity_off, st);
    return LF_OK;
  }
  // G domain.  No filter: G = softmax * |scale| (lse2 = lse log2e - log2|scale|).
  // Filter (eps >= 2^-100): lse2 = lse log2e + log2(eps) + 126, so the exp
  // argument is < -126 exactly when softmax < eps and ex2.approx.ftz flushes
  // it; survivors are scaled by 2^64, i.e. G = softmax * 2^-62 / eps, and the
  // read-out multiplies by scale * eps * 2^62 (sign included).  Below 2^-100
  // the filtered entries are far under fp32 resolution of the accumulated
  // gradient and the unfiltered kernel is used.
  if (eps > 2.0) eps = 2.0;  // softmax <= 1: every eps > 1 filters every off-target entry
  const bool filt = eps >= 0x1p-100;
  const bool count = filt && counters != nullptr;
  const bool tgt_in = filt && (count || eps >= 0x1p-12);
  const int flags = filt ? (kFilt | (count ? kCount : 0) | (tgt_in ? kTgtIn : 0)) : 0;
  const double sub = filt ? -std::log2(eps) - 126.0 : std::log2(std::fabs(scale));
  const bool noscale = LF_NOSCALE != 0 && !tgt_in;
  const double gscale = filt ? std::ldexp(1.0, noscale ? -126 : -62) / eps : std::fabs(scale);
  const double out_scale =
      filt ? scale * eps * std::ldexp(1.0, noscale ? 126 : 62) : (scale < 0 ? -1.0 : 1.0);
  constexpr int BN = Geo<BWD_ROWS>::BN;        // dX pass stream tile (items)
  const int BNi = bn_items(static_cast<int>(D));  // dE pass stream tile (rows), = Geo<BWD_ITEMS, D>::BN
  const int64_t row_tiles = ceil_div(n, BM);
  const int64_t item_tiles = ceil_div(v, BM);     // dE owner tiles
  const int64_t item_stream = ceil_div(v, BN);    // dX stream tiles
  const int64_t n_pad = std::max(row_tiles * BM, ceil_div(n, BN) * BN);
  Scratch tgt, lse2;
  int rc = tgt.alloc(sizeof(int32_t) * n_pad, st);
  if (!rc) rc = lse2.alloc(sizeof(float) * n_pad, st);
  if (rc) return rc;
  prep_rows<<<ceil_div(n_pad, 256), 256, 0, st>>>(targets, lse, n, n_pad, v, v_offset, sub,
                                                 tgt.as<int32_t>(), lse2.as<float>());
  LF_LAUNCHED();
  // read-out form (!tgt_in): 1 - p_t per row, full precision
  Scratch tw;
  if (!tgt_in) {
    rc = tw.alloc(sizeof(float) * n_pad, st);
    if (rc) return rc;
    target_weight<<<ceil_div(n_pad, 8), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(X),
                                                      static_cast<const __nv_bfloat16*>(E), tgt.as<int32_t>(),
                                                      lse, n, n_pad, static_cast<int>(D), tw.as<float>());
    LF_LAUNCHED();
  }
  CUtensorMap mx_own, mx_str, me_own, me_str;  // owner box 128 rows, stream box BN rows
  rc = make_map(&mx_own, X, n, D, BM);
  if (!rc) rc = make_map(&mx_str, X, n, D, BNi);
  if (!rc) rc = make_map(&me_own, E, v, D, BM);
  if (!rc) rc = make_map(&me_str, E, v, D, BN);
  if (rc) return rc;

  // ---- pass 1: dX (owner rows, stream items), V split into a few chunks ----
  // (dX == nullptr: the caller has dX from the fused forward; the skip
  // statistics are then counted by the dE pass)
  if (dX) {
  const int64_t chunks = pick_chunks(row_tiles, item_stream, 8);
  const int64_t tiles_per = ceil_div(item_stream, chunks);
  const int64_t P = ceil_div(item_stream, tiles_per);
  Scratch dxp;
  float* dx_out = dX;
  if (P > 1) {
    rc = dxp.alloc(sizeof(float) * P * n * D, st);
    if (rc) return rc;
    dx_out = dxp.as<float>();
  }
  TcParams p{};
  p.n_owner = n;
  p.n_stream = v;
  p.owner_tiles = row_tiles;
  p.chunk = tiles_per * BN;
  p.n_chunks = P;
  p.units = row_tiles * P;
  p.tgt = tgt.as<int32_t>();
  p.lse2 = lse2.as<float>();
  p.abs_scale = static_cast<float>(gscale);
  p.out_scale = static_cast<float>(out_scale);
  p.out = dx_out;
  p.counters = counters;
  p.fix_rows = static_cast<const __nv_bfloat16*>(E);
  p.fix_scale = static_cast<float>(scale);
  p.tw = tw.as<float>();
  rc = launch_d<BWD_ROWS>(D, flags, mx_own, me_str, mx_own, mx_own, p, st);
  if (rc) return rc;
  if (push) {  // chunk reduction fused with the all-gather of this rank's dX partial
    rc = peer_reduce_push(dx_out, static_cast<int>(P), n * D, push->peers, push->world, push->rank,
                          push->parity_off, st);
    if (rc) return rc;
  } else if (P > 1) {
    rc = launch_reduce_f32(dx_out, static_cast<int>(P), n * D, dX, st);
    if (rc) return rc;
  }
  }
  // ---- pass 2: dE (owner items, stream rows) ----
  TcParams q{};
  q.n_owner = v;
  q.n_stream = n;
  q.owner_tiles = item_tiles;
  q.chunk = ceil_div(n, BNi) * BNi;
  q.n_chunks = 1;
  q.units = item_tiles;
  q.tgt = tgt.as<int32_t>();
  q.lse2 = lse2.as<float>();
  q.abs_scale = static_cast<float>(gscale);
  q.out_scale = static_cast<float>(out_scale);
  q.out = dE;
  q.counters = counters;
  q.fix_rows = static_cast<const __nv_bfloat16*>(X);
  q.fix_scale = static_cast<float>(scale);
  q.tw = tw.as<float>();
  Scratch keys, fix_list, fix_off, hit_list, hit_off, hits;
  if (!tgt_in) {
    // rows grouped by local target item (stable, so each item's rows are
    // summed in row order at the dE read-out); out-of-shard targets -> item v
    rc = keys.alloc(sizeof(int64_t) * n, st);
    if (rc) return rc;
    target_keys<<<ceil_div(n, 256), 256, 0, st>>>(tgt.as<int32_t>(), n, v, keys.as<int64_t>(), 0);
    LF_LAUNCHED();
    rc = sort_by_item(keys.as<int64_t>(), n, v + 1, fix_list, fix_off, st);
    if (rc) return rc;
    q.fix_off = fix_off.as<uint32_t>();
    q.fix_list = fix_list.as<uint32_t>();
    // ... and by the target's 128-item owner tile, ascending within a tile:
    // the dE epilogue walks them to leave each target entry out of G
    target_keys<<<ceil_div(n, 256), 256, 0, st>>>(tgt.as<int32_t>(), n, item_tiles, keys.as<int64_t>(), 7);
    LF_LAUNCHED();
    rc = sort_by_item(keys.as<int64_t>(), n, item_tiles + 1, hit_list, hit_off, st);
    if (!rc) rc = hits.alloc(sizeof(uint64_t) * n, st);
    if (rc) return rc;
    pack_hits<<<ceil_div(n, 256), 256, 0, st>>>(hit_list.as<uint32_t>(), tgt.as<int32_t>(), n,
                                                hits.as<uint64_t>());
    LF_LAUNCHED();
    q.hit_off = hit_off.as<uint32_t>();
    q.hit_list = hits.as<uint64_t>();
  }
  // bias columns folding -lse2 into the dE pass's S MMA (see bias_columns)
  Scratch bias, ones;
  rc = bias.alloc(sizeof(__nv_bfloat16) * 16 * n_pad, st);
  if (!rc) rc = ones.alloc(sizeof(__nv_bfloat16) * 16 * BM, st);
  if (rc) return rc;
  bias_columns<<<ceil_div(n_pad, 256), 256, 0, st>>>(lse, n, n_pad, sub, bias.as<__nv_bfloat16>(),
                                                     ones.as<__nv_bfloat16>());
  LF_LAUNCHED();
  CUtensorMap mbias, mones;
  rc = make_map_k16(&mbias, bias.ptr, n_pad, BNi);
  if (!rc) rc = make_map_k16(&mones, ones.ptr, BM, BM);
  if (rc) return rc;
  rc = launch_d<BWD_ITEMS>(D, dX ? (flags & ~kCount) : flags, me_own, mx_str, mbias, mones, q, st);
  return rc;
}

}  // namespace lf
