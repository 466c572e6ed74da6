"""ctypes bindings for the CPU checkers under oracle/ (TEST INFRASTRUCTURE).

Two libraries:
  * ``oracle/liboracle.so``            — the C restatement (oracle/oracle.c)
  * ``oracle/_ref/liblseforge_ref.so`` — the unmodified reference hot-path sources
                                          compiled in place (oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  Layouts are the reference's: E n×d float32, C d×v float32,
outputs float64 (proj/include/lseforge/losses.hpp:15-27).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "liblseforge_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_sz = C.c_size_t


def _load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    return C.CDLL(path)


class _Rng(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("state", C.c_uint64)]


_orc = None


def orc():
    global _orc
    if _orc is None:
        L = _load(ORACLE_SO)
        L.orc_rng_init.argtypes = [C.POINTER(_Rng), C.c_uint64]
        L.orc_rng_next.argtypes = [C.POINTER(_Rng)]
        L.orc_rng_next.restype = C.c_uint64
        L.orc_rng_bounded.argtypes = [C.POINTER(_Rng), C.c_uint64]
        L.orc_rng_bounded.restype = C.c_uint64
        L.orc_rng_uniform.argtypes = [C.POINTER(_Rng)]
        L.orc_rng_uniform.restype = C.c_double
        L.orc_make_instance.argtypes = [C.POINTER(_Rng), _sz, _sz, _sz, C.c_double, _f32p, _f32p, _i64p]
        L.orc_make_candidates.argtypes = [C.POINTER(_Rng), _i64p, _sz, _sz, _sz, _i64p]
        L.orc_sample_uniform.argtypes = [_i64p, _sz, _sz, _sz, C.c_uint64, C.c_int, _i64p]
        L.orc_sample_uniform.restype = C.c_int
        L.orc_cce_forward.argtypes = [_f32p, _f32p, _i64p, _sz, _sz, _sz, _f64p, _f64p]
        L.orc_cce_forward.restype = C.c_double
        L.orc_cce_backward.argtypes = [_f32p, _f32p, _i64p, _f64p, C.c_double, C.c_double, _sz,
                                       _sz, _sz, _sz, _f64p, _f64p, C.POINTER(C.c_uint64)]
        L.orc_cce_backward.restype = C.c_double
        L.orc_cce_forward_partial.argtypes = [_f32p, _f32p, _i64p, _sz, _sz, _sz, _sz, _sz,
                                              _f64p, _f64p, _f64p, _i32p]
        L.orc_ccem_forward.argtypes = [_f32p, _f32p, _i64p, _sz, _sz, _sz, _sz, _f64p, _f64p]
        L.orc_ccem_forward.restype = C.c_double
        L.orc_ccem_backward_rows.argtypes = [_f32p, _f32p, _i64p, _f64p, _f64p, _sz, _sz, _sz, _sz,
                                             _f64p, _f64p]
        L.orc_validate_targets.argtypes = [_i64p, _sz, _sz]
        L.orc_validate_targets.restype = C.c_int64
        L.orc_validate_inds.argtypes = [_i64p, _sz, _sz, _sz]
        L.orc_validate_inds.restype = C.c_int64
        L.orc_estimate_flops.argtypes = [_sz, _sz, _sz, _sz, C.c_int, C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64)]
        L.orc_eval_rank_topk.argtypes = [_f64p, _f32p, _i64p, _sz, _sz, _sz, _sz, _sz, _sz,
                                         _i64p, _i64p, _f64p]
        L.orc_eval_summary.argtypes = [_i64p, _i64p, _sz, _sz, _i64p, _sz, _f64p]
        L.orc_eval_summary.restype = C.c_int
        L.orc_encode_batch.argtypes = [_i64p, _i64p, _sz, _f32p, _f32p, _f32p, _sz, _f64p, _f64p,
                                       _f32p, _i64p, _i64p]
        L.orc_encoder_backward.argtypes = [_i64p, _i64p, _sz, _f32p, _sz, _sz, _f64p, _f64p, _i64p,
                                           _sz, _f64p, _f64p, _f64p, _f64p]
        L.orc_sample_popularity.argtypes = [_i64p, _sz, _sz, _i64p, _sz, C.c_double, C.c_uint64,
                                            C.c_int, _i64p]
        L.orc_sample_popularity.restype = C.c_int
        L.orc_adam_apply.argtypes = [_f32p, _f64p, _f64p, _f64p, _sz, C.c_double, C.c_double,
                                     C.c_double, C.c_double, C.c_uint64]
        _orc = L
    return _orc


_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        L = _load(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_stream.argtypes = [C.c_uint64, _u64p, C.c_int]
        L.ref_make_instance.argtypes = [C.c_uint64, _sz, _sz, _sz, C.c_double, _f32p, _f32p, _i64p]
        L.ref_make_instance_candidates.argtypes = [C.c_uint64, _sz, _sz, _sz, _sz, _f32p, _f32p,
                                                   _i64p, _i64p]
        L.ref_sample_uniform.argtypes = [_i64p, _sz, _sz, _sz, C.c_uint64, _i64p]
        L.ref_cce_forward.argtypes = [_f32p, _f32p, _i64p, _sz, _sz, _sz, _sz, _sz, C.c_int,
                                      _f64p, _f64p, C.POINTER(C.c_double)]
        L.ref_cce_backward.argtypes = [_f32p, _f32p, _i64p, _f64p, C.c_double, C.c_double, _sz,
                                       _sz, _sz, _sz, _sz, C.c_int, _f64p, _f64p,
                                       C.POINTER(C.c_double)]
        L.ref_ccem_forward.argtypes = [_f32p, _f32p, _i64p, _sz, _sz, _sz, _sz, _sz, C.c_int,
                                       _f64p, _f64p, C.POINTER(C.c_double)]
        L.ref_ccem_backward_rows.argtypes = [_f32p, _f32p, _i64p, _f64p, _f64p, _sz, _sz, _sz,
                                             _sz, _sz, C.c_int, _f64p, _f64p]
        L.ref_ce_full.argtypes = [_f32p, _f32p, _i64p, _sz, _sz, _sz, C.c_double, _f64p, _f64p,
                                  C.POINTER(C.c_double), C.c_void_p, C.c_void_p]
        L.ref_ce_sampled.argtypes = [_f32p, _f32p, _i64p, _sz, _sz, _sz, _sz, C.c_double, _f64p,
                                     _f64p, C.POINTER(C.c_double), C.c_void_p, C.c_void_p]
        L.ref_validate_targets.argtypes = [_sz, _sz, _sz, _i64p, _sz]
        L.ref_validate_inds.argtypes = [_i64p, _sz, _sz, _sz]
        L.ref_estimate_flops.argtypes = [_sz, _sz, _sz, _sz, C.c_int, C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64)]
        L.ref_eval_instance.argtypes = [_sz, _sz, C.c_uint64, _sz, _sz, _i64p, _i64p, _sz, _i64p,
                                        C.c_int, _f64p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_sample_popularity.argtypes = [_i64p, _sz, _sz, _i64p, _sz, C.c_double, C.c_uint64,
                                            _i64p]
        L.ref_adam_steps.argtypes = [_sz, _sz, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_int, _f64p, _f32p]
        L.ref_encoder.argtypes = [_sz, _sz, _f32p, _f32p, _f32p, _i64p, _i64p, _sz, _f64p, _f64p,
                                  _f64p, _f32p, _i64p, _f64p, _f64p, _f64p]
        L.ref_encoder_init.argtypes = [_sz, _sz, C.c_uint64, _f32p]
        _ref = L
    return _ref


def _chk(rc, lib):
    if rc != 0:
        raise ValueError(lib.ref_last_error().decode())


# ---------------------------------------------------------------------------
# Restatement (oracle.c) wrappers — numpy in, numpy out
# ---------------------------------------------------------------------------
class Rng:
    """SplitMix64 (rng.hpp:13-60) backed by the C restatement."""

    def __init__(self, seed: int):
        self._s = _Rng()
        orc().orc_rng_init(C.byref(self._s), C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF))

    def next(self) -> int:
        return orc().orc_rng_next(C.byref(self._s))

    def bounded(self, b: int) -> int:
        return orc().orc_rng_bounded(C.byref(self._s), b)

    def uniform(self) -> float:
        return orc().orc_rng_uniform(C.byref(self._s))


@dataclass
class Instance:
    E: np.ndarray        # n×d float32 (reference "E" = B200 "X")
    C: np.ndarray        # d×v float32 (reference "C" = B200 "E"^T)
    targets: np.ndarray  # n int64


def make_instance(rng: Rng, n: int, d: int, v: int, half_width: float = 1.0) -> Instance:
    """support.hpp:27-37, same draw order (E, then C, then targets)."""
    E = np.empty((n, d), np.float32)
    Cm = np.empty((d, v), np.float32)
    t = np.empty(n, np.int64)
    orc().orc_make_instance(C.byref(rng._s), n, d, v, half_width, E, Cm, t)
    return Instance(E, Cm, t)


def make_candidates(rng: Rng, targets: np.ndarray, ns: int, v: int) -> np.ndarray:
    """support.hpp:41-56."""
    n = targets.shape[0]
    inds = np.empty((n, 1 + ns), np.int64)
    orc().orc_make_candidates(C.byref(rng._s), np.ascontiguousarray(targets), n, ns, v, inds)
    return inds


def sample_uniform(positives: np.ndarray, ns: int, catalog: int, seed: int, retry_cap: int = 100):
    """sampler.cpp:44-75 (per-row derived(i) streams)."""
    n = positives.shape[0]
    inds = np.empty((n, 1 + ns), np.int64)
    rc = orc().orc_sample_uniform(np.ascontiguousarray(positives), n, ns, catalog, seed,
                                  retry_cap, inds)
    if rc != 0:
        raise RuntimeError("sampler: retry cap exhausted")
    return inds


def sample_popularity(positives, ns, counts, seed, exponent=1.0, retry_cap=100):
    n = len(positives)
    inds = np.empty((n, 1 + ns), np.int64)
    rc = orc().orc_sample_popularity(np.ascontiguousarray(positives, np.int64), n, ns,
                                     np.ascontiguousarray(counts, np.int64), len(counts), exponent,
                                     seed, retry_cap, inds)
    if rc == -2:
        raise ValueError("sample_popularity: all item weights are zero")
    if rc:
        raise RuntimeError("sampler: retry cap exhausted")
    return inds


def ref_sample_popularity(positives, ns, counts, seed, exponent=1.0):
    L = ref()
    n = len(positives)
    inds = np.empty((n, 1 + ns), np.int64)
    _chk(L.ref_sample_popularity(np.ascontiguousarray(positives, np.int64), n, ns,
                                 np.ascontiguousarray(counts, np.int64), len(counts), exponent, seed,
                                 inds), L)
    return inds


def cce_forward(E, Cm, x):
    n, d = E.shape
    v = Cm.shape[1]
    pos = np.empty(n)
    lse = np.empty(n)
    loss = orc().orc_cce_forward(E, Cm, x, n, d, v, pos, lse)
    return loss, pos, lse


def cce_backward(E, Cm, x, lse, upstream=1.0, eps=0.0, col_block=256):
    n, d = E.shape
    v = Cm.shape[1]
    dE = np.empty((n, d))
    dC = np.empty((d, v))
    sk = C.c_uint64()
    frac = orc().orc_cce_backward(E, Cm, x, np.ascontiguousarray(lse, np.float64), upstream, eps,
                                  col_block, n, d, v, dE, dC, C.byref(sk))
    return dE, dC, frac, sk.value


def cce_forward_partial(E, Cm, x, v0, v1):
    n, d = E.shape
    v = Cm.shape[1]
    m = np.empty(n)
    s = np.empty(n)
    t = np.empty(n)
    h = np.empty(n, np.int32)
    orc().orc_cce_forward_partial(E, Cm, x, n, d, v, v0, v1, m, s, t, h)
    return m, s, t, h


def ccem_forward(E, Cm, inds):
    n, d = E.shape
    v = Cm.shape[1]
    w = inds.shape[1]
    pos = np.empty(n)
    lse = np.empty(n)
    loss = orc().orc_ccem_forward(E, Cm, np.ascontiguousarray(inds), n, d, v, w, pos, lse)
    return loss, pos, lse


def ccem_backward_rows(E, Cm, inds, lse, row_upstream):
    n, d = E.shape
    v = Cm.shape[1]
    w = inds.shape[1]
    dE = np.empty((n, d))
    dC = np.empty((d, v))
    orc().orc_ccem_backward_rows(E, Cm, np.ascontiguousarray(inds),
                                 np.ascontiguousarray(lse, np.float64),
                                 np.ascontiguousarray(row_upstream, np.float64), n, d, v, w, dE,
                                 dC)
    return dE, dC


def ccem_backward(E, Cm, inds, lse, upstream=1.0):
    n = E.shape[0]
    return ccem_backward_rows(E, Cm, inds, lse, np.full(n, upstream / n))


def estimate_flops(n, d, v, ns, backend: int):
    f, b = C.c_uint64(), C.c_uint64()
    orc().orc_estimate_flops(n, d, v, ns, backend, C.byref(f), C.byref(b))
    return f.value, b.value


def eval_rank_topk(H, Cm, targets, k, v0=0, v1=None):
    """metrics.cpp:46-72 over items [v0, v1): (ahead, top_idx, top_score)."""
    n, d = H.shape
    v = Cm.shape[1]
    v1 = v if v1 is None else v1
    ahead = np.empty(n, np.int64)
    top = np.empty((n, k), np.int64)
    score = np.empty((n, k))
    orc().orc_eval_rank_topk(np.ascontiguousarray(H, np.float64), np.ascontiguousarray(Cm, np.float32),
                             np.ascontiguousarray(targets, np.int64), n, d, v, v0, v1, k, ahead,
                             top, score)
    return ahead, top, score


def eval_summary(rank, top, counts):
    """metrics.cpp:26-33, 62, 74-103 -> (ndcg, coverage, surprisal)."""
    n, k = top.shape
    out = np.empty(3)
    rc = orc().orc_eval_summary(np.ascontiguousarray(rank, np.int64), np.ascontiguousarray(top, np.int64),
                                n, k, np.ascontiguousarray(counts, np.int64), len(counts), out)
    if rc == 1:
        raise ValueError("evaluate: negative popularity count")
    if rc == 2:
        raise ValueError("evaluate: popularity table needs at least 2 training events")
    return tuple(out)


def evaluate(H, Cm, targets, k, counts):
    """evaluate() minus the encoder: k_eff = min(k, v) (metrics.cpp:34)."""
    k_eff = min(k, Cm.shape[1])
    ahead, top, _ = eval_rank_topk(H, Cm, targets, k_eff)
    return eval_summary(ahead + 1, top, counts)


def encoder(emb, W, b, items, win_off, dh=None):
    """orc_encode_batch (+ orc_encoder_backward when dh is given).
    Returns dict(a, h, e, targets, row_pos[, d_emb, d_W, d_b])."""
    catalog, d = emb.shape
    nw = len(win_off) - 1
    rows = int(np.sum(np.diff(win_off) - 1))
    out = dict(a=np.empty((rows, d)), h=np.empty((rows, d)), e=np.empty((rows, d), np.float32),
               targets=np.empty(rows, np.int64), row_pos=np.empty(rows, np.int64))
    items = np.ascontiguousarray(items, np.int64)
    win_off = np.ascontiguousarray(win_off, np.int64)
    orc().orc_encode_batch(items, win_off, nw, np.ascontiguousarray(emb, np.float32),
                           np.ascontiguousarray(W, np.float32), np.ascontiguousarray(b, np.float32), d,
                           out["a"], out["h"], out["e"], out["targets"], out["row_pos"])
    if dh is not None:
        out.update(d_emb=np.empty((catalog, d)), d_W=np.empty((d, d)), d_b=np.empty(d))
        orc().orc_encoder_backward(items, win_off, nw, np.ascontiguousarray(W, np.float32), catalog, d,
                                   out["a"], out["h"], out["row_pos"], rows,
                                   np.ascontiguousarray(dh, np.float64), out["d_emb"], out["d_W"],
                                   out["d_b"])
    return out


def adam_apply(param, grad, m, v, lr, b1, b2, eps, t):
    """adam.cpp:22-36 in place on float32 param / float64 m, v (numpy)."""
    orc().orc_adam_apply(param, np.ascontiguousarray(grad, np.float64), m, v, param.size, lr, b1, b2,
                         eps, t)


# ---------------------------------------------------------------------------
# Reference (oracle/_ref) wrappers
# ---------------------------------------------------------------------------
def ref_cce_forward(E, Cm, x, rb=128, cb=256, workers=1):
    L = ref()
    n, d = E.shape
    v = Cm.shape[1]
    pos = np.empty(n)
    lse = np.empty(n)
    loss = C.c_double()
    _chk(L.ref_cce_forward(E, Cm, x, n, d, v, rb, cb, workers, pos, lse, C.byref(loss)), L)
    return loss.value, pos, lse


def ref_cce_backward(E, Cm, x, lse, upstream=1.0, eps=0.0, rb=128, cb=256, workers=1):
    L = ref()
    n, d = E.shape
    v = Cm.shape[1]
    dE = np.empty((n, d))
    dC = np.empty((d, v))
    frac = C.c_double()
    _chk(L.ref_cce_backward(E, Cm, x, np.ascontiguousarray(lse, np.float64), upstream, eps, n, d,
                            v, rb, cb, workers, dE, dC, C.byref(frac)), L)
    return dE, dC, frac.value


def ref_ccem_forward(E, Cm, inds, rb=128, workers=1):
    L = ref()
    n, d = E.shape
    v = Cm.shape[1]
    w = inds.shape[1]
    pos = np.empty(n)
    lse = np.empty(n)
    loss = C.c_double()
    _chk(L.ref_ccem_forward(E, Cm, np.ascontiguousarray(inds), n, d, v, w, rb, workers, pos, lse,
                            C.byref(loss)), L)
    return loss.value, pos, lse


def ref_ccem_backward_rows(E, Cm, inds, lse, row_upstream, rb=128, workers=1):
    L = ref()
    n, d = E.shape
    v = Cm.shape[1]
    w = inds.shape[1]
    dE = np.empty((n, d))
    dC = np.empty((d, v))
    _chk(L.ref_ccem_backward_rows(E, Cm, np.ascontiguousarray(inds),
                                  np.ascontiguousarray(lse, np.float64),
                                  np.ascontiguousarray(row_upstream, np.float64), n, d, v, w, rb,
                                  workers, dE, dC), L)
    return dE, dC


def ref_ce_full(E, Cm, x, upstream=1.0, grads=True):
    L = ref()
    n, d = E.shape
    v = Cm.shape[1]
    pos = np.empty(n)
    lse = np.empty(n)
    loss = C.c_double()
    dE = np.empty((n, d)) if grads else None
    dC = np.empty((d, v)) if grads else None
    _chk(L.ref_ce_full(E, Cm, x, n, d, v, upstream, pos, lse, C.byref(loss),
                       dE.ctypes.data if grads else None, dC.ctypes.data if grads else None), L)
    return loss.value, pos, lse, dE, dC


def ref_ce_sampled(E, Cm, inds, upstream=1.0, grads=True):
    L = ref()
    n, d = E.shape
    v = Cm.shape[1]
    w = inds.shape[1]
    pos = np.empty(n)
    lse = np.empty(n)
    loss = C.c_double()
    dE = np.empty((n, d)) if grads else None
    dC = np.empty((d, v)) if grads else None
    _chk(L.ref_ce_sampled(E, Cm, np.ascontiguousarray(inds), n, d, v, w, upstream, pos, lse,
                          C.byref(loss), dE.ctypes.data if grads else None,
                          dC.ctypes.data if grads else None), L)
    return loss.value, pos, lse, dE, dC


def ref_rng_stream(seed, count=16):
    out = np.empty(count, np.uint64)
    ref().ref_rng_stream(seed, out, count)
    return out


def ref_sample_uniform(positives, ns, catalog, seed):
    L = ref()
    n = positives.shape[0]
    inds = np.empty((n, 1 + ns), np.int64)
    _chk(L.ref_sample_uniform(np.ascontiguousarray(positives), n, ns, catalog, seed, inds), L)
    return inds


def rel_err(got, want):
    """support.hpp:74-77 / acceptance.cpp:69-71: |got-want| / max(1, |want|)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return np.abs(got - want) / np.maximum(1.0, np.abs(want))


def ref_eval_instance(catalog, hidden, seed, prefixes, targets, k, counts, workers=1, extras=True):
    """The reference's evaluate() on ToyEncoderParams::Init(catalog, hidden,
    SplitMix64(seed)): (out3, H, C, ranks) — see oracle/ref_capi.cpp.  With
    extras=False only evaluate() itself runs (timing) and H, C, ranks are None."""
    L = ref()
    prefixes = np.ascontiguousarray(prefixes, np.int64)
    n, Lp = prefixes.shape
    out = np.empty(3)
    H = np.empty((n, hidden)) if extras else None
    Cm = np.empty((hidden, catalog), np.float32) if extras else None
    ranks = np.empty(n, np.int64) if extras else None
    ptr = lambda a: a.ctypes.data if a is not None else None  # noqa: E731
    _chk(L.ref_eval_instance(catalog, hidden, seed, n, Lp, prefixes,
                             np.ascontiguousarray(targets, np.int64), k,
                             np.ascontiguousarray(counts, np.int64), workers, out, ptr(H), ptr(Cm),
                             ptr(ranks)), L)
    return tuple(out), H, Cm, ranks


def ref_adam_steps(catalog, hidden, seed, lr, b1, b2, eps, grads):
    """AdamState::step x len(grads) on ToyEncoderParams::Init; grads[s] is the
    concatenated [d_emb | d_w | d_b | d_classifier] doubles -> final params
    (float32, same order)."""
    L = ref()
    g = np.ascontiguousarray(np.stack(grads), np.float64)
    out = np.empty(g.shape[1], np.float32)
    _chk(L.ref_adam_steps(catalog, hidden, seed, lr, b1, b2, eps, len(grads), g.reshape(-1), out), L)
    return out


def ref_encoder_init(catalog, hidden, seed):
    L = ref()
    out = np.empty(catalog * hidden * 2 + hidden * hidden + hidden, np.float32)
    _chk(L.ref_encoder_init(catalog, hidden, seed, out), L)
    return out


def ref_encoder(emb, W, b, items, win_off, dh):
    """The reference's encode_batch + encoder_backward (oracle/_ref)."""
    L = ref()
    catalog, d = emb.shape
    rows = int(np.sum(np.diff(win_off) - 1))
    out = dict(a=np.empty((rows, d)), h=np.empty((rows, d)), e=np.empty((rows, d), np.float32),
               targets=np.empty(rows, np.int64), d_emb=np.empty((catalog, d)), d_W=np.empty((d, d)),
               d_b=np.empty(d))
    _chk(L.ref_encoder(catalog, d, np.ascontiguousarray(emb, np.float32), np.ascontiguousarray(W, np.float32),
                       np.ascontiguousarray(b, np.float32), np.ascontiguousarray(items, np.int64),
                       np.ascontiguousarray(win_off, np.int64), len(win_off) - 1,
                       np.ascontiguousarray(dh, np.float64), out["a"], out["h"], out["e"], out["targets"],
                       out["d_emb"], out["d_W"], out["d_b"]), L)
    return out
