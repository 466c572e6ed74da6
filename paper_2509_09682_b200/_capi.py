"""ctypes binding of liblseforge_b200.so (include/lseforge_b200.h).

The shared library is built in-tree (``make -C paper_2509_09682_b200``, or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
every entry point raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# LSEFORGE_B200_LIB selects an alternative in-tree build (tuning variants).
LIB_PATH = os.environ.get("LSEFORGE_B200_LIB") or os.path.join(_HERE, "liblseforge_b200.so")

LF_OK, LF_EINVAL, LF_EUNSUPPORTED, LF_ECUDA, LF_ENOMEM, LF_ERUNTIME = 0, -1, -2, -3, -4, -5
LF_F32, LF_F64, LF_BF16 = 0, 1, 2
LF_FLAG_NONE, LF_FLAG_ATOMIC_DE, LF_FLAG_FILTER_DX = 0, 1, 2

# Every symbol include/lseforge_b200.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "lf_abi_version", "lf_last_error", "lf_cce_forward", "lf_cce_backward",
    "lf_cce_forward_partial", "lf_cce_combine", "lf_cce_backward_shard", "lf_ccem_forward",
    "lf_ccem_backward", "lf_validate_targets", "lf_validate_inds", "lf_estimate_flops",
    "lf_workspace_stats", "lf_workspace_reset_peak", "lf_launch_count", "lf_launch_count_reset",
    "lf_profile_enable", "lf_profile_read", "lf_profile_reset", "lf_classifier_to_items",
    "lf_convert_rows", "lf_items_grad_to_classifier", "lf_widen_grad", "lf_sample_uniform",
    "lf_ce_forward", "lf_ce_backward", "lf_eval_rank_topk", "lf_eval_merge", "lf_eval_summary",
    "lf_evaluate", "lf_adam_step", "lf_encode_batch", "lf_encoder_backward", "lf_peer_alloc",
    "lf_peer_open", "lf_peer_close", "lf_peer_free", "lf_peer_barrier", "lf_peer_sum",
    "lf_cce_forward_partial_peer", "lf_cce_backward_shard_peer", "lf_sample_popularity",
    "lf_cem_forward", "lf_cem_backward", "lf_cce_forward_backward", "lf_cce_fused_supported",
    "lf_comm_nccl", "lf_peer_comm_handle_bytes", "lf_peer_comm_create", "lf_peer_comm_open",
    "lf_peer_comm_abort", "lf_peer_comm_status", "lf_peer_comm_destroy", "lf_cce_forward_sharded",
    "lf_cce_backward_sharded", "lf_cce_forward_backward_sharded", "lf_cce_fwdx_shard_begin",
    "lf_cce_fwdx_shard_end", "lf_cce_work_free", "lf_peer_status", "lf_ccem_forward_backward",
)
KERNEL_KINDS = ("cce_fwd", "cce_bwd_dx", "cce_bwd_de", "cce_simt", "ccem_fwd", "ccem_bwd", "aux",
                "eval", "cce_fwd_dx")


class CceConfigC(C.Structure):
    _fields_ = [("filter_eps", C.c_double), ("dtype", C.c_int32), ("flags", C.c_int32)]


class CceStatsC(C.Structure):
    _fields_ = [("skipped_elems", C.c_uint64), ("skipped_tiles", C.c_uint64),
                ("total_tiles", C.c_uint64), ("skipped_fraction", C.c_double)]


class LfError(RuntimeError):
    """Raised for LF_ECUDA / LF_ENOMEM / LF_EUNSUPPORTED statuses."""


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {_HERE}` or "
                "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i64, dp = C.c_void_p, C.c_int64, C.c_void_p
        cfgp = C.POINTER(CceConfigC)
        stp = C.POINTER(CceStatsC)
        L.lf_abi_version.restype = C.c_int
        L.lf_last_error.restype = C.c_char_p
        L.lf_cce_forward.argtypes = [vp, vp, vp, i64, i64, i64, cfgp, dp, dp, dp, vp]
        L.lf_cce_backward.argtypes = [vp, vp, vp, dp, C.c_double, i64, i64, i64, cfgp, vp, vp,
                                      stp, vp]
        L.lf_cce_forward_backward.argtypes = [vp, vp, vp, i64, i64, i64, C.c_double, cfgp, dp, dp,
                                              dp, vp, vp, stp, vp]
        L.lf_cce_fused_supported.argtypes = [cfgp, i64]
        L.lf_cce_fwdx_shard_begin.argtypes = [vp, vp, vp, i64, i64, i64, i64, cfgp, vp,
                                              C.POINTER(C.c_void_p), vp]
        L.lf_cce_fwdx_shard_end.argtypes = [vp, vp, C.c_int32, C.c_double, i64, dp, dp, dp, vp, vp,
                                            stp, vp]
        L.lf_cce_work_free.argtypes = [vp]
        L.lf_cce_forward_partial.argtypes = [vp, vp, vp, i64, i64, i64, i64, cfgp, vp, vp]
        L.lf_cce_combine.argtypes = [vp, C.c_int32, i64, dp, dp, dp, vp]
        L.lf_cce_backward_shard.argtypes = [vp, vp, vp, dp, C.c_double, i64, i64, i64, i64, i64,
                                            cfgp, vp, vp, stp, vp]
        L.lf_ccem_forward.argtypes = [vp, vp, vp, i64, i64, i64, i64, cfgp, dp, dp, dp, vp]
        L.lf_ccem_backward.argtypes = [vp, vp, vp, dp, dp, C.c_double, i64, i64, i64, i64, cfgp,
                                       vp, vp, vp]
        L.lf_ccem_forward_backward.argtypes = [vp, vp, vp, i64, i64, i64, i64, dp, C.c_double,
                                               cfgp, dp, dp, dp, vp, vp, vp]
        L.lf_validate_targets.argtypes = [vp, i64, i64, vp]
        L.lf_validate_inds.argtypes = [vp, i64, i64, i64, vp]
        L.lf_estimate_flops.argtypes = [i64, i64, i64, i64, C.c_int32, C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_uint64)]
        L.lf_workspace_stats.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.lf_sample_uniform.argtypes = [vp, i64, i64, i64, C.c_uint64, C.c_int32, vp, vp]
        L.lf_ce_forward.argtypes = [vp, vp, vp, i64, i64, i64, cfgp, dp, dp, dp, vp]
        L.lf_ce_backward.argtypes = [vp, vp, vp, C.c_double, i64, i64, i64, cfgp, vp, vp, vp]
        L.lf_classifier_to_items.argtypes = [vp, i64, i64, C.c_int32, vp, vp]
        L.lf_convert_rows.argtypes = [vp, i64, C.c_int32, vp, vp]
        L.lf_items_grad_to_classifier.argtypes = [vp, C.c_int32, i64, i64, vp, vp]
        L.lf_widen_grad.argtypes = [vp, C.c_int32, i64, vp, vp]
        L.lf_eval_rank_topk.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, C.c_int32, C.c_int32,
                                        vp, vp, vp, vp]
        L.lf_eval_merge.argtypes = [vp, vp, vp, C.c_int32, i64, C.c_int32, vp, vp, vp, vp]
        L.lf_eval_summary.argtypes = [vp, vp, i64, C.c_int32, vp, i64, C.POINTER(C.c_double), vp]
        L.lf_evaluate.argtypes = [vp, vp, vp, i64, i64, i64, C.c_int32, C.c_int32, vp,
                                  C.POINTER(C.c_double), vp]
        L.lf_adam_step.argtypes = [vp, vp, C.c_int32, vp, vp, i64, C.c_double, C.c_double,
                                   C.c_double, C.c_double, i64, vp, C.c_int32, vp]
        L.lf_encode_batch.argtypes = [vp, vp, i64, vp, vp, vp, i64, i64, i64, C.c_int32, vp, vp, vp,
                                      vp, vp, vp, vp]
        L.lf_encoder_backward.argtypes = [vp, vp, i64, vp, i64, i64, vp, vp, vp, i64, vp, C.c_int32,
                                          vp, vp, vp, vp]
        L.lf_peer_alloc.argtypes = [C.c_uint64, C.POINTER(C.c_void_p), C.c_void_p]
        L.lf_peer_open.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
        L.lf_peer_close.argtypes = [vp]
        L.lf_peer_free.argtypes = [vp]
        L.lf_peer_barrier.argtypes = [vp, C.c_int32, C.c_int32, C.c_uint32, vp]
        L.lf_peer_sum.argtypes = [vp, C.c_int32, i64, vp, vp]
        L.lf_cce_forward_partial_peer.argtypes = [vp, vp, vp, i64, i64, i64, i64, cfgp, vp, C.c_int32,
                                                  C.c_int32, i64, vp]
        L.lf_cce_backward_shard_peer.argtypes = [vp, vp, vp, dp, C.c_double, i64, i64, i64, i64, i64,
                                                 cfgp, vp, stp, vp, C.c_int32, C.c_int32, i64, vp]
        L.lf_sample_popularity.argtypes = [vp, i64, i64, vp, i64, C.c_double, C.c_uint64, C.c_int32,
                                           vp, vp]
        L.lf_cem_forward.argtypes = [vp, vp, vp, i64, i64, i64, i64, cfgp, dp, dp, dp, vp]
        L.lf_cem_backward.argtypes = [vp, vp, vp, C.c_double, i64, i64, i64, i64, cfgp, vp, vp, vp]
        L.lf_launch_count.restype = C.c_uint64
        L.lf_profile_enable.argtypes = [C.c_int]
        L.lf_profile_enable.restype = C.c_int
        L.lf_profile_read.argtypes = [C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        L.lf_profile_read.restype = C.c_int
        for name in ("lf_cce_forward", "lf_cce_backward", "lf_cce_forward_partial",
                     "lf_cce_combine", "lf_cce_backward_shard", "lf_ccem_forward",
                     "lf_ccem_backward", "lf_validate_targets", "lf_validate_inds",
                     "lf_estimate_flops", "lf_workspace_stats", "lf_workspace_reset_peak",
                     "lf_sample_uniform", "lf_classifier_to_items", "lf_convert_rows",
                     "lf_items_grad_to_classifier", "lf_widen_grad", "lf_ce_forward",
                     "lf_ce_backward", "lf_eval_rank_topk", "lf_eval_merge", "lf_eval_summary",
                     "lf_evaluate", "lf_adam_step", "lf_encode_batch", "lf_encoder_backward",
                     "lf_peer_alloc", "lf_peer_open", "lf_peer_close", "lf_peer_free",
                     "lf_peer_barrier", "lf_peer_sum", "lf_cce_forward_partial_peer",
                     "lf_cce_backward_shard_peer", "lf_sample_popularity", "lf_cem_forward",
                     "lf_cem_backward", "lf_cce_forward_backward", "lf_cce_fused_supported",
                     "lf_cce_fwdx_shard_begin", "lf_cce_fwdx_shard_end", "lf_cce_work_free",
                     "lf_peer_status", "lf_peer_comm_status", "lf_ccem_forward_backward"):
            getattr(L, name).restype = C.c_int
        if L.lf_abi_version() != 1:
            raise ImportError("liblseforge_b200.so ABI mismatch")
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a status code to the reference's exception types (std::invalid_argument
    -> ValueError)."""
    if rc == LF_OK:
        return
    msg = lib().lf_last_error().decode()
    if rc == LF_EINVAL:
        raise ValueError(msg)
    if rc == LF_ERUNTIME:  # the reference's std::runtime_error cases
        raise RuntimeError(msg)
    raise LfError(f"[status {rc}] {msg}")
