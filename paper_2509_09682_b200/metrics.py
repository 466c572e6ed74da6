"""Full-catalog evaluation on the GPU — lseforge::evaluate (metrics.hpp:12-24,
metrics.cpp:13-103) with the encoder left to the caller.

The reference scores every eval pair against the whole catalog in double,
ranks the target (ties to the smaller item id) and aggregates NDCG@k,
coverage@k and surprisal@k.  Here the scores X.E^T are never materialised:
the ranking runs fused in liblseforge_b200.so (tcgen05 kernel for bf16,
fp32/fp64 CUDA-core kernels; fp64 reproduces the reference bit for bit).

    X [n, d]  encoded rows h (encode(), metrics.cpp:46)
    E [v, d]  item rows (the reference's classifier C transposed)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Tuple

import torch

from . import _capi
from .cce import _stream
from .losses import lf_dtype


@dataclass
class EvalSummary:
    """metrics.hpp:12-16."""
    ndcg: float = 0.0
    coverage: float = 0.0
    surprisal: float = 0.0


def _dev(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"evaluate: {name} must be a CUDA device tensor")


def rank_topk(X: torch.Tensor, E: torch.Tensor, targets: torch.Tensor, k: int,
              v_offset: int = 0, target_rows: Optional[torch.Tensor] = None
              ) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Over the catalog shard E (items v_offset .. v_offset + len(E)):
    (ahead [n] int64 — items ranked ahead of the target, metrics.cpp:56-60;
    top_idx [n, k] int64 global ids, -1 past the shard; top_score [n, k]
    float64).  target_rows [n, d] supplies each row's target item row when the
    target may lie in another shard."""
    for t, nm in ((X, "X"), (E, "E"), (targets, "targets")):
        _dev(t, nm)
    if X.dtype != E.dtype:
        raise ValueError("evaluate: X and E must share a dtype")
    n, d = X.shape
    X, E = X.contiguous(), E.contiguous()
    tg = targets.to(torch.int64).contiguous()
    tr = None
    if target_rows is not None:
        tr = target_rows.to(X.dtype).contiguous()
    ahead = torch.empty(n, dtype=torch.int64, device=X.device)
    top = torch.empty((n, k), dtype=torch.int64, device=X.device)
    score = torch.empty((n, k), dtype=torch.float64, device=X.device)
    _capi.check(_capi.lib().lf_eval_rank_topk(
        X.data_ptr(), E.data_ptr(), tg.data_ptr(), tr.data_ptr() if tr is not None else None, n, d,
        E.shape[0], int(v_offset), int(k), lf_dtype(X), ahead.data_ptr(), top.data_ptr(),
        score.data_ptr(), _stream(X)))
    return ahead, top, score


def merge_shards(ahead: torch.Tensor, top_idx: torch.Tensor, top_score: torch.Tensor
                 ) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Fold P shards' outputs ([P, n], [P, n, k], [P, n, k]) into 1-based ranks
    and the merged global top-k (score desc, id asc)."""
    P, n = ahead.shape
    k = top_idx.shape[2]
    rank = torch.empty(n, dtype=torch.int64, device=ahead.device)
    top = torch.empty((n, k), dtype=torch.int64, device=ahead.device)
    score = torch.empty((n, k), dtype=torch.float64, device=ahead.device)
    _capi.check(_capi.lib().lf_eval_merge(
        ahead.contiguous().data_ptr(), top_idx.contiguous().data_ptr(),
        top_score.contiguous().data_ptr(), P, n, k, rank.data_ptr(), top.data_ptr(),
        score.data_ptr(), _stream(ahead)))
    return rank, top, score


def summarize(rank: torch.Tensor, top_idx: torch.Tensor, popularity: torch.Tensor) -> EvalSummary:
    """metrics.cpp:26-33, 62, 74-103 from 1-based ranks and the top-k_eff lists."""
    _dev(rank, "rank")
    pop = popularity.to(device=rank.device, dtype=torch.int64).contiguous()
    n, k = top_idx.shape
    out = (C.c_double * 3)()
    _capi.check(_capi.lib().lf_eval_summary(rank.contiguous().data_ptr(),
                                            top_idx.contiguous().data_ptr(), n, k, pop.data_ptr(),
                                            pop.numel(), out, _stream(rank)))
    return EvalSummary(out[0], out[1], out[2])


def evaluate(X: torch.Tensor, E: torch.Tensor, targets: torch.Tensor, k: int,
             popularity: torch.Tensor) -> EvalSummary:
    """lseforge::evaluate(params, pairs, k, popularity_counts) for encoded rows
    X: k_eff = min(k, v); ValueError for the reference's invalid_argument cases."""
    for t, nm in ((X, "X"), (E, "E"), (targets, "targets")):
        _dev(t, nm)
    if popularity.numel() != E.shape[0]:
        raise ValueError("evaluate: popularity table size does not match the catalog")
    n, d = X.shape
    pop = popularity.to(device=X.device, dtype=torch.int64).contiguous()
    tg = targets.to(torch.int64).contiguous()
    out = (C.c_double * 3)()
    _capi.check(_capi.lib().lf_evaluate(X.contiguous().data_ptr(), E.contiguous().data_ptr(),
                                        tg.data_ptr(), n, d, E.shape[0], int(k), lf_dtype(X),
                                        pop.data_ptr(), out, _stream(X)))
    return EvalSummary(out[0], out[1], out[2])
