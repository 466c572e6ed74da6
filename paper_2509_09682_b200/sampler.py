"""Negative samplers on the GPU — drop-ins for lseforge::sample_uniform and
sample_popularity (proj/include/lseforge/sampler.hpp, proj/src/sampler.cpp:44-127).

Produces the same N x (1 + ns) int64 index matrix as the reference for the
same positives and SplitMix64 seed (slot 0 = positive), directly on the
device, so CCE- inputs (cfg3: 51 200 x 513) never cross the host link.
"""
from __future__ import annotations

import torch

from . import _capi


def sample_uniform(positives: torch.Tensor, ns: int, catalog: int, seed: int,
                   retry_cap: int = 100) -> torch.Tensor:
    """sampler.cpp:44-75 with SplitMix64(seed) (only the construction seed
    matters: rows use rng.derived(i), rng.hpp:46-48).  ValueError for the
    reference's std::invalid_argument cases, RuntimeError for the retry cap."""
    if not positives.is_cuda:
        raise ValueError("sample_uniform: positives must be a CUDA device tensor")
    pos = positives.to(torch.int64).contiguous()
    n = pos.numel()
    inds = torch.empty((n, 1 + int(ns)), dtype=torch.int64, device=pos.device)
    _capi.check(_capi.lib().lf_sample_uniform(
        pos.data_ptr(), n, int(ns), int(catalog), int(seed) & 0xFFFFFFFFFFFFFFFF, int(retry_cap),
        inds.data_ptr(), torch.cuda.current_stream(pos.device).cuda_stream))
    return inds


def sample_popularity(positives: torch.Tensor, ns: int, counts: torch.Tensor, seed: int,
                      exponent: float = 1.0, retry_cap: int = 100) -> torch.Tensor:
    """sampler.cpp:77-127: inverse CDF over the running sum of count^exponent,
    rows from SplitMix64(seed).derived(i).  Index-for-index the reference's
    output for exponent 1.  ValueError / RuntimeError as the reference."""
    if not positives.is_cuda:
        raise ValueError("sample_popularity: positives must be a CUDA device tensor")
    pos = positives.to(torch.int64).contiguous()
    cnt = counts.to(device=pos.device, dtype=torch.int64).contiguous()
    n = pos.numel()
    inds = torch.empty((n, 1 + int(ns)), dtype=torch.int64, device=pos.device)
    _capi.check(_capi.lib().lf_sample_popularity(
        pos.data_ptr(), n, int(ns), cnt.data_ptr(), cnt.numel(), float(exponent),
        int(seed) & 0xFFFFFFFFFFFFFFFF, int(retry_cap), inds.data_ptr(),
        torch.cuda.current_stream(pos.device).cuda_stream))
    return inds
