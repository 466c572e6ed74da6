"""Result types and shared input validation of the loss layer.

Mirrors proj/include/lseforge/losses.hpp:15-27 (LossOutput, GradPair) and
losses.cpp:48-69 (validate_loss_inputs) for device tensors.  Naming: the
B200 library calls the hidden states X [n x d] and the item table E [v x d];
the reference calls them E and C (C = E^T, d x v).  ``GradPair.d_embeddings``
is dX [n x d] and ``GradPair.d_classifier`` is dE [v x d] (= reference
d_classifier^T).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch

from . import _capi


@dataclass
class LossOutput:
    """losses.hpp:15-19.  ``loss`` is a 0-d float64 device tensor (no host sync);
    ``float(out.loss)`` reads it."""
    loss: torch.Tensor
    pos_logits: torch.Tensor  # [n] float64
    lse: torch.Tensor         # [n] float64


@dataclass
class GradPair:
    """losses.hpp:24-27 (B200 layout: d_classifier is v x d)."""
    d_embeddings: torch.Tensor
    d_classifier: torch.Tensor


DTYPES = {torch.bfloat16: _capi.LF_BF16, torch.float32: _capi.LF_F32, torch.float64: _capi.LF_F64}


def lf_dtype(t: torch.Tensor) -> int:
    try:
        return DTYPES[t.dtype]
    except KeyError:
        raise ValueError(f"loss: unsupported element type {t.dtype} "
                         "(bfloat16, float32 or float64)") from None


def grad_dtype(t: torch.Tensor) -> torch.dtype:
    return torch.float64 if t.dtype == torch.float64 else torch.float32


def check_device_matrix(name: str, t: torch.Tensor):
    if not isinstance(t, torch.Tensor) or t.dim() != 2:
        raise ValueError(f"loss: {name} must be a 2-D tensor")
    if not t.is_cuda:
        raise ValueError(f"loss: {name} must live on a CUDA device (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"loss: {name} must be contiguous row-major")


def validate_loss_inputs(X: torch.Tensor, E: torch.Tensor, x: torch.Tensor,
                         check_range: bool = True, stream: Optional[int] = None):
    """losses.cpp:48-69 — same messages; the index range scan runs on device
    (lf_validate_targets) and synchronizes."""
    check_device_matrix("hidden states", X)
    check_device_matrix("item embeddings", E)
    if X.shape[0] == 0:
        raise ValueError("loss: embedding matrix has zero rows; the mean loss is undefined")
    if X.shape[1] != E.shape[1]:
        raise ValueError(f"loss: embedding width {X.shape[1]} does not match classifier height "
                         f"{E.shape[1]}")
    if x.dim() != 1 or x.shape[0] != X.shape[0]:
        raise ValueError(f"loss: {x.numel()} targets for {X.shape[0]} embedding rows")
    if x.dtype != torch.int64 or not x.is_cuda or not x.is_contiguous():
        raise ValueError("loss: targets must be a contiguous int64 CUDA tensor")
    if X.dtype != E.dtype:
        raise ValueError(f"loss: X is {X.dtype} but E is {E.dtype}")
    if check_range:
        st = torch.cuda.current_stream(X.device).cuda_stream if stream is None else stream
        _capi.check(_capi.lib().lf_validate_targets(x.data_ptr(), X.shape[0], E.shape[0], st))


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def ce_full_forward(X: torch.Tensor, E: torch.Tensor, x: torch.Tensor,
                    validate: bool = True) -> LossOutput:
    """losses.cpp:71-96 — the MATERIALISING baseline: the n x v logit matrix is
    written to device memory (cuBLAS GEMM) before the row log-sum-exp."""
    import ctypes as C
    validate_loss_inputs(X, E, x, check_range=validate)
    n, d = X.shape
    v = E.shape[0]
    lse = torch.empty(n, dtype=torch.float64, device=X.device)
    pos = torch.empty(n, dtype=torch.float64, device=X.device)
    loss = torch.empty((), dtype=torch.float64, device=X.device)
    c = _capi.CceConfigC(0.0, lf_dtype(X), 0)
    _capi.check(_capi.lib().lf_ce_forward(X.data_ptr(), E.data_ptr(), x.data_ptr(), n, d, v,
                                          C.byref(c), lse.data_ptr(), pos.data_ptr(),
                                          loss.data_ptr(), _stream(X)))
    return LossOutput(loss, pos, lse)


def ce_full_backward(X: torch.Tensor, E: torch.Tensor, x: torch.Tensor, upstream: float = 1.0,
                     validate: bool = True) -> GradPair:
    """losses.cpp:98-140 — recomputes and materialises the logits and an n x v
    coefficient matrix, then two cuBLAS GEMMs for dX and dE."""
    import ctypes as C
    validate_loss_inputs(X, E, x, check_range=validate)
    n, d = X.shape
    v = E.shape[0]
    gd = grad_dtype(X)
    dX = torch.empty((n, d), dtype=gd, device=X.device)
    dE = torch.empty((v, d), dtype=gd, device=X.device)
    c = _capi.CceConfigC(0.0, lf_dtype(X), 0)
    _capi.check(_capi.lib().lf_ce_backward(X.data_ptr(), E.data_ptr(), x.data_ptr(),
                                           float(upstream), n, d, v, C.byref(c), dX.data_ptr(),
                                           dE.data_ptr(), _stream(X)))
    return GradPair(dX, dE)


def ce_sampled_forward(X: torch.Tensor, E: torch.Tensor, inds: torch.Tensor,
                       validate: bool = True) -> LossOutput:
    """losses.cpp:142-173 — the MATERIALISING sampled baseline ("cem"): the
    n x (1+K) candidate logits are written to device memory.  Inputs are
    checked as the reference does (losses.cpp:144-152: row count, widths,
    inds.validate over every slot, the positives included)."""
    import ctypes as C
    from .ccem import _validate_sampled
    _validate_sampled(X, E, inds, validate)
    n, d = X.shape
    v = E.shape[0]
    I = inds.to(torch.int64).contiguous()
    lse = torch.empty(n, dtype=torch.float64, device=X.device)
    pos = torch.empty(n, dtype=torch.float64, device=X.device)
    loss = torch.empty((), dtype=torch.float64, device=X.device)
    c = _capi.CceConfigC(0.0, lf_dtype(X), 0)
    _capi.check(_capi.lib().lf_cem_forward(X.contiguous().data_ptr(), E.contiguous().data_ptr(),
                                           I.data_ptr(), n, d, v, I.shape[1], C.byref(c),
                                           lse.data_ptr(), pos.data_ptr(), loss.data_ptr(), _stream(X)))
    return LossOutput(loss, pos, lse)


def ce_sampled_backward(X: torch.Tensor, E: torch.Tensor, inds: torch.Tensor,
                        upstream: float = 1.0, validate: bool = True) -> GradPair:
    """losses.cpp:175-221 — materialised logits and coefficients, dE scattered
    with atomics (duplicate candidates accumulate).  Checked as
    ce_sampled_forward."""
    import ctypes as C
    from .ccem import _validate_sampled
    _validate_sampled(X, E, inds, validate)
    n, d = X.shape
    v = E.shape[0]
    I = inds.to(torch.int64).contiguous()
    gd = grad_dtype(X)
    dX = torch.empty((n, d), dtype=gd, device=X.device)
    dE = torch.empty((v, d), dtype=gd, device=X.device)
    c = _capi.CceConfigC(0.0, lf_dtype(X), 0)
    _capi.check(_capi.lib().lf_cem_backward(X.contiguous().data_ptr(), E.contiguous().data_ptr(),
                                            I.data_ptr(), float(upstream), n, d, v, I.shape[1],
                                            C.byref(c), dX.data_ptr(), dE.data_ptr(), _stream(X)))
    return GradPair(dX, dE)
