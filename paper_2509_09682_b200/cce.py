"""Cut Cross-Entropy (full catalog) — B200 drop-in for lseforge::cce_forward /
cce_backward (proj/include/lseforge/cce.hpp:36-54, proj/src/cce.cpp).

Element type follows X/E: bfloat16 -> tcgen05 tensor-core kernels, float32 ->
FFMA kernels, float64 -> "exact" kernels in the reference's operand order.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch

from . import _capi
from .accountant import MemAccountant
from .losses import (GradPair, LossOutput, grad_dtype, lf_dtype, validate_loss_inputs)

kFp16MinPositive = 6e-8  # cce.hpp:15


@dataclass
class CceConfig:
    """cce.hpp:18-31.  row_block / col_block / workers are CPU tiling knobs; the
    GPU accepts and ignores them (results never depend on them)."""
    row_block: int = 128
    col_block: int = 256
    filter_eps: float = 0.0
    workers: int = 0
    atomic_de: bool = False  # CCE- only: LF_FLAG_ATOMIC_DE
    filter_dx: bool = False  # cce_forward_backward: filter dX too (LF_FLAG_FILTER_DX)

    @staticmethod
    def Fp16SaturationPreset() -> "CceConfig":  # cce.hpp:26-30
        return CceConfig(filter_eps=kFp16MinPositive)

    def validate(self):  # cce.cpp:17-27
        if self.row_block < 1 or self.col_block < 1:
            raise ValueError(f"CceConfig: block sizes must be >= 1 (row_block={self.row_block}, "
                             f"col_block={self.col_block})")
        if not (self.filter_eps >= 0.0):
            raise ValueError(f"CceConfig: filter_eps must be >= 0, got {self.filter_eps:f}")

    def to_c(self, dtype: int) -> _capi.CceConfigC:
        return _capi.CceConfigC(float(self.filter_eps), dtype,
                                (_capi.LF_FLAG_ATOMIC_DE if self.atomic_de else 0)
                                | (_capi.LF_FLAG_FILTER_DX if self.filter_dx else 0))


@dataclass
class CceBackwardResult:
    """cce.hpp:40-45 plus the tile statistics of the B200 kernel."""
    grads: GradPair
    skipped_fraction: Optional[float] = None
    skipped_tiles: Optional[int] = None
    total_tiles: Optional[int] = None


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _charge_scratch(acct: Optional[MemAccountant], tag: str, before_peak: int):
    if acct is None:
        return
    cur, peak = C.c_uint64(), C.c_uint64()
    _capi.lib().lf_workspace_stats(C.byref(cur), C.byref(peak))
    scalars = max(1, (int(peak.value) - before_peak + 3) // 4)
    acct.record_alloc(tag, scalars)
    acct.record_free(tag, scalars)


def _reset_peak() -> int:
    L = _capi.lib()
    L.lf_workspace_reset_peak()
    cur, peak = C.c_uint64(), C.c_uint64()
    L.lf_workspace_stats(C.byref(cur), C.byref(peak))
    return int(peak.value)


def cce_forward(X: torch.Tensor, E: torch.Tensor, x: torch.Tensor, cfg: CceConfig = CceConfig(),
                acct: Optional[MemAccountant] = None, validate: bool = True) -> LossOutput:
    """cce.cpp:65-145: per-row lse and target logit; mean loss.  X [n,d], E [v,d]."""
    validate_loss_inputs(X, E, x, check_range=validate)
    cfg.validate()
    n, d = X.shape
    v = E.shape[0]
    if acct is not None:
        acct.record_ensure("retained/cce/pos_logits", n)  # cce.cpp:81-82
        acct.record_ensure("retained/cce/lse", n)
    base = _reset_peak() if acct is not None else 0
    lse = torch.empty(n, dtype=torch.float64, device=X.device)
    pos = torch.empty(n, dtype=torch.float64, device=X.device)
    loss = torch.empty((), dtype=torch.float64, device=X.device)
    c = cfg.to_c(lf_dtype(X))
    _capi.check(_capi.lib().lf_cce_forward(X.data_ptr(), E.data_ptr(), x.data_ptr(), n, d, v,
                                           C.byref(c), lse.data_ptr(), pos.data_ptr(),
                                           loss.data_ptr(), _stream(X)))
    _charge_scratch(acct, "scratch/cce/forward", base)
    return LossOutput(loss, pos, lse)


def cce_backward(X: torch.Tensor, E: torch.Tensor, x: torch.Tensor, lse: torch.Tensor,
                 upstream: float = 1.0, cfg: CceConfig = CceConfig(),
                 acct: Optional[MemAccountant] = None, validate: bool = True,
                 stats: bool = True) -> CceBackwardResult:
    """cce.cpp:147-272: dX = G E, dE = G^T X with G = softmax - onehot, scaled by
    upstream / n and filtered below cfg.filter_eps.  ``stats=True`` reads the
    skip counters back (one stream sync); ``stats=False`` never syncs."""
    validate_loss_inputs(X, E, x, check_range=validate)
    cfg.validate()
    n, d = X.shape
    v = E.shape[0]
    if lse.numel() != n:  # cce.cpp:153-156
        raise ValueError(f"cce_backward: LSE vector has {lse.numel()} entries for {n} rows")
    lse = lse.to(dtype=torch.float64).contiguous()
    if acct is not None:
        acct.record_ensure("retained/cce/lse", n)
    base = _reset_peak() if acct is not None else 0
    gd = grad_dtype(X)
    dX = torch.empty((n, d), dtype=gd, device=X.device)
    dE = torch.empty((v, d), dtype=gd, device=X.device)
    c = cfg.to_c(lf_dtype(X))
    st = _capi.CceStatsC()
    _capi.check(_capi.lib().lf_cce_backward(X.data_ptr(), E.data_ptr(), x.data_ptr(),
                                            lse.data_ptr(), float(upstream), n, d, v, C.byref(c),
                                            dX.data_ptr(), dE.data_ptr(),
                                            C.byref(st) if stats else None, _stream(X)))
    _charge_scratch(acct, "scratch/cce/backward", base)
    res = CceBackwardResult(GradPair(dX, dE))
    if stats:
        res.skipped_fraction = float(st.skipped_fraction)
        res.skipped_tiles = int(st.skipped_tiles)
        res.total_tiles = int(st.total_tiles)
    return res


def cce_forward_backward(X: torch.Tensor, E: torch.Tensor, x: torch.Tensor, upstream: float = 1.0,
                         cfg: CceConfig = CceConfig(), acct: Optional[MemAccountant] = None,
                         validate: bool = True, stats: bool = False):
    """cce_forward then cce_backward(lse, upstream) on the same inputs — the
    pair run_loss_layer issues (trainer.cpp:71-77) — as one call
    (lf_cce_forward_backward).  bf16 with d = 64 / 128 / 256 and filter_eps < 2^-12
    runs the fused kernel: the LSE and dX's softmax-weighted item sum in one
    pass over the logits, then the dE pass; dX is then the unfiltered
    gradient (each dropped entry is below eps), dE and the skip statistics
    follow the filter.  Returns (LossOutput, CceBackwardResult)."""
    validate_loss_inputs(X, E, x, check_range=validate)
    cfg.validate()
    n, d = X.shape
    v = E.shape[0]
    if acct is not None:
        acct.record_ensure("retained/cce/pos_logits", n)  # cce.cpp:81-82
        acct.record_ensure("retained/cce/lse", n)
    base = _reset_peak() if acct is not None else 0
    lse = torch.empty(n, dtype=torch.float64, device=X.device)
    pos = torch.empty(n, dtype=torch.float64, device=X.device)
    loss = torch.empty((), dtype=torch.float64, device=X.device)
    gd = grad_dtype(X)
    dX = torch.empty((n, d), dtype=gd, device=X.device)
    dE = torch.empty((v, d), dtype=gd, device=X.device)
    c = cfg.to_c(lf_dtype(X))
    st = _capi.CceStatsC()
    _capi.check(_capi.lib().lf_cce_forward_backward(
        X.data_ptr(), E.data_ptr(), x.data_ptr(), n, d, v, float(upstream), C.byref(c),
        lse.data_ptr(), pos.data_ptr(), loss.data_ptr(), dX.data_ptr(), dE.data_ptr(),
        C.byref(st) if stats else None, _stream(X)))
    _charge_scratch(acct, "scratch/cce/forward_backward", base)
    res = CceBackwardResult(GradPair(dX, dE))
    if stats:
        res.skipped_fraction = float(st.skipped_fraction)
        res.skipped_tiles = int(st.skipped_tiles)
        res.total_tiles = int(st.total_tiles)
    return LossOutput(loss, pos, lse), res
