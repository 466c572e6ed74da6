"""The toy sequence encoder around the loss, on the device —
lseforge::encode_batch / encoder_backward (encoder.hpp:46-66,
encoder.cpp:64-173), so a training step (trainer.cpp:209-227: encode ->
loss -> encoder backward -> Adam) never leaves the GPU.

Windows are a CSR on the device: ``items[win_off[w]:win_off[w+1]]``.  Params
in the reference layout: emb [catalog, d], W [d, d], b [d] (float32).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _capi
from .cce import _stream
from .losses import DTYPES


@dataclass
class EncodedBatch:
    """encoder.hpp:50-57 (plus the window CSR it was built from)."""
    X: torch.Tensor           # [rows, d] the loss input (float(h) in the requested dtype)
    a: torch.Tensor           # [rows, d] float64 pooled means
    h: torch.Tensor           # [rows, d] float64 tanh outputs
    targets: torch.Tensor     # [rows] int64
    window_of: torch.Tensor   # [rows] int64
    position_of: torch.Tensor  # [rows] int64 (1-based prefix length)
    items: torch.Tensor
    win_off: torch.Tensor


def encode_batch(emb: torch.Tensor, W: torch.Tensor, b: torch.Tensor, items: torch.Tensor,
                 win_off: torch.Tensor, x_dtype: torch.dtype = torch.bfloat16) -> EncodedBatch:
    """encoder.cpp:64-116.  ValueError with the reference's messages."""
    catalog, d = emb.shape
    items = items.to(torch.int64).contiguous()
    win_off = win_off.to(torch.int64).contiguous()
    rows = int((win_off[1:] - win_off[:-1] - 1).clamp_min(0).sum())
    dev = emb.device
    X = torch.empty((rows, d), dtype=x_dtype, device=dev)
    a = torch.empty((rows, d), dtype=torch.float64, device=dev)
    h = torch.empty((rows, d), dtype=torch.float64, device=dev)
    tg = torch.empty(rows, dtype=torch.int64, device=dev)
    rw = torch.empty(rows, dtype=torch.int64, device=dev)
    rp = torch.empty(rows, dtype=torch.int64, device=dev)
    _capi.check(_capi.lib().lf_encode_batch(
        items.data_ptr(), win_off.data_ptr(), win_off.numel() - 1, emb.contiguous().data_ptr(),
        W.contiguous().data_ptr(), b.contiguous().data_ptr(), catalog, d, rows, DTYPES[x_dtype],
        X.data_ptr(), a.data_ptr(), h.data_ptr(), tg.data_ptr(), rw.data_ptr(), rp.data_ptr(),
        _stream(emb)))
    return EncodedBatch(X, a, h, tg, rw, rp, items, win_off)


def encoder_backward(catalog: int, W: torch.Tensor, batch: EncodedBatch, d_h: torch.Tensor):
    """encoder.cpp:118-173: (d_emb [catalog, d], d_W [d, d], d_b [d]) float64
    from d_h = the loss's dX [rows, d] (float32 or float64)."""
    d = W.shape[0]
    rows = batch.a.shape[0]
    if d_h.shape != (rows, d):
        raise ValueError("encoder_backward: d_h shape does not match the batch")
    dh = d_h.contiguous()
    if dh.dtype not in (torch.float32, torch.float64):
        dh = dh.float()
    dev = W.device
    d_emb = torch.empty((catalog, d), dtype=torch.float64, device=dev)
    d_W = torch.empty((d, d), dtype=torch.float64, device=dev)
    d_b = torch.empty(d, dtype=torch.float64, device=dev)
    _capi.check(_capi.lib().lf_encoder_backward(
        batch.items.data_ptr(), batch.win_off.data_ptr(), batch.win_off.numel() - 1,
        W.contiguous().data_ptr(), catalog, d, batch.a.data_ptr(), batch.h.data_ptr(),
        batch.position_of.data_ptr(), rows, dh.data_ptr(), DTYPES[dh.dtype], d_emb.data_ptr(),
        d_W.data_ptr(), d_b.data_ptr(), _stream(W)))
    return d_emb, d_W, d_b
