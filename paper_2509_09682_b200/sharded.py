"""Catalog-sharded CCE across the GPUs of one node (one process per GPU).

Rank p owns the contiguous item slice [v_begin, v_end) of E (and of dE); X,
targets and the per-row outputs are replicated.  The reference has no
distributed layer (SPEC.md:243 lists vocabulary sharding as a non-goal); this
is the exchange the north star specifies:

  forward   each rank computes per-row partial triples (m, s, t) over its
            slice (lf_cce_forward_partial) -> ONE all-gather of n x 16 bytes
            -> every rank combines them (lf_cce_combine): lse = M + log sum_p
            s_p 2^(m_p - M) (log2 units), pos = the t of the shard that owns
            the target, loss = mean(lse - pos).
  backward  dE rows of the local slice are complete; dX is a partial sum over
            the local items -> ONE all-reduce(sum) of n x d fp32.  The skip
            count is summed across ranks before dividing by n (v_total - 1)
            (cce.cpp:264-268).

The collectives go through torch.distributed (NCCL on GPUs, gloo in the CPU
tests); the kernels behind ``kernels`` are the C-ABI (``DeviceKernels``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Tuple

import torch
import torch.distributed as dist

from . import _capi
from .cce import CceBackwardResult, CceConfig, _stream
from .losses import GradPair, LossOutput, grad_dtype, lf_dtype


def shard_bounds(v_total: int, P: int, p: int) -> Tuple[int, int]:
    """Near-equal contiguous split of [0, v_total) into P slices; slice p."""
    base, rem = divmod(v_total, P)
    begin = p * base + min(p, rem)
    return begin, begin + base + (1 if p < rem else 0)


@dataclass
class ShardStats:
    skipped_elems: int
    skipped_tiles: int
    total_tiles: int


class DeviceKernels:
    """The C-ABI kernels of liblseforge_b200.so on CUDA tensors."""

    def forward_partial(self, X, E_shard, targets, v_offset: int, cfg: CceConfig) -> torch.Tensor:
        n, d = X.shape
        part = torch.empty((n, 4), dtype=torch.float32, device=X.device)
        c = cfg.to_c(lf_dtype(X))
        _capi.check(_capi.lib().lf_cce_forward_partial(
            X.data_ptr(), E_shard.data_ptr(), targets.data_ptr(), n, d, E_shard.shape[0], v_offset,
            C.byref(c), part.data_ptr(), _stream(X)))
        return part

    def combine(self, parts: torch.Tensor) -> LossOutput:
        P, n, _ = parts.shape
        lse = torch.empty(n, dtype=torch.float64, device=parts.device)
        pos = torch.empty(n, dtype=torch.float64, device=parts.device)
        loss = torch.empty((), dtype=torch.float64, device=parts.device)
        _capi.check(_capi.lib().lf_cce_combine(parts.data_ptr(), P, n, lse.data_ptr(),
                                               pos.data_ptr(), loss.data_ptr(), _stream(parts)))
        return LossOutput(loss, pos, lse)

    def backward_shard(self, X, E_shard, targets, lse, upstream, v_offset, v_total, cfg,
                       stats: bool):
        n, d = X.shape
        vs = E_shard.shape[0]
        gd = grad_dtype(X)
        dX = torch.empty((n, d), dtype=gd, device=X.device)
        dE = torch.empty((vs, d), dtype=gd, device=X.device)
        c = cfg.to_c(lf_dtype(X))
        st = _capi.CceStatsC()
        _capi.check(_capi.lib().lf_cce_backward_shard(
            X.data_ptr(), E_shard.data_ptr(), targets.data_ptr(),
            lse.to(torch.float64).contiguous().data_ptr(), float(upstream), n, d, vs, v_offset,
            v_total, C.byref(c), dX.data_ptr(), dE.data_ptr(), C.byref(st) if stats else None,
            _stream(X)))
        s = ShardStats(int(st.skipped_elems), int(st.skipped_tiles), int(st.total_tiles)) if stats else None
        return dX, dE, s


    # ---- the fused step (lf_cce_fwdx_shard_begin / _end) ----
    def fused_supported(self, X, cfg: CceConfig) -> bool:
        c = cfg.to_c(lf_dtype(X))
        return bool(_capi.lib().lf_cce_fused_supported(C.byref(c), X.shape[1]))

    def fwdx_begin(self, X, E_shard, targets, v_offset: int, cfg: CceConfig):
        n, d = X.shape
        part = torch.empty((n, 4), dtype=torch.float32, device=X.device)
        c = cfg.to_c(lf_dtype(X))
        work = C.c_void_p()
        _capi.check(_capi.lib().lf_cce_fwdx_shard_begin(
            X.data_ptr(), E_shard.data_ptr(), targets.data_ptr(), n, d, E_shard.shape[0], v_offset,
            C.byref(c), part.data_ptr(), C.byref(work), _stream(X)))
        return part, work

    def fwdx_end(self, work, parts, X, E_shard, upstream, v_total, stats: bool):
        P, n, _ = parts.shape
        d = X.shape[1]
        lse = torch.empty(n, dtype=torch.float64, device=X.device)
        pos = torch.empty(n, dtype=torch.float64, device=X.device)
        loss = torch.empty((), dtype=torch.float64, device=X.device)
        dX = torch.empty((n, d), dtype=torch.float32, device=X.device)
        dE = torch.empty((E_shard.shape[0], d), dtype=torch.float32, device=X.device)
        st = _capi.CceStatsC()
        _capi.check(_capi.lib().lf_cce_fwdx_shard_end(
            work, parts.data_ptr(), P, float(upstream), v_total, lse.data_ptr(), pos.data_ptr(),
            loss.data_ptr(), dX.data_ptr(), dE.data_ptr(), C.byref(st) if stats else None,
            _stream(X)))
        s = ShardStats(int(st.skipped_elems), int(st.skipped_tiles), int(st.total_tiles)) if stats else None
        return LossOutput(loss, pos, lse), dX, dE, s

    def fwdx_abandon(self, work):
        _capi.lib().lf_cce_work_free(work)


class DeviceEvalKernels:
    """The C-ABI evaluation kernels (metrics.py) on CUDA tensors."""

    def rank_topk(self, X, E_shard, targets, k, v_offset, target_rows):
        from .metrics import rank_topk
        return rank_topk(X, E_shard, targets, k, v_offset, target_rows)

    def merge(self, ahead, top_idx, top_score):
        from .metrics import merge_shards
        return merge_shards(ahead, top_idx, top_score)

    def summarize(self, rank, top_idx, popularity):
        from .metrics import summarize
        return summarize(rank, top_idx, popularity)


class ShardedEval:
    """Catalog-sharded evaluate() (metrics.cpp:13-103): every rank ranks the
    replicated rows against its item slice.  Exchanges: one all-reduce of the
    rows' target item rows (n x d; each target's owner contributes it, so
    every rank scores the target on the same arithmetic path), then one
    all-gather of the per-shard (ahead, top-k ids, top-k scores); ranks add,
    lists merge, and every rank aggregates the same summary."""

    def __init__(self, v_total: int, group=None, kernels=None):
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.v_total = v_total
        self.v_begin, self.v_end = shard_bounds(v_total, self.P, self.rank)
        self.kernels = kernels if kernels is not None else DeviceEvalKernels()

    def target_rows(self, E_shard: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        local = targets.to(torch.int64) - self.v_begin
        mine = (local >= 0) & (local < E_shard.shape[0])
        wire = torch.float64 if E_shard.dtype == torch.float64 else torch.float32
        rows = torch.zeros((targets.numel(), E_shard.shape[1]), dtype=wire, device=E_shard.device)
        rows[mine] = E_shard[local[mine]].to(wire)
        if self.P > 1:
            dist.all_reduce(rows, op=dist.ReduceOp.SUM, group=self.group)
        return rows.to(E_shard.dtype)

    def _gather(self, t: torch.Tensor) -> torch.Tensor:
        if self.P == 1:
            return t.unsqueeze(0)
        flat = torch.empty((self.P * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(flat, t.contiguous(), group=self.group)
        return flat.view((self.P,) + tuple(t.shape))

    def rank_topk(self, X, E_shard, targets, k: int):
        """(1-based rank [n], global top-k ids [n, k], scores [n, k])."""
        if E_shard.shape[0] != self.v_end - self.v_begin:
            raise ValueError(f"sharded eval: rank {self.rank} expects {self.v_end - self.v_begin} "
                             f"item rows, got {E_shard.shape[0]}")
        rows = self.target_rows(E_shard, targets)
        ahead, top, score = self.kernels.rank_topk(X, E_shard, targets, k, self.v_begin, rows)
        return self.kernels.merge(self._gather(ahead), self._gather(top), self._gather(score))

    def evaluate(self, X, E_shard, targets, k: int, popularity):
        if X.shape[0] == 0:
            raise ValueError("evaluate: no eval pairs")
        if k < 1:
            raise ValueError("evaluate: k must be >= 1")
        if popularity.numel() != self.v_total:
            raise ValueError("evaluate: popularity table size does not match the catalog")
        k_eff = min(k, self.v_total)
        rank, top, _ = self.rank_topk(X, E_shard, targets, k_eff)
        return self.kernels.summarize(rank, top, popularity)


class PeerExchange:
    """Exchange buffers every rank maps (CUDA IPC): rank p's buffer holds
    [2 parities][world slots][slot_elems] plus a flag array.  Handles are
    swapped once over the process group (any backend); the data never goes
    through NCCL — the producing kernels store into peers' slots directly and
    lf_peer_barrier orders the exchange on the device."""

    def __init__(self, slot_bytes: int, group=None, device=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.slot_bytes = (int(slot_bytes) + 255) // 256 * 256
        self.half = self.world * self.slot_bytes
        L = _capi.lib()
        self.flag_bytes = 256 * ((4 * self.world + 255) // 256)
        total = self.flag_bytes + 2 * self.half
        base = C.c_void_p()
        handle = (C.c_char * 64)()
        _capi.check(L.lf_peer_alloc(total, C.byref(base), handle))
        self.local = base.value
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=self.group)
        self.bases = []
        for r, h in enumerate(handles):
            if r == self.rank:
                self.bases.append(self.local)
            else:
                ptr = C.c_void_p()
                _capi.check(L.lf_peer_open((C.c_char * 64).from_buffer_copy(h), C.byref(ptr)))
                self.bases.append(ptr.value)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.flags_dev = torch.tensor(self.bases, dtype=torch.int64, device=dev)
        self.slots_dev = torch.tensor([b + self.flag_bytes for b in self.bases], dtype=torch.int64, device=dev)
        self.epoch = 0

    def next_epoch(self):
        self.epoch += 1
        return self.epoch, (self.epoch & 1) * self.half  # byte offset of this epoch's half

    def local_view(self, parity_off: int, shape, dtype=torch.float32):
        """The local buffer's current half as a tensor [world, *shape] (no copy)."""
        numel = self.world * int(torch.Size(shape).numel())
        esize = torch.tensor([], dtype=dtype).element_size()
        ptr = self.local + self.flag_bytes + parity_off
        # wrap the raw device pointer (no copy) through __cuda_array_interface__;
        # ordering is the caller's stream (the barrier kernel precedes every read)
        class _Arr:
            __cuda_array_interface__ = {"shape": (numel,), "typestr": "<f4" if esize == 4 else "<f8",
                                        "data": (ptr, False), "version": 2}
        flat = torch.as_tensor(_Arr(), device=self.flags_dev.device)
        per = numel // self.world
        return flat.view(self.world, *shape) if per else flat

    def barrier(self, epoch: int, stream) -> None:
        _capi.check(_capi.lib().lf_peer_barrier(self.flags_dev.data_ptr(), self.world, self.rank,
                                                epoch, stream))

    def close(self):
        L = _capi.lib()
        for r, b in enumerate(self.bases):
            if r != self.rank:
                L.lf_peer_close(b)
        L.lf_peer_free(self.local)


class ShardedCce:
    """Catalog-sharded cce_forward / cce_backward over a process group.

    exchange="collective": torch.distributed collectives (NCCL on GPUs).
    exchange="peer": peer-memory exchange (PeerExchange) with the collective
    fused into the producing kernels (bf16 / f32)."""

    def __init__(self, v_total: int, group=None, kernels=None, exchange: str = "collective"):
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.v_total = v_total
        self.v_begin, self.v_end = shard_bounds(v_total, self.P, self.rank)
        self.kernels = kernels if kernels is not None else DeviceKernels()
        if exchange not in ("collective", "peer"):
            raise ValueError(f"sharded cce: unknown exchange {exchange!r}")
        self.exchange = exchange
        self._peer = None

    def _peer_for(self, slot_bytes: int) -> PeerExchange:
        if self._peer is None or self._peer.slot_bytes < slot_bytes:
            if self._peer is not None:
                torch.cuda.synchronize()
                dist.barrier(group=self.group)
                self._peer.close()
            self._peer = PeerExchange(slot_bytes, self.group)
        return self._peer

    def _forward_peer(self, X, E_shard, targets, cfg):
        n, d = X.shape
        px = self._peer_for(max(16 * n, 4 * n * d))
        epoch, off = px.next_epoch()
        c = cfg.to_c(lf_dtype(X))
        st = _stream(X)
        _capi.check(_capi.lib().lf_cce_forward_partial_peer(
            X.data_ptr(), E_shard.data_ptr(), targets.data_ptr(), n, d, E_shard.shape[0], self.v_begin,
            C.byref(c), self._slot_table(px, off), self.P,
            self.rank, 0, st))
        px.barrier(epoch, st)
        parts = px.local_view(off, (n, 4))
        return self.kernels.combine(parts)

    def _slot_table(self, px: PeerExchange, off: int) -> int:
        # device table of this epoch's slot bases (peer bases + flag area + parity half)
        key = ("tab", off)
        tab = getattr(px, "_tabs", {})
        if key not in tab:
            tab[key] = px.slots_dev + off
            px._tabs = tab
        return tab[key].data_ptr()

    def _backward_peer(self, X, E_shard, targets, lse, upstream, cfg, stats):
        n, d = X.shape
        vs = E_shard.shape[0]
        px = self._peer_for(max(16 * n, 4 * n * d))
        epoch, off = px.next_epoch()
        dE = torch.empty((vs, d), dtype=torch.float32, device=X.device)
        c = cfg.to_c(lf_dtype(X))
        stc = _capi.CceStatsC()
        st = _stream(X)
        _capi.check(_capi.lib().lf_cce_backward_shard_peer(
            X.data_ptr(), E_shard.data_ptr(), targets.data_ptr(),
            lse.to(torch.float64).contiguous().data_ptr(), float(upstream), n, d, vs, self.v_begin,
            self.v_total, C.byref(c), dE.data_ptr(), C.byref(stc) if stats else None,
            self._slot_table(px, off), self.P, self.rank, 0, st))
        px.barrier(epoch, st)
        dX = torch.empty((n, d), dtype=torch.float32, device=X.device)
        slots = px.local_view(off, (n, d))
        _capi.check(_capi.lib().lf_peer_sum(slots.data_ptr(), self.P, n * d, dX.data_ptr(), st))
        s = ShardStats(int(stc.skipped_elems), int(stc.skipped_tiles), int(stc.total_tiles)) if stats else None
        return dX, dE, s

    @property
    def v_shard(self) -> int:
        return self.v_end - self.v_begin

    def forward(self, X, E_shard, targets, cfg: CceConfig = CceConfig()) -> LossOutput:
        if E_shard.shape[0] != self.v_shard:
            raise ValueError(f"sharded cce: rank {self.rank} expects {self.v_shard} item rows, "
                             f"got {E_shard.shape[0]}")
        if self.exchange == "peer":
            return self._forward_peer(X, E_shard, targets, cfg)
        part = self.kernels.forward_partial(X, E_shard, targets, self.v_begin, cfg)
        if self.P == 1:
            return self.kernels.combine(part.unsqueeze(0))
        n = part.shape[0]
        flat = torch.empty((self.P * n,) + tuple(part.shape[1:]), dtype=part.dtype,
                           device=part.device)
        dist.all_gather_into_tensor(flat, part.contiguous(), group=self.group)
        return self.kernels.combine(flat.view((self.P, n) + tuple(part.shape[1:])))

    def forward_backward(self, X, E_shard, targets, upstream: float = 1.0,
                         cfg: CceConfig = CceConfig(), stats: bool = False):
        """forward + backward(lse, upstream) as one step.  Where the fused
        kernel applies (bf16, d = 64 / 128 / 256, eps < 2^-12, collective exchange)
        the shard's LSE partials and dX's item sum come from one pass over its
        logits (lf_cce_fwdx_shard_begin), then the all-gather of the (m, s, t)
        triples, dX normalised by the global lse and the dE pass
        (lf_cce_fwdx_shard_end), then the dX all-reduce.  Returns
        (LossOutput, CceBackwardResult)."""
        if E_shard.shape[0] != self.v_shard:
            raise ValueError(f"sharded cce: rank {self.rank} expects {self.v_shard} item rows, "
                             f"got {E_shard.shape[0]}")
        fused = getattr(self.kernels, "fused_supported", None)
        if self.exchange == "peer" or fused is None or not fused(X, cfg):
            out = self.forward(X, E_shard, targets, cfg)
            return out, self.backward(X, E_shard, targets, out.lse, upstream, cfg, stats)
        part, work = self.kernels.fwdx_begin(X, E_shard, targets, self.v_begin, cfg)
        try:
            n = part.shape[0]
            if self.P == 1:
                parts = part.unsqueeze(0)
            else:
                flat = torch.empty((self.P * n, 4), dtype=part.dtype, device=part.device)
                dist.all_gather_into_tensor(flat, part.contiguous(), group=self.group)
                parts = flat.view(self.P, n, 4)
        except Exception:
            self.kernels.fwdx_abandon(work)
            raise
        out, dX, dE, st = self.kernels.fwdx_end(work, parts, X, E_shard, upstream, self.v_total, stats)
        if self.P > 1:
            dist.all_reduce(dX, op=dist.ReduceOp.SUM, group=self.group)
        return out, self._with_stats(CceBackwardResult(GradPair(dX, dE)), st, X.shape[0], stats)

    def _with_stats(self, res: CceBackwardResult, st, n: int, stats: bool) -> CceBackwardResult:
        if stats:
            cnt = torch.tensor([st.skipped_elems, st.skipped_tiles, st.total_tiles],
                               dtype=torch.float64, device=res.grads.d_embeddings.device)
            if self.P > 1:
                dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=self.group)
            off = n * (self.v_total - 1)
            res.skipped_fraction = float(cnt[0]) / off if off else 0.0
            res.skipped_tiles, res.total_tiles = int(cnt[1]), int(cnt[2])
        return res

    def backward(self, X, E_shard, targets, lse, upstream: float = 1.0,
                 cfg: CceConfig = CceConfig(), stats: bool = True) -> CceBackwardResult:
        if self.exchange == "peer":
            dX, dE, st = self._backward_peer(X, E_shard, targets, lse, upstream, cfg, stats)
        else:
            dX, dE, st = self.kernels.backward_shard(X, E_shard, targets, lse, upstream, self.v_begin,
                                                     self.v_total, cfg, stats)
            if self.P > 1:
                dist.all_reduce(dX, op=dist.ReduceOp.SUM, group=self.group)
        return self._with_stats(CceBackwardResult(GradPair(dX, dE)), st, X.shape[0], stats)
