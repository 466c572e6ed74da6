"""CPU, world_size 2 (gloo): the catalog-sharding host logic of
paper_2509_09682_b200/sharded.py — shard bounds, the all-gather of per-row
(m, s, t) partials, the combine, the dX all-reduce and the cross-rank skip
count — with the per-shard kernels replaced by the CPU oracle (test-only
backend).  The device kernels behind the same interface are covered by
tests/test_sharded_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_bind as ob

LOG2E = 1.4426950408889634


class OracleKernels:
    """Test backend: per-shard partials / gradients from oracle/oracle.c.
    Tensors are CPU tensors in the B200 layout (X n x d, E v x d)."""

    def __init__(self, Eh, Ch_full, t):
        self.Eh, self.Ch, self.t = Eh, Ch_full, t

    def forward_partial(self, X, E_shard, targets, v_offset, cfg):
        v1 = v_offset + E_shard.shape[0]
        m, s, tt, h = ob.cce_forward_partial(self.Eh, self.Ch, self.t, v_offset, v1)
        return torch.from_numpy(np.stack([m * LOG2E, s, tt, h.astype(np.float64)], 1)).float()

    def combine(self, parts):
        from paper_2509_09682_b200.losses import LossOutput
        p = parts.double().numpy()
        M = p[:, :, 0].max(0)
        S = (p[:, :, 1] * np.exp2(p[:, :, 0] - M)).sum(0)
        lse = (M + np.log2(S)) / LOG2E
        pos = (p[:, :, 2] * p[:, :, 3]).sum(0)
        return LossOutput(torch.tensor(float(np.mean(lse - pos)), dtype=torch.float64),
                          torch.from_numpy(pos), torch.from_numpy(lse))

    def backward_shard(self, X, E_shard, targets, lse, upstream, v_offset, v_total, cfg, stats):
        from paper_2509_09682_b200.sharded import ShardStats
        v1 = v_offset + E_shard.shape[0]
        Cs = np.ascontiguousarray(self.Ch[:, v_offset:v1])
        local_t = np.where((self.t >= v_offset) & (self.t < v1), self.t - v_offset, -1)
        dE, dC, _, sk = ob.cce_backward(self.Eh, Cs, local_t.astype(np.int64), lse.numpy(),
                                        upstream, cfg.filter_eps)
        return (torch.from_numpy(dE), torch.from_numpy(np.ascontiguousarray(dC.T)),
                ShardStats(int(sk), 0, 0))


class FusedOracleKernels(OracleKernels):
    """Test backend for ShardedCce.forward_backward's fused phases
    (lf_cce_fwdx_shard_begin / _end): begin = the shard's folded (m, s, t)
    partial, end = combine + the shard's dX partial and dE rows."""

    def fused_supported(self, X, cfg):
        return True

    def fwdx_begin(self, X, E_shard, targets, v_offset, cfg):
        return self.forward_partial(X, E_shard, targets, v_offset, cfg), (v_offset, E_shard, cfg)

    def fwdx_end(self, work, parts, X, E_shard, upstream, v_total, stats):
        v_offset, E_shard, cfg = work
        out = self.combine(parts)
        dX, dE, st = self.backward_shard(X, E_shard, None, out.lse, upstream, v_offset, v_total, cfg,
                                         stats)
        return out, dX, dE, st

    def fwdx_abandon(self, work):
        pass


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, seed, n, d, v, eps, q, fused=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_09682_b200 import CceConfig
        from paper_2509_09682_b200.sharded import ShardedCce, shard_bounds
        rng = ob.Rng(seed)
        inst = ob.make_instance(rng, n, d, v)
        K = FusedOracleKernels if fused else OracleKernels
        sh = ShardedCce(v, kernels=K(inst.E, inst.C, inst.targets))
        assert (sh.v_begin, sh.v_end) == shard_bounds(v, world, rank)
        X = torch.from_numpy(inst.E)
        E_shard = torch.from_numpy(np.ascontiguousarray(inst.C.T[sh.v_begin:sh.v_end]))
        x = torch.from_numpy(inst.targets)
        cfg = CceConfig(filter_eps=eps)
        if fused:
            out, res = sh.forward_backward(X, E_shard, x, 1.0, cfg, stats=True)
        else:
            out = sh.forward(X, E_shard, x, cfg)
            res = sh.backward(X, E_shard, x, out.lse, 1.0, cfg)
        q.put((rank, sh.v_begin, sh.v_end, float(out.loss), out.lse.numpy(),
               out.pos_logits.numpy(), res.grads.d_embeddings.numpy(),
               res.grads.d_classifier.numpy(), res.skipped_fraction))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("eps,fused", [(0.0, False), (1e-3, False), (0.0, True), (1e-3, True)])
def test_two_rank_catalog_sharding_matches_unsharded(eps, fused):
    world, seed, n, d, v = 2, 4242, 23, 7, 101
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, n, d, v, eps, q, fused))
             for r in range(world)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = ob.Rng(seed)
    inst = ob.make_instance(rng, n, d, v)
    loss, pos, lse = ob.cce_forward(inst.E, inst.C, inst.targets)
    dE_rows = np.zeros((v, d))
    for rank, b, e, l, lse_r, pos_r, dx_r, de_r, frac_r in results:
        # the backward consumes the combined lse; compare with the oracle on it
        dE, dC, frac, _ = ob.cce_backward(inst.E, inst.C, inst.targets, lse_r, 1.0, eps)
        # partial triples travel as float32 (the C-ABI's float4 exchange format)
        assert abs(l - loss) < 1e-6 * max(1.0, abs(loss))
        assert ob.rel_err(lse_r, lse).max() < 1e-6
        assert ob.rel_err(pos_r, pos).max() < 1e-6
        assert np.abs(dx_r - dE).max() < 1e-12  # all-reduced partial dX
        assert frac_r == frac                   # skip count summed across ranks
        dE_rows[b:e] = de_r
    assert np.array_equal(dE_rows, dC.T)        # item-owned: bitwise per column


def test_shard_bounds_cover_catalog():
    from paper_2509_09682_b200.sharded import shard_bounds
    for v in (1, 7, 1000, 1_000_003):
        for P in (1, 2, 3, 8):
            b = [shard_bounds(v, P, p) for p in range(P)]
            assert b[0][0] == 0 and b[-1][1] == v
            assert all(b[i][1] == b[i + 1][0] for i in range(P - 1))
            assert max(e - s for s, e in b) - min(e - s for s, e in b) <= 1


class OracleEvalKernels:
    """Test backend for ShardedEval: per-shard ranking from oracle/oracle.c on
    the full instance (H n x d double, C d x v float); checks that the
    exchanged target rows are the targets' item rows."""

    def __init__(self, H, Cm, t):
        self.H, self.Cm, self.t = H, Cm, t

    def rank_topk(self, X, E_shard, targets, k, v_offset, target_rows):
        want = np.ascontiguousarray(self.Cm.T[self.t]).astype(np.float64)
        assert np.array_equal(target_rows.numpy(), want)
        a, top, sc = ob.eval_rank_topk(self.H, self.Cm, self.t, k, v_offset,
                                       v_offset + E_shard.shape[0])
        return torch.from_numpy(a), torch.from_numpy(top), torch.from_numpy(sc)

    def merge(self, ahead, top_idx, top_score):
        P, n, k = top_idx.shape
        rank = ahead.sum(0) + 1
        top = np.empty((n, k), np.int64)
        sc = np.empty((n, k))
        for i in range(n):
            cand = sorted((-float(top_score[p, i, e]), int(top_idx[p, i, e]))
                          for p in range(P) for e in range(k) if top_idx[p, i, e] >= 0)[:k]
            top[i] = [c[1] for c in cand]
            sc[i] = [-c[0] for c in cand]
        return rank, torch.from_numpy(top), torch.from_numpy(sc)

    def summarize(self, rank, top_idx, popularity):
        from paper_2509_09682_b200.metrics import EvalSummary
        return EvalSummary(*ob.eval_summary(rank.numpy(), top_idx.numpy(), popularity.numpy()))


def _eval_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_09682_b200.sharded import ShardedEval
        g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "eval_ref.npz"))
        H, Cm, t, counts, k = g["0_H"], g["0_C"], g["0_t"], g["0_counts"], int(g["0_k"])
        se = ShardedEval(Cm.shape[1], kernels=OracleEvalKernels(H, Cm, t))
        E_shard = torch.from_numpy(np.ascontiguousarray(Cm.T[se.v_begin:se.v_end]).astype(np.float64))
        s = se.evaluate(torch.from_numpy(H), E_shard, torch.from_numpy(t), k, torch.from_numpy(counts))
        r, top, _ = se.rank_topk(torch.from_numpy(H), E_shard, torch.from_numpy(t), k)
        q.put((rank, (s.ndcg, s.coverage, s.surprisal), r.numpy(), top.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_evaluate_matches_reference():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_eval_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "eval_ref.npz"))
    _, top_full, _ = ob.eval_rank_topk(g["0_H"], g["0_C"], g["0_t"], int(g["0_k"]))
    for _, out3, r, top in results:
        assert out3 == tuple(g["0_out3"])            # the reference's evaluate(), bitwise
        assert np.array_equal(r, g["0_ranks"])
        assert np.array_equal(top, top_full)
