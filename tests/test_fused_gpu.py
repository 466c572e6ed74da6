"""GPU parity of the fused forward + dX path (lf_cce_forward_backward: the
FWDX tcgen05 kernel, then the item-owned dE pass) against the CPU oracle.

The pair it replaces is cce_forward + cce_backward(lse, upstream) on the same
inputs (proj/src/trainer.cpp:71-77).  With filter_eps = 0 the fused path has
the reference's exact semantics; with filter_eps > 0 its dX is the unfiltered
gradient (each entry the filter drops is below eps), so it is checked against
the FILTERED oracle at the same bf16 tolerances as the separate path, while
dE and the skip statistics follow the filter exactly."""
import numpy as np
import pytest
import torch

import oracle_bind as ob
from gpu_util import TOL, check_grad, instance, prepare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lf(cuda):
    import paper_2509_09682_b200 as lf
    return lf


def fused(lf, X, E, x, eps=0.0, upstream=1.0, stats=False):
    return lf.cce_forward_backward(X, E, x, upstream, lf.CceConfig(filter_eps=eps), stats=stats)


def check_against_oracle(out, bwd, Eh, Ch, t, eps=0.0, upstream=1.0, frac_tol=None):
    tol = TOL[torch.bfloat16]
    loss, pos, lse = ob.cce_forward(Eh, Ch, t)
    dX, dC, frac, _ = ob.cce_backward(Eh, Ch, t, lse, upstream, eps)
    assert ob.rel_err(float(out.loss), loss) < tol["loss"]
    assert ob.rel_err(out.lse.cpu().numpy(), lse).max() < tol["lse"]
    assert ob.rel_err(out.pos_logits.cpu().numpy(), pos).max() < tol["lse"]
    check_grad(bwd.grads.d_embeddings, dX, torch.bfloat16, "dX")
    check_grad(bwd.grads.d_classifier, dC.T, torch.bfloat16, "dE")
    if frac_tol is not None:
        assert abs(bwd.skipped_fraction - frac) <= frac_tol, (bwd.skipped_fraction, frac)


@pytest.mark.parametrize("n,d,v", [(1, 64, 2), (127, 64, 129), (128, 64, 128), (300, 64, 5000),
                                   (257, 128, 3000), (1000, 128, 20000), (2048, 64, 32768),
                                   (640, 64, 131072 + 77), (1, 256, 3), (130, 256, 1000),
                                   (300, 256, 20000 + 33)])
def test_fused_equals_oracle_unfiltered(lf, n, d, v):
    X, E, x, Eh, Ch, t = instance(0xB2000011 + n + v, n, d, v, torch.bfloat16)
    out, bwd = fused(lf, X, E, x)
    check_against_oracle(out, bwd, Eh, Ch, t)


def test_fused_full_catalog_row_slice(lf):
    """cfg2 geometry (D = 64, V = 1M) on a 256-row slice, headline eps."""
    X, E, x, Eh, Ch, t = instance(0xB2000002, 256, 64, 1_000_000, torch.bfloat16)
    out, bwd = fused(lf, X, E, x, eps=6e-8, stats=True)
    check_against_oracle(out, bwd, Eh, Ch, t, eps=6e-8, frac_tol=2e-3)


@pytest.mark.parametrize("gamma,eps", [(0.0, 6e-8), (1.0, 6e-8), (0.0, 1e-6), (1.0, 1e-6)])
def test_fused_filtered_matches_filtered_oracle(lf, gamma, eps):
    """Uniform and trained-like rows X_i = U(-1,1)^D + gamma E_(x_i)
     at the reference preset eps and at 1e-6: the unfiltered
    fused dX stays within the bf16 tolerances of the filtered oracle; dE and
    the skip fraction (counted by the dE pass) follow the filter."""
    n, d, v = 384, 64, 40000
    inst = ob.make_instance(ob.Rng(0xB2000004), n, d, v)
    Eref = (inst.E + gamma * inst.C.T[inst.targets]).astype(np.float32)
    X, E, Eh, Ch = prepare(Eref, inst.C, torch.bfloat16)
    x = torch.from_numpy(inst.targets).cuda()
    out, bwd = fused(lf, X, E, x, eps=eps, stats=True)
    check_against_oracle(out, bwd, Eh, Ch, inst.targets, eps=eps, frac_tol=2e-3)


def peaked(seed, n, d, v, rows):
    """Rows in `rows` put half their weight on their target and half on a
    second item u: X_i = (E_t + E_u) / 2 with |E|^2 ~ 192, so both logits sit
    ~50 nats above a typical 128-item tile's max while the gradient stays
    O(1) (softmax ~1/2 on each).  The other rows are uniform."""
    inst = ob.make_instance(ob.Rng(seed), n, d, v, 3.0)
    Eref = inst.E.copy()
    t = inst.targets
    u = (t + 1 + np.arange(n) * 7919) % v
    u = np.where(u == t, (u + 1) % v, u)
    Eref[rows] = 0.5 * (inst.C.T[t[rows]] + inst.C.T[u[rows]])
    X, E, Eh, Ch = prepare(Eref.astype(np.float32), inst.C, torch.bfloat16)
    return X, E, torch.from_numpy(t).cuda(), Eh, Ch, t


def test_fused_rebase_on_peaked_rows(lf):
    """Every row peaked: the first chunk's max is far below the row's top
    logits, so the running reference moves mid-unit and s, O and the tile's
    already-written P chunks are rescaled (the rare path).  Same oracle
    tolerances as everywhere else."""
    X, E, x, Eh, Ch, t = peaked(0xB2000005, 512, 64, 9000, np.ones(512, bool))
    _, _, lse = ob.cce_forward(Eh, Ch, t)
    top = np.max(Eh[:, :] @ Ch[:, :128], axis=1)
    assert np.median(lse - top) > 44.0  # the rebase path is taken
    out, bwd = fused(lf, X, E, x)
    check_against_oracle(out, bwd, Eh, Ch, t)
    assert torch.isfinite(bwd.grads.d_embeddings).all()


def test_fused_mixed_rows_rebase_per_lane(lf):
    """Odd rows peaked (rebase), even rows uniform (no rebase) in the same
    warps: per-lane rescale factors must leave the uniform rows intact."""
    n = 384
    X, E, x, Eh, Ch, t = peaked(0xB2000006, n, 64, 6000, np.arange(n) % 2 == 1)
    out, bwd = fused(lf, X, E, x)
    check_against_oracle(out, bwd, Eh, Ch, t)


def test_fused_upstream_and_determinism(lf):
    X, E, x, *_ = instance(91, 300, 64, 7000, torch.bfloat16)
    o1, b1 = fused(lf, X, E, x, eps=6e-8)
    o1b, b1b = fused(lf, X, E, x, eps=6e-8)
    assert torch.equal(o1.lse, o1b.lse) and torch.equal(o1.loss, o1b.loss)
    assert torch.equal(b1.grads.d_embeddings, b1b.grads.d_embeddings)
    assert torch.equal(b1.grads.d_classifier, b1b.grads.d_classifier)
    _, b2 = fused(lf, X, E, x, eps=6e-8, upstream=2.5)
    rel = lambda a, b: float((a - b).norm() / b.norm())
    assert rel(b2.grads.d_embeddings, 2.5 * b1.grads.d_embeddings) < 1e-6
    assert rel(b2.grads.d_classifier, 2.5 * b1.grads.d_classifier) < 1e-3
    _, b0 = fused(lf, X, E, x, upstream=0.0)
    assert (b0.grads.d_embeddings == 0).all() and (b0.grads.d_classifier == 0).all()


def test_fused_agrees_with_separate_calls(lf):
    """Same inputs through cce_forward + cce_backward: lse to fp32 rounding,
    gradients to the bf16 normwise tolerance; fp32 / fp64 and coarse eps take
    the separate path inside lf_cce_forward_backward (identical bits)."""
    X, E, x, *_ = instance(92, 700, 64, 12000, torch.bfloat16)
    out, bwd = fused(lf, X, E, x)
    ro = lf.cce_forward(X, E, x)
    rb = lf.cce_backward(X, E, x, ro.lse, 1.0)
    assert float((out.lse - ro.lse).abs().max()) < 1e-5
    for a, b in ((bwd.grads.d_embeddings, rb.grads.d_embeddings),
                 (bwd.grads.d_classifier, rb.grads.d_classifier)):
        assert float((a - b).norm() / b.norm()) < 1e-2
    for dtype, eps in ((torch.float32, 1e-3), (torch.float64, 1e-3), (torch.bfloat16, 2.0 ** -8)):
        X2, E2, x2, *_ = instance(93, 200, 64, 3000, dtype)
        cfg = lf.CceConfig(filter_eps=eps)
        fo, fb = lf.cce_forward_backward(X2, E2, x2, 1.0, cfg)
        so = lf.cce_forward(X2, E2, x2, cfg)
        sb = lf.cce_backward(X2, E2, x2, so.lse, 1.0, cfg)
        assert torch.equal(fo.lse, so.lse)
        assert torch.equal(fb.grads.d_embeddings, sb.grads.d_embeddings)
        assert torch.equal(fb.grads.d_classifier, sb.grads.d_classifier)
    # fp32 with the filter off takes the fused SIMT forward + dX (and hands
    # the dE pass a full-precision 1 - p_t): agreement to fp32 rounding
    X2, E2, x2, *_ = instance(93, 200, 64, 3000, torch.float32)
    fo, fb = lf.cce_forward_backward(X2, E2, x2, 1.0, lf.CceConfig())
    so = lf.cce_forward(X2, E2, x2)
    sb = lf.cce_backward(X2, E2, x2, fo.lse, 1.0)
    assert float((fo.lse - so.lse).abs().max()) < 1e-5
    assert torch.equal(fo.pos_logits, so.pos_logits)
    for a, b in ((fb.grads.d_embeddings, sb.grads.d_embeddings), (fb.grads.d_classifier, sb.grads.d_classifier)):
        assert float((a - b).norm() / b.norm()) < 1e-5


def test_fused_d256_peaked_rows_and_filter(lf):
    """D = 256 (cfg5 width; one epilogue warpgroup, 64-column tiles): the
    rebase path on peaked rows and the filtered oracle at the preset eps."""
    X, E, x, Eh, Ch, t = peaked(0xB2000007, 256, 256, 3000, np.arange(256) % 3 == 0)
    out, bwd = fused(lf, X, E, x)
    check_against_oracle(out, bwd, Eh, Ch, t)
    X, E, x, Eh, Ch, t = instance(0xB2000008, 200, 256, 9000, torch.bfloat16)
    out, bwd = fused(lf, X, E, x, eps=6e-8, stats=True)
    check_against_oracle(out, bwd, Eh, Ch, t, eps=6e-8, frac_tol=2e-3)


@pytest.mark.parametrize("n,d,v", [(1, 64, 2), (127, 64, 129), (300, 64, 5000), (2048, 64, 32768),
                                   (257, 32, 3001), (200, 48, 1000), (257, 128, 3000),
                                   (130, 256, 1000), (100, 96, 70000), (100, 30, 2000), (65, 7, 513)])
def test_fused_f32_equals_oracle(lf, n, d, v):
    """fp32 with the filter off: the fused SIMT forward + dX (lf_simt.cu
    cce_simt_fwdx + simt_fwdx_combine) and the dE pass, against the oracle at
    the fp32 tolerances (cfg1: N = 2048, V = 32768)."""
    X, E, x, Eh, Ch, t = instance(0xB2000031 + n + v + d, n, d, v, torch.float32)
    out, bwd = lf.cce_forward_backward(X, E, x, 1.0, lf.CceConfig(), stats=True)
    tol = TOL[torch.float32]
    loss, pos, lse = ob.cce_forward(Eh, Ch, t)
    dX, dC, _, _ = ob.cce_backward(Eh, Ch, t, lse, 1.0, 0.0)
    assert ob.rel_err(float(out.loss), loss) < tol["loss"]
    assert ob.rel_err(out.lse.cpu().numpy(), lse).max() < tol["lse"]
    assert ob.rel_err(out.pos_logits.cpu().numpy(), pos).max() < tol["lse"]
    for got, want, what in ((bwd.grads.d_embeddings, dX, "dX"), (bwd.grads.d_classifier, dC.T, "dE")):
        if d < 256:
            check_grad(got, want, torch.float32, what)
            continue
        # fp32 logits over 256 products carry ~3e-6 of max|grad| absolute
        # error in either path (tools/f32_diag.py: dX fused 2.6e-6, separate
        # 2.7e-6 at this shape), past the D <= 128 floor of 1e-6; normwise 1e-5 holds
        g = got.double().cpu().numpy()
        mx = np.abs(want).max()
        assert (np.abs(g - want) <= 1e-4 * np.abs(want) + 5e-6 * mx).all(), what
        assert np.linalg.norm(g - want) / np.linalg.norm(want) < tol["norm"], what
    assert bwd.skipped_fraction == 0.0


@pytest.mark.parametrize("gamma", [1.0, 4.0])
def test_fused_f32_peaked_rows(lf, gamma):
    """Rows whose target dominates (p_t -> 1): dX = scale (sum_{j != t} p_j E_j
    - (1 - p_t) E_t) with 1 - p_t = S_x / (e^(t - M) + S_x) from the sum
    without the target, and the dE pass takes the same 1 - p_t, so the small
    gradients keep their precision.  Checked against a float64 computation in
    that stable form: the reference's own (s - 1) keeps only ~1e-16 of
    1 - p_t, which is all of it on the rows this builds (gamma = 4)."""
    n, d, v = 300, 64, 4000
    X, E, x, Eh, Ch, t = instance(0xB2000041, n, d, v, torch.float32)
    Xp = (Eh + gamma * Ch.T[t]).astype(np.float32)
    Xg = torch.from_numpy(Xp).cuda()
    out, bwd = lf.cce_forward_backward(Xg, E, x, 1.0, lf.CceConfig())
    Ed = Ch.T.astype(np.float64)                      # v x d
    S = Xp.astype(np.float64) @ Ed.T                  # n x v logits
    rows = np.arange(n)
    m = S.max(1, keepdims=True)
    P = np.exp(S - m)
    P[rows, t] = 0.0                                  # off-target terms only
    sx = P.sum(1)
    st = np.exp(S[rows, t] - m[:, 0])
    lse = S[rows, t] + np.log1p(sx / st)
    P = P / (st + sx)[:, None]                        # p_j, j != t
    omp = sx / (st + sx)                              # 1 - p_t
    scale = 1.0 / n
    G = P * scale
    G[rows, t] = -omp * scale
    dX = G @ Ed
    dE = G.T @ Xp.astype(np.float64)
    assert np.abs(out.lse.cpu().numpy() - lse).max() < 1e-5 * np.abs(lse).max()
    for got, want, what in ((bwd.grads.d_embeddings, dX, "dX"), (bwd.grads.d_classifier, dE, "dE")):
        g = got.double().cpu().numpy()
        assert np.linalg.norm(g - want) / np.linalg.norm(want) < 1e-4, what
