"""GPU parity of the CCE path (cce_forward / cce_backward) against the CPU
oracle and the reference's golden fixtures.  Cases follow
proj/tests/test_cce.cpp and acceptance.cpp criteria 1 and 3."""
import math
import os

import numpy as np
import pytest
import torch

import oracle_bind as ob
from gpu_util import TOL, check_grad, instance, prepare

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def lf(cuda):
    import paper_2509_09682_b200 as lf
    return lf


def run(lf, X, E, x, eps=0.0, upstream=1.0):
    cfg = lf.CceConfig(filter_eps=eps)
    out = lf.cce_forward(X, E, x, cfg)
    bwd = lf.cce_backward(X, E, x, out.lse, upstream, cfg)
    return out, bwd


def compare(out, bwd, Eh, Ch, t, dtype, eps=0.0, frac_tol=0.0):
    tol = TOL[dtype]
    loss, pos, lse = ob.cce_forward(Eh, Ch, t)
    dE, dC, frac, _ = ob.cce_backward(Eh, Ch, t, lse, 1.0, eps)
    assert ob.rel_err(float(out.loss), loss) < tol["loss"]
    assert ob.rel_err(out.lse.cpu().numpy(), lse).max() < tol["lse"]
    if dtype == torch.float64:  # same operand order: bitwise (test_cce.cpp:41)
        assert np.array_equal(out.pos_logits.cpu().numpy(), pos)
    else:
        assert ob.rel_err(out.pos_logits.cpu().numpy(), pos).max() < tol["lse"]
    check_grad(bwd.grads.d_embeddings, dE, dtype, "dX")
    check_grad(bwd.grads.d_classifier, dC.T, dtype, "dE")
    assert abs(bwd.skipped_fraction - frac) <= frac_tol, (bwd.skipped_fraction, frac)


def test_exact_mode_equals_oracle_on_random_instances(lf):
    """test_cce.cpp:55-68 (fewer trials): fp64 exact mode, pos bitwise."""
    rng = ob.Rng(1001)
    for _ in range(40):
        n, d, v = 1 + rng.bounded(32), 1 + rng.bounded(16), 2 + rng.bounded(127)
        inst = ob.make_instance(rng, n, d, v)
        X, E, Eh, Ch = prepare(inst.E, inst.C, torch.float64)
        x = torch.from_numpy(inst.targets).cuda()
        out, bwd = run(lf, X, E, x)
        compare(out, bwd, Eh, Ch, inst.targets, torch.float64)
        assert bwd.skipped_fraction == 0.0


def test_golden_fixtures_all_dtypes(lf):
    g = np.load(os.path.join(GOLDEN, "cce_ref.npz"))
    for k in range(int(g["count"])):
        Eh, Ch, t = g[f"{k}_E"], g[f"{k}_C"], g[f"{k}_t"]
        d = Eh.shape[1]
        for dtype in (torch.float64, torch.float32, torch.bfloat16):
            if dtype == torch.bfloat16 and d % 64:
                continue
            X, E, Eh2, Ch2 = prepare(Eh, Ch, dtype)
            x = torch.from_numpy(t).cuda()
            out, bwd = run(lf, X, E, x)
            if dtype == torch.float64:
                assert float(out.loss) == pytest.approx(float(g[f"{k}_loss"]), rel=1e-12)
                assert np.array_equal(out.pos_logits.cpu().numpy(), g[f"{k}_pos"])
                check_grad(bwd.grads.d_embeddings, g[f"{k}_dE"], dtype)
                check_grad(bwd.grads.d_classifier, g[f"{k}_dC"].T, dtype)
                out, bwd = run(lf, X, E, x, eps=1e-3)
                assert bwd.skipped_fraction == float(g[f"{k}_frac_eps"])
                check_grad(bwd.grads.d_embeddings, g[f"{k}_dE_eps"], dtype)
                check_grad(bwd.grads.d_classifier, g[f"{k}_dC_eps"].T, dtype)
            else:
                compare(out, bwd, Eh2, Ch2, t, dtype)


@pytest.mark.parametrize("n,d,v", [(1, 64, 2), (127, 64, 129), (128, 64, 128), (300, 64, 5000),
                                   (257, 128, 3000), (200, 192, 700), (130, 256, 1000),
                                   (2048, 64, 32768)])
def test_bf16_tensor_core_path(lf, n, d, v):
    X, E, x, Eh, Ch, t = instance(0xB2000001 + n + v, n, d, v, torch.bfloat16)
    out, bwd = run(lf, X, E, x)
    compare(out, bwd, Eh, Ch, t, torch.bfloat16)


def test_fp32_cfg1_shape(lf):
    """BASELINE cfg1: fp32, N=2048, D=64, V=32768, filtering off; loss 1e-5."""
    X, E, x, Eh, Ch, t = instance(0xB2000001, 2048, 64, 32768, torch.float32)
    out, bwd = run(lf, X, E, x)
    compare(out, bwd, Eh, Ch, t, torch.float32)


def test_bf16_full_catalog_row_slice(lf):
    """cfg2 geometry (D=64, V=1M) on a 256-row slice: every item tile and the
    V-split combine are exercised at full catalog width."""
    X, E, x, Eh, Ch, t = instance(0xB2000002, 256, 64, 1_000_000, torch.bfloat16)
    out, bwd = run(lf, X, E, x)
    compare(out, bwd, Eh, Ch, t, torch.bfloat16)


def test_log2_known_answer(lf):  # test_cce.cpp:82-88
    for dtype in (torch.float64, torch.float32):
        X = torch.tensor([[0.5]], dtype=dtype, device="cuda")
        E = torch.tensor([[0.25], [0.25]], dtype=dtype, device="cuda")
        x = torch.tensor([1], device="cuda")
        out = lf.cce_forward(X, E, x)
        assert float(out.loss) == pytest.approx(math.log(2.0), rel=1e-12 if dtype == torch.float64 else 1e-6)
    X = torch.full((1, 64), 0.0, dtype=torch.bfloat16, device="cuda")
    E = torch.zeros((2, 64), dtype=torch.bfloat16, device="cuda")
    out = lf.cce_forward(X, E, torch.tensor([1], device="cuda"))
    assert float(out.loss) == pytest.approx(math.log(2.0), rel=1e-6)


def test_filter_everything_keeps_only_target_terms(lf):  # test_cce.cpp:90-118
    for dtype in (torch.float64, torch.bfloat16):
        d = 4 if dtype == torch.float64 else 64
        X, E, x, Eh, Ch, t = instance(7, 6, d, 15, dtype)
        out, bwd = run(lf, X, E, x, eps=1.0)
        assert bwd.skipped_fraction == 1.0
        _, pos, lse = ob.cce_forward(Eh, Ch, t)
        coeff = (np.exp(pos - lse) - 1.0) / 6
        want = coeff[:, None] * Ch[:, t].T
        check_grad(bwd.grads.d_embeddings, want, dtype)
        dE = bwd.grads.d_classifier.double().cpu().numpy()
        untouched = np.setdiff1d(np.arange(15), t)
        assert (dE[untouched] == 0.0).all()


def test_margin40_filtering_skips_nearly_everything_and_stays_exact(lf):
    """test_cce.cpp:120-154 (eps = 2^-23 on one-hot geometry)."""
    rng = ob.Rng(900)
    eps = 2.0 ** -23
    for _ in range(5):
        n, v = 2 + rng.bounded(10), 8 + rng.bounded(24)
        d = v
        Eh = np.zeros((n, d), np.float32)
        Ch = np.zeros((d, v), np.float32)
        t = np.array([rng.bounded(v) for _ in range(n)], np.int64)
        for j in range(v):
            Ch[j, j] = 40.0
        Eh[np.arange(n), t] = 1.0
        X, E, _, _ = prepare(Eh, Ch, torch.float64)
        x = torch.from_numpy(t).cuda()
        cfg_f = lf.CceConfig(filter_eps=eps)
        out = lf.cce_forward(X, E, x, cfg_f)
        filt = lf.cce_backward(X, E, x, out.lse, 1.0, cfg_f)
        exact = lf.cce_backward(X, E, x, out.lse, 1.0, lf.CceConfig())
        assert filt.skipped_fraction > 0.9
        for a, b in ((filt.grads.d_embeddings, exact.grads.d_embeddings),
                     (filt.grads.d_classifier, exact.grads.d_classifier)):
            assert ob.rel_err(a.cpu().numpy(), b.cpu().numpy()).max() < 1e-6


def test_skip_fraction_monotone_and_matches_oracle(lf):  # test_cce.cpp:156-168
    for dtype, d in ((torch.float64, 5), (torch.bfloat16, 64)):
        X, E, x, Eh, Ch, t = instance(133, 12, d, 40, dtype)
        out = lf.cce_forward(X, E, x)
        _, _, lse = ob.cce_forward(Eh, Ch, t)
        prev = -1.0
        for eps in (0.0, 1e-8, 1e-6, 1e-4, 1e-2, 1.0):
            res = lf.cce_backward(X, E, x, out.lse, 1.0, lf.CceConfig(filter_eps=eps))
            assert res.skipped_fraction >= prev
            prev = res.skipped_fraction
            _, _, frac, _ = ob.cce_backward(Eh, Ch, t, lse, 1.0, eps)
            if dtype == torch.float64:
                assert res.skipped_fraction == frac
            else:  # fp32 decision near the threshold may flip a handful of elements
                assert abs(res.skipped_fraction - frac) <= 0.01
        assert prev == 1.0


def test_bf16_filtering_matches_oracle_on_random_data(lf):
    X, E, x, Eh, Ch, t = instance(0xB2000002, 1000, 64, 20000, torch.bfloat16)
    out, bwd = run(lf, X, E, x, eps=1e-6)
    compare(out, bwd, Eh, Ch, t, torch.bfloat16, eps=1e-6, frac_tol=2e-3)


def test_results_are_bitwise_deterministic(lf):  # test_cce.cpp:170-196
    for dtype, d in ((torch.float64, 8), (torch.float32, 64), (torch.bfloat16, 64)):
        X, E, x, *_ = instance(271, 370, d, 5300, dtype)
        ref_out, ref_bwd = run(lf, X, E, x)
        for rb, cb, w in ((16, 32, 2), (3, 5, 8)):
            cfg = lf.CceConfig(row_block=rb, col_block=cb, workers=w)
            out = lf.cce_forward(X, E, x, cfg)
            bwd = lf.cce_backward(X, E, x, out.lse, 1.0, cfg)
            assert torch.equal(out.lse, ref_out.lse) and torch.equal(out.loss, ref_out.loss)
            assert torch.equal(out.pos_logits, ref_out.pos_logits)
            assert torch.equal(bwd.grads.d_embeddings, ref_bwd.grads.d_embeddings)
            assert torch.equal(bwd.grads.d_classifier, ref_bwd.grads.d_classifier)


def test_backward_linear_in_upstream(lf):  # test_oracles.cpp:71-87
    X, E, x, *_ = instance(77, 130, 64, 700, torch.bfloat16)
    out = lf.cce_forward(X, E, x)
    g1 = lf.cce_backward(X, E, x, out.lse, 1.0).grads
    g2 = lf.cce_backward(X, E, x, out.lse, 2.0).grads
    gn = lf.cce_backward(X, E, x, out.lse, -0.5).grads
    g0 = lf.cce_backward(X, E, x, out.lse, 0.0).grads
    rel = lambda a, b: float((a - b).norm() / b.norm())
    # bf16: scaling moves the exp argument by log2|upstream|, so G rounds
    # differently; linearity holds to the bf16 normwise tolerance (1e-2).
    assert rel(g2.d_embeddings, 2 * g1.d_embeddings) < 1e-3
    assert rel(g2.d_classifier, 2 * g1.d_classifier) < 1e-3
    assert rel(gn.d_classifier, -0.5 * g1.d_classifier) < 1e-3
    assert (g0.d_embeddings == 0).all() and (g0.d_classifier == 0).all()


def test_retained_memory_is_two_scalars_per_row(lf):  # test_cce.cpp:198-215
    X, E, x, *_ = instance(64, 8, 64, 16, torch.bfloat16)
    acct = lf.MemAccountant()
    out = lf.cce_forward(X, E, x, lf.CceConfig(), acct)
    acct.expect_scratch_released()
    rep = acct.report()
    assert rep.current.retained_real == 16 and rep.current.scratch_real == 0
    assert rep.peak.scratch_real > 0
    lf.cce_backward(X, E, x, out.lse, 1.0, lf.CceConfig(), acct)
    acct.expect_scratch_released()
    assert acct.report().current.retained_real == 16


def test_invalid_inputs_name_the_row(lf):  # test_oracles.cpp:215-231, test_cce.cpp:217-224
    X, E, x, *_ = instance(3, 4, 64, 8, torch.bfloat16)
    bad = x.clone()
    bad[1] = 8
    with pytest.raises(ValueError, match="row 1 targets item 8, outside catalog of 8"):
        lf.cce_forward(X, E, bad)
    with pytest.raises(ValueError, match="LSE vector has 3 entries for 4 rows"):
        lf.cce_backward(X, E, x, torch.zeros(3, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("gamma", [0.0, 1.0, 2.0])
def test_bf16_filtered_backward_matches_filtered_oracle(lf, gamma):
    """The headline configuration's filter (eps = kFp16MinPositive = 6e-8,
    cce.hpp:26-30) on uniform (gamma = 0) and "trained-like" rows
    X_i = U(-1,1)^D + gamma E_{x_i}.  gamma 0 and 1: the bf16
    gradients match the oracle's FILTERED gradients at the bf16 tolerances.
    gamma 2 is nearly converged (loss ~4e-4): every row's gradient is the
    small difference (softmax_t - 1) E_t + sum_j softmax_j E_j, where fp32
    logits (not the reference's double) leave ~1e-5 relative error in
    softmax_t, i.e. percent-level error in the difference — so there only the
    loss, the skip count and a 10 % normwise bound are checked."""
    n, d, v = 384, 64, 40000
    inst = ob.make_instance(ob.Rng(0xB2000002), n, d, v)
    Eref = (inst.E + gamma * inst.C.T[inst.targets]).astype(np.float32)
    X, E, Eh, Ch = prepare(Eref, inst.C, torch.bfloat16)
    x = torch.from_numpy(inst.targets).cuda()
    out, bwd = run(lf, X, E, x, eps=6e-8)
    if gamma < 2.0:
        compare(out, bwd, Eh, Ch, inst.targets, torch.bfloat16, eps=6e-8, frac_tol=2e-3)
        return
    loss, pos, lse = ob.cce_forward(Eh, Ch, inst.targets)
    dX, dC, frac, _ = ob.cce_backward(Eh, Ch, inst.targets, lse, 1.0, 6e-8)
    assert abs(float(out.loss) - loss) <= 1e-2 * abs(loss) + 1e-6
    assert abs(bwd.skipped_fraction - frac) <= 2e-3
    gx = bwd.grads.d_embeddings.double().cpu().numpy()
    ge = bwd.grads.d_classifier.double().cpu().numpy()
    assert np.linalg.norm(gx - dX) <= 0.1 * np.linalg.norm(dX)
    assert np.linalg.norm(ge - dC.T) <= 0.1 * np.linalg.norm(dC)


@pytest.mark.parametrize("gamma", [0.0, 1.0])
def test_bf16_filtered_backward_without_stats(lf, gamma):
    """stats=False selects the production kernels (no skip counters): with
    eps < 2^-12 the onehot part of softmax - onehot is applied at the
    accumulator read-out instead of inside the tile loop.  Same gradients as
    the filtered oracle at the bf16 tolerances."""
    n, d, v = 384, 64, 40000
    inst = ob.make_instance(ob.Rng(0xB2000003), n, d, v)
    Eref = (inst.E + gamma * inst.C.T[inst.targets]).astype(np.float32)
    X, E, Eh, Ch = prepare(Eref, inst.C, torch.bfloat16)
    x = torch.from_numpy(inst.targets).cuda()
    cfg = lf.CceConfig(filter_eps=6e-8)
    out = lf.cce_forward(X, E, x, cfg)
    bwd = lf.cce_backward(X, E, x, out.lse, 1.0, cfg, stats=False)
    loss, pos, lse = ob.cce_forward(Eh, Ch, inst.targets)
    dX, dC, _, _ = ob.cce_backward(Eh, Ch, inst.targets, lse, 1.0, 6e-8)
    check_grad(bwd.grads.d_embeddings, dX, torch.bfloat16, "dX")
    check_grad(bwd.grads.d_classifier, dC.T, torch.bfloat16, "dE")
    # negative upstream flips the sign of both gradients exactly
    neg = lf.cce_backward(X, E, x, out.lse, -1.0, cfg, stats=False)
    assert torch.equal(neg.grads.d_embeddings, -bwd.grads.d_embeddings)
    assert torch.equal(neg.grads.d_classifier, -bwd.grads.d_classifier)
