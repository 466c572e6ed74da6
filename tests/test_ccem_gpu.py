"""GPU parity of CCE- (ccem_forward / ccem_backward / ccem_backward_rows)
against the oracle and the reference's golden fixtures; cases follow
proj/tests/test_ccem.cpp."""
import os

import numpy as np
import pytest
import torch

import oracle_bind as ob
from gpu_util import TOL, check_grad, prepare

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def lf(cuda):
    import paper_2509_09682_b200 as lf
    return lf


def to_dev(Eh, Ch, inds, dtype):
    X, E, Eh2, Ch2 = prepare(Eh, Ch, dtype)
    return X, E, torch.from_numpy(np.ascontiguousarray(inds)).cuda(), Eh2, Ch2


def compare(lf, X, E, I, Eh, Ch, inds, dtype, atomic=False, row_up=None):
    tol = TOL[dtype]
    cfg = lf.CceConfig(atomic_de=atomic)
    out = lf.ccem_forward(X, E, I, cfg)
    n = X.shape[0]
    up = np.full(n, 1.0 / n) if row_up is None else row_up
    if row_up is None:
        g = lf.ccem_backward(X, E, I, out.lse, 1.0, cfg)
    else:
        g = lf.ccem_backward_rows(X, E, I, out.lse, torch.from_numpy(row_up).cuda(), cfg)
    loss, pos, lse = ob.ccem_forward(Eh, Ch, inds)
    dE, dC = ob.ccem_backward_rows(Eh, Ch, inds, lse, up)
    assert ob.rel_err(float(out.loss), loss) < tol["loss"]
    assert ob.rel_err(out.lse.cpu().numpy(), lse).max() < tol["lse"]
    if dtype == torch.float64:
        assert np.array_equal(out.pos_logits.cpu().numpy(), pos)  # test_ccem.cpp:53
    check_grad(g.d_embeddings, dE, dtype, "dX")
    check_grad(g.d_classifier, dC.T, dtype, "dE")
    return out, g


def test_exact_mode_random_instances(lf):  # test_ccem.cpp:36-64
    rng = ob.Rng(2002)
    for _ in range(40):
        n, d, v = 1 + rng.bounded(32), 1 + rng.bounded(16), 2 + rng.bounded(127)
        ns = min(rng.bounded(32), v - 1)
        inst = ob.make_instance(rng, n, d, v)
        inds = ob.make_candidates(rng, inst.targets, ns, v)
        X, E, I, Eh, Ch = to_dev(inst.E, inst.C, inds, torch.float64)
        compare(lf, X, E, I, Eh, Ch, inds, torch.float64)


def test_golden_fixtures(lf):
    g = np.load(os.path.join(GOLDEN, "ccem_ref.npz"))
    for k in range(int(g["count"])):
        Eh, Ch, inds = g[f"{k}_E"], g[f"{k}_C"], g[f"{k}_inds"]
        for dtype in (torch.float64, torch.float32, torch.bfloat16):
            if dtype == torch.bfloat16 and Eh.shape[1] % 64:
                continue
            X, E, I, Eh2, Ch2 = to_dev(Eh, Ch, inds, dtype)
            out, gr = compare(lf, X, E, I, Eh2, Ch2, inds, dtype)
            if dtype == torch.float64:
                assert float(out.loss) == pytest.approx(float(g[f"{k}_loss"]), rel=1e-12)
                assert np.array_equal(out.pos_logits.cpu().numpy(), g[f"{k}_pos"])
                # ordered segment reduce in (row, slot) order = reference order
                assert ob.rel_err(gr.d_classifier.cpu().numpy(), g[f"{k}_dC"].T).max() < 1e-12


@pytest.mark.parametrize("dtype,d", [(torch.float32, 64), (torch.bfloat16, 64),
                                     (torch.bfloat16, 128), (torch.float32, 24)])
@pytest.mark.parametrize("atomic", [False, True])
def test_sampled_shapes(lf, dtype, d, atomic):
    if atomic and d % 64:
        pytest.skip("atomic dE needs d % 64 == 0")
    n, v, ns = 333, 4096, 127
    rng = ob.Rng(0xB2000003)
    inst = ob.make_instance(rng, n, d, v)
    inds = ob.sample_uniform(inst.targets, ns, v, 0xB2000003 + 7)
    X, E, I, Eh, Ch = to_dev(inst.E, inst.C, inds, dtype)
    compare(lf, X, E, I, Eh, Ch, inds, dtype, atomic=atomic)


def test_cfg3_geometry_row_slice(lf):
    """cfg3: D=64, V=1M, K=512 uniform negatives (sampler.cpp:44-75) on 2048 rows."""
    n, d, v, ns = 2048, 64, 1_000_000, 512
    rng = ob.Rng(0xB2000003)
    inst = ob.make_instance(rng, n, d, v)
    inds = ob.sample_uniform(inst.targets, ns, v, 0xB2000003 + 7)
    X, E, I, Eh, Ch = to_dev(inst.E, inst.C, inds, torch.bfloat16)
    compare(lf, X, E, I, Eh, Ch, inds, torch.bfloat16)


def test_zero_negatives_loss_is_zero(lf):  # test_ccem.cpp:66-76
    rng = ob.Rng(12)
    inst = ob.make_instance(rng, 5, 3, 9)
    inds = inst.targets.reshape(-1, 1).copy()
    X, E, I, _, _ = to_dev(inst.E, inst.C, inds, torch.float64)
    out = lf.ccem_forward(X, E, I)
    assert float(out.loss) == 0.0
    assert torch.equal(out.lse, out.pos_logits)


def test_full_coverage_collapses_to_full_loss(lf):  # test_ccem.cpp:78-103
    rng = ob.Rng(21)
    inst = ob.make_instance(rng, 6, 4, 10)
    inds = np.stack([np.concatenate([[t], [j for j in range(10) if j != t]])
                     for t in inst.targets]).astype(np.int64)
    X, E, I, _, _ = to_dev(inst.E, inst.C, inds, torch.float64)
    x = torch.from_numpy(inst.targets).cuda()
    full = lf.cce_forward(X, E, x)
    samp = lf.ccem_forward(X, E, I)
    assert ob.rel_err(float(samp.loss), float(full.loss)) < 1e-10
    gf = lf.cce_backward(X, E, x, full.lse, 1.0).grads
    gs = lf.ccem_backward(X, E, I, samp.lse, 1.0)
    assert ob.rel_err(gs.d_embeddings.cpu().numpy(), gf.d_embeddings.cpu().numpy()).max() < 1e-10
    assert ob.rel_err(gs.d_classifier.cpu().numpy(), gf.d_classifier.cpu().numpy()).max() < 1e-10


def test_slot_permutation_invariance(lf):  # test_ccem.cpp:105-135
    rng = ob.Rng(31)
    inst = ob.make_instance(rng, 8, 5, 30)
    inds = ob.make_candidates(rng, inst.targets, 7, 30)
    perm = inds.copy()
    for r in range(perm.shape[0]):
        perm[r, 1:] = perm[r, 1:][::-1]
        if r % 2 == 0:
            perm[r, [1, 3]] = perm[r, [3, 1]]
    X, E, I, _, _ = to_dev(inst.E, inst.C, inds, torch.float64)
    P = torch.from_numpy(perm).cuda()
    a, b = lf.ccem_forward(X, E, I), lf.ccem_forward(X, E, P)
    assert ob.rel_err(float(a.loss), float(b.loss)) < 1e-10
    assert torch.equal(a.pos_logits, b.pos_logits)
    ga, gb = lf.ccem_backward(X, E, I, a.lse), lf.ccem_backward(X, E, P, b.lse)
    assert ob.rel_err(ga.d_embeddings.cpu().numpy(), gb.d_embeddings.cpu().numpy()).max() < 1e-10
    assert ob.rel_err(ga.d_classifier.cpu().numpy(), gb.d_classifier.cpu().numpy()).max() < 1e-10


def test_shared_negative_hand_case(lf):  # test_ccem.cpp:137-169
    Eh = np.array([[1.0, 0.0], [0.0, 2.0]], np.float32)
    Ch = np.array([[0.3, -0.2, 0.1], [-0.5, 0.4, 0.2]], np.float32)
    inds = np.array([[0, 2], [1, 2]], np.int64)
    X, E, I, _, _ = to_dev(Eh, Ch, inds, torch.float64)
    out = lf.ccem_forward(X, E, I)
    g = lf.ccem_backward(X, E, I, out.lse, 1.0)
    lse = out.lse.cpu().numpy()
    want = np.zeros(2)
    for i in range(2):
        logit = sum(float(Eh[i, k]) * float(Ch[k, 2]) for k in range(2))
        want += 0.5 * np.exp(logit - lse[i]) * Eh[i].astype(np.float64)
    dE = g.d_classifier.cpu().numpy()
    assert np.allclose(dE[2], want, rtol=1e-12, atol=0)
    s00 = np.exp(out.pos_logits.cpu().numpy()[0] - lse[0])
    assert dE[0, 0] == pytest.approx(0.5 * (s00 - 1.0), rel=1e-12)
    assert dE[0, 1] == 0.0


def test_untouched_columns_exact_zero(lf):  # test_ccem.cpp:171-185
    rng = ob.Rng(47)
    inst = ob.make_instance(rng, 4, 64, 25)
    inds = ob.make_candidates(rng, inst.targets, 2, 25)
    for dtype in (torch.float64, torch.bfloat16):
        X, E, I, _, _ = to_dev(inst.E, inst.C, inds, dtype)
        out = lf.ccem_forward(X, E, I)
        g = lf.ccem_backward(X, E, I, out.lse)
        untouched = np.setdiff1d(np.arange(25), np.unique(inds))
        assert (g.d_classifier.cpu()[untouched] == 0).all()


def test_row_upstream_generalizes_scalar(lf):  # test_ccem.cpp:208-223
    rng = ob.Rng(88)
    inst = ob.make_instance(rng, 6, 4, 14)
    inds = ob.make_candidates(rng, inst.targets, 3, 14)
    X, E, I, Eh, Ch = to_dev(inst.E, inst.C, inds, torch.float64)
    out = lf.ccem_forward(X, E, I)
    a = lf.ccem_backward(X, E, I, out.lse, 2.5)
    b = lf.ccem_backward_rows(X, E, I, out.lse, torch.full((6,), 2.5 / 6, dtype=torch.float64,
                                                            device="cuda"))
    assert torch.equal(a.d_embeddings, b.d_embeddings)
    assert torch.equal(a.d_classifier, b.d_classifier)
    compare(lf, X, E, I, Eh, Ch, inds, torch.float64, row_up=np.linspace(0.1, 3.0, 6))


def test_deterministic_default_is_bitwise_stable(lf):  # test_ccem.cpp:242-262
    rng = ob.Rng(272)
    inst = ob.make_instance(rng, 410, 64, 6700)
    inds = ob.make_candidates(rng, inst.targets, 90, 6700)
    X, E, I, _, _ = to_dev(inst.E, inst.C, inds, torch.bfloat16)
    out = lf.ccem_forward(X, E, I)
    ref = lf.ccem_backward(X, E, I, out.lse)
    for _ in range(3):
        g = lf.ccem_backward(X, E, I, out.lse)
        assert torch.equal(g.d_embeddings, ref.d_embeddings)
        assert torch.equal(g.d_classifier, ref.d_classifier)


def test_retained_memory_two_scalars_plus_indices(lf):  # test_ccem.cpp:225-240
    rng = ob.Rng(5)
    inst = ob.make_instance(rng, 8, 4, 32)
    for ns in (0, 3, 31):
        inds = ob.make_candidates(rng, inst.targets, ns, 32)
        X, E, I, _, _ = to_dev(inst.E, inst.C, inds, torch.float64)
        acct = lf.MemAccountant()
        out = lf.ccem_forward(X, E, I, lf.CceConfig(), acct)
        acct.expect_scratch_released()
        rep = acct.report()
        assert rep.current.retained_real == 16 and rep.current.retained_index == 8 * (1 + ns)
        lf.ccem_backward(X, E, I, out.lse, 1.0, lf.CceConfig(), acct)
        acct.expect_scratch_released()
        assert acct.report().current.retained_real == 16


def test_invalid_indices_name_the_row(lf):  # neg_index.cpp:13-25
    rng = ob.Rng(9)
    inst = ob.make_instance(rng, 4, 4, 10)
    inds = ob.make_candidates(rng, inst.targets, 3, 10)
    bad = inds.copy()
    bad[2, 1] = bad[2, 0]
    X, E, I, _, _ = to_dev(inst.E, inst.C, bad, torch.float64)
    with pytest.raises(ValueError, match="row 2 repeats its positive item"):
        lf.ccem_forward(X, E, I)
    bad = inds.copy()
    bad[1, 2] = 10
    I = torch.from_numpy(bad).cuda()
    with pytest.raises(ValueError, match="row 1 slot 2 holds 10, outside catalog of 10"):
        lf.ccem_forward(X, E, I)


@pytest.mark.parametrize("v", [300, 150, 40])
def test_segment_length_classes(lf, v):
    # items with ~85, ~170 and ~640 entries: the 128- and 256-key warp sorts
    # and the radix fallback of the deterministic dE; exact against the
    # oracle's tolerance and bitwise stable
    rng = ob.Rng(900 + v)
    inst = ob.make_instance(rng, 400, 64, v)
    inds = ob.make_candidates(rng, inst.targets, 63, v)
    X, E, I, Eh, Ch = to_dev(inst.E, inst.C, inds, torch.bfloat16)
    out, g = compare(lf, X, E, I, Eh, Ch, inds, torch.bfloat16)
    g2 = lf.ccem_backward(X, E, I, out.lse)
    assert torch.equal(g.d_classifier, g2.d_classifier)
