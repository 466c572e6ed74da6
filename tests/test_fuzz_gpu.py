"""GPU: seeded randomized parity sweep over the bf16 tensor-core paths — the
fused forward + dX (lf_cce_forward_backward), the separate forward / backward,
and the fused CCE- call — against the CPU oracle, across widths (64 / 128 /
256), ragged row and catalog counts, filter thresholds (exact, the preset
6e-8, 1e-6, and the coarse 2^-12 / 2^-8 that take the 3-pass path) and
uniform vs trained-like rows (X_i = U(-1,1)^D + gamma E_(x_i)), at the
tolerances every other bf16 test uses (tests/gpu_util.py TOL).

The logit margin of a trained-like row grows as gamma * D, so gamma is drawn
per 64 dimensions (gamma_64 * 64 / D, gamma_64 in {0, 0.5, 1}): losses from
~14 down to ~0.1.  Sharper rows (loss << 1e-3) leave this tolerance's reach
on any fp32 path — 1 - p_t approaches the fp32 resolution of the lse — and
are measured, not asserted, by tools/target_accuracy.py."""
import numpy as np
import pytest
import torch

import oracle_bind as ob
from gpu_util import TOL, check_grad, prepare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lf(cuda):
    import paper_2509_09682_b200 as lf
    return lf


def draw_cases(seed, count):
    r = np.random.default_rng(seed)
    cases = []
    for k in range(count):
        d = int(r.choice([64, 128, 256]))
        n = int(r.integers(1, 700))
        v = int(r.integers(2, 40000 if d < 256 else 12000))
        eps = float(r.choice([0.0, 6e-8, 1e-6, 2.0 ** -12, 2.0 ** -8]))
        gamma = float(r.choice([0.0, 0.5, 1.0])) * 64 / d
        cases.append((k, n, d, v, eps, gamma))
    return cases


def instance(k, n, d, v, gamma):
    inst = ob.make_instance(ob.Rng(0xF0220000 + k), n, d, v)
    Eref = (inst.E + gamma * inst.C.T[inst.targets]).astype(np.float32)
    X, E, Eh, Ch = prepare(Eref, inst.C, torch.bfloat16)
    return X, E, torch.from_numpy(inst.targets).cuda(), Eh, Ch, inst.targets


def check(out, res, Eh, Ch, t, eps):
    tol = TOL[torch.bfloat16]
    loss, pos, lse = ob.cce_forward(Eh, Ch, t)
    dX, dC, frac, _ = ob.cce_backward(Eh, Ch, t, lse, 1.0, eps)
    assert ob.rel_err(float(out.loss), loss) < tol["loss"]
    assert ob.rel_err(out.lse.cpu().numpy(), lse).max() < tol["lse"]
    check_grad(res.grads.d_embeddings, dX, torch.bfloat16, "dX")
    check_grad(res.grads.d_classifier, dC.T, torch.bfloat16, "dE")
    assert abs(res.skipped_fraction - frac) <= 2e-3, (res.skipped_fraction, frac)


@pytest.mark.parametrize("k,n,d,v,eps,gamma", draw_cases(0x5EED, 24))
def test_fused_and_separate_match_oracle(lf, k, n, d, v, eps, gamma):
    X, E, x, Eh, Ch, t = instance(k, n, d, v, gamma)
    cfg = lf.CceConfig(filter_eps=eps)
    out, res = lf.cce_forward_backward(X, E, x, 1.0, cfg, stats=True)
    check(out, res, Eh, Ch, t, eps)
    o2 = lf.cce_forward(X, E, x, cfg)
    r2 = lf.cce_backward(X, E, x, o2.lse, 1.0, cfg, stats=True)
    check(o2, r2, Eh, Ch, t, eps)


@pytest.mark.parametrize("k", range(8))
def test_fused_ccem_matches_oracle(lf, k):
    r = np.random.default_rng(0xCC3 + k)
    d = int(r.choice([64, 128, 256]))
    n, v = int(r.integers(1, 500)), int(r.integers(2, 6000))
    ns = int(r.integers(0, min(300, v - 1) + 1))
    inst = ob.make_instance(ob.Rng(0xF0330000 + k), n, d, v)
    inds = ob.make_candidates(ob.Rng(0xF0340000 + k), inst.targets, ns, v)
    X, E, Eh, Ch = prepare(inst.E, inst.C, torch.bfloat16)
    I = torch.from_numpy(np.ascontiguousarray(inds)).cuda()
    out, g = lf.ccem_forward_backward(X, E, I, 1.0)
    tol = TOL[torch.bfloat16]
    loss, pos, lse = ob.ccem_forward(Eh, Ch, inds)
    dE, dC = ob.ccem_backward_rows(Eh, Ch, inds, lse, np.full(n, 1.0 / n))
    assert ob.rel_err(float(out.loss), loss) < tol["loss"]
    assert ob.rel_err(out.lse.cpu().numpy(), lse).max() < tol["lse"]
    check_grad(g.d_embeddings, dE, torch.bfloat16, "dX")
    check_grad(g.d_classifier, dC.T, torch.bfloat16, "dE")


@pytest.mark.parametrize("gamma", [1.0, 1.5])
@pytest.mark.parametrize("eps", [0.0, 6e-8])
def test_well_fit_rows_keep_gradient_accuracy(lf, gamma, eps):
    """Rows the model already fits (p_t -> 1, loss 0.13 / 1e-3): the softmax
    enters the tensor cores in bf16, and rounding p_t there before subtracting
    the one-hot would swamp 1 - p_t (normwise errors of 1 % / 20 % before the
    read-out form).  Each row's target entry is left out of the product and
    added back as -(1 - p_t) with 1 - p_t = -expm1(t - lse) in full precision."""
    n, d, v = 1500, 64, 30000
    inst = ob.make_instance(ob.Rng(0xACC0 + int(gamma * 10)), n, d, v)
    Eref = (inst.E + gamma * inst.C.T[inst.targets]).astype(np.float32)
    X, E, Eh, Ch = prepare(Eref, inst.C, torch.bfloat16)
    x = torch.from_numpy(inst.targets).cuda()
    loss, _, lse = ob.cce_forward(Eh, Ch, inst.targets)
    dX, dC, _, _ = ob.cce_backward(Eh, Ch, inst.targets, lse, 1.0, eps)
    cfg = lf.CceConfig(filter_eps=eps)
    out, res = lf.cce_forward_backward(X, E, x, 1.0, cfg)
    o2 = lf.cce_forward(X, E, x, cfg)
    r2 = lf.cce_backward(X, E, x, o2.lse, 1.0, cfg)

    def nerr(got, want):
        return np.linalg.norm(got.double().cpu().numpy() - want) / np.linalg.norm(want)

    bound = 3e-3 if gamma == 1.0 else 6e-3
    for g in (res.grads, r2.grads):
        assert nerr(g.d_embeddings, dX) < bound
        assert nerr(g.d_classifier, dC.T) < bound
