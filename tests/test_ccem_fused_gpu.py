"""GPU parity of the fused CCE- forward + backward (lf_ccem_forward_backward,
one gather pass for lse / pos / dX and the entries' logits) against the
oracle (ccem.cpp:48-194) and against the two unfused calls: loss / lse / pos
within the dtype's tolerance of the oracle, dX within tolerance, dE bitwise
equal to lf_ccem_backward's (same logits, same coefficient formula, same
ordered reduce).  Cases follow proj/tests/test_ccem.cpp."""
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


def run_case(lf, Eh, Ch, inds, dtype, row_up=None, upstream=1.0):
    X, E, Eh2, Ch2 = prepare(Eh, Ch, dtype)
    I = torch.from_numpy(np.ascontiguousarray(inds)).cuda()
    n = X.shape[0]
    ru = None if row_up is None else torch.from_numpy(row_up).cuda()
    out, g = lf.ccem_forward_backward(X, E, I, upstream, row_upstream=ru)
    tol = TOL[dtype]
    loss, pos, lse = ob.ccem_forward(Eh2, Ch2, inds)
    up = np.full(n, upstream / n) if row_up is None else row_up
    dE, dC = ob.ccem_backward_rows(Eh2, Ch2, inds, lse, up)
    assert ob.rel_err(float(out.loss), loss) < tol["loss"]
    assert ob.rel_err(out.lse.cpu().numpy(), lse).max() < tol["lse"]
    assert ob.rel_err(out.pos_logits.cpu().numpy(), pos).max() < tol["lse"]
    check_grad(g.d_embeddings, dE, dtype, "dX")
    check_grad(g.d_classifier, dC.T, dtype, "dE")
    # the unfused pair on the same inputs: identical logits; fed the fused
    # call's lse, the unfused backward forms the same coefficients -> the
    # same dE bits (the two forwards' lse may differ in the last ulp: the
    # fused pass merges its per-group sums in a different order)
    o2 = lf.ccem_forward(X, E, I)
    assert torch.equal(out.pos_logits, o2.pos_logits)
    assert ob.rel_err(out.lse.cpu().numpy(), o2.lse.cpu().numpy()).max() < 1e-6
    if row_up is None:
        g2 = lf.ccem_backward(X, E, I, out.lse, upstream)
    else:
        g2 = lf.ccem_backward_rows(X, E, I, out.lse, ru)
    assert torch.equal(g.d_classifier, g2.d_classifier)
    return out, g


@pytest.mark.parametrize("dtype,d", [(torch.float32, 64), (torch.bfloat16, 64), (torch.bfloat16, 128),
                                     (torch.float32, 128), (torch.bfloat16, 256)])
def test_fused_matches_oracle_and_unfused(lf, dtype, d):
    n, v, ns = 333, 4096, 127
    rng = ob.Rng(0xB2000003)
    inst = ob.make_instance(rng, n, d, v)
    inds = ob.sample_uniform(inst.targets, ns, v, 0xB2000003 + 7)
    run_case(lf, inst.E, inst.C, inds, dtype)


@pytest.mark.parametrize("ns", [0, 1, 2, 3, 5, 17])
def test_fused_narrow_widths(lf, ns):
    """w = 1 + ns below one warp step (groups without slots merge as empty)."""
    n, d, v = 77, 64, 300
    rng = ob.Rng(77 + ns)
    inst = ob.make_instance(rng, n, d, v)
    inds = ob.make_candidates(rng, inst.targets, ns, v)
    out, _ = run_case(lf, inst.E, inst.C, inds, torch.float32)
    if ns == 0:  # only the positive: every loss term is zero (test_ccem.cpp:66-76)
        assert abs(float(out.loss)) < 1e-6


def test_fused_row_upstream_and_scalar_upstream(lf):
    n, d, v, ns = 129, 64, 2048, 63
    rng = ob.Rng(4242)
    inst = ob.make_instance(rng, n, d, v)
    inds = ob.sample_uniform(inst.targets, ns, v, 99)
    row_up = np.linspace(-0.5, 2.0, n)
    run_case(lf, inst.E, inst.C, inds, torch.float32, row_up=row_up)
    run_case(lf, inst.E, inst.C, inds, torch.bfloat16, upstream=-3.0)


def test_fused_duplicate_negatives_accumulate(lf):
    """Duplicated items inside a row add up (ccem.cpp:170-187)."""
    n, d, v, ns = 64, 64, 16, 40
    rng = ob.Rng(5)
    inst = ob.make_instance(rng, n, d, v)
    inds = ob.make_candidates(rng, inst.targets, ns, v)
    run_case(lf, inst.E, inst.C, inds, torch.float32)


def test_fused_falls_back_for_exact_and_atomic(lf):
    """f64 and LF_FLAG_ATOMIC_DE run the two unfused calls (same results)."""
    n, d, v, ns = 50, 24, 500, 31
    rng = ob.Rng(11)
    inst = ob.make_instance(rng, n, d, v)
    inds = ob.make_candidates(rng, inst.targets, ns, v)
    X, E, Eh, Ch = prepare(inst.E, inst.C, torch.float64)
    I = torch.from_numpy(np.ascontiguousarray(inds)).cuda()
    out, g = lf.ccem_forward_backward(X, E, I, 1.0)
    loss, pos, lse = ob.ccem_forward(Eh, Ch, inds)
    assert np.array_equal(out.pos_logits.cpu().numpy(), pos)
    dE, dC = ob.ccem_backward_rows(Eh, Ch, inds, lse, np.full(n, 1.0 / n))
    check_grad(g.d_embeddings, dE, torch.float64, "dX")
    Xb, Eb, Ehb, Chb = prepare(np.pad(inst.E, ((0, 0), (0, 40))), np.pad(inst.C, ((0, 40), (0, 0))),
                               torch.bfloat16)
    cfg = lf.CceConfig(atomic_de=True)
    out2, g2 = lf.ccem_forward_backward(Xb, Eb, I, 1.0, cfg)
    l2, _, lse2 = ob.ccem_forward(Ehb, Chb, inds)
    assert ob.rel_err(float(out2.loss), l2) < TOL[torch.bfloat16]["loss"]


def test_fused_cfg3_geometry_row_slice(lf):
    """cfg3: D = 64, V = 1M, K = 512 uniform negatives on 2048 rows."""
    n, d, v, ns = 2048, 64, 1_000_000, 512
    rng = ob.Rng(0xB2000003)
    inst = ob.make_instance(rng, n, d, v)
    inds = ob.sample_uniform(inst.targets, ns, v, 0xB2000003 + 7)
    run_case(lf, inst.E, inst.C, inds, torch.bfloat16)
