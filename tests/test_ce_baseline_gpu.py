"""GPU: the materialising CE baseline (lf_ce_*, losses.cpp:71-140) matches the
oracle, and equals the fused CCE path on the same inputs (the paper's CE == CCE
equivalence, test_trainer.cpp:211-237) — CCE just never writes the logits."""
import numpy as np
import pytest
import torch

import oracle_bind as ob
from gpu_util import check_grad, instance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lf(cuda):
    import paper_2509_09682_b200 as lf
    return lf


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16])
def test_ce_matches_oracle_and_cce(lf, dtype):
    X, E, x, Eh, Ch, t = instance(0xCE, 300, 64, 5000, dtype)
    out = lf.ce_full_forward(X, E, x)
    g = lf.ce_full_backward(X, E, x, 1.0)
    loss, pos, lse = ob.cce_forward(Eh, Ch, t)
    dX, dC, _, _ = ob.cce_backward(Eh, Ch, t, lse, 1.0, 0.0)
    tol = {torch.float64: 1e-9, torch.float32: 1e-5, torch.bfloat16: 1e-2}[dtype]
    assert abs(float(out.loss) - loss) <= tol * max(1.0, abs(loss))
    assert np.abs(out.lse.cpu().numpy() - lse).max() <= 1e-3 if dtype == torch.bfloat16 else True
    check_grad(g.d_embeddings, dX, dtype if dtype != torch.float64 else torch.float32, "dX")
    check_grad(g.d_classifier, dC.T, dtype if dtype != torch.float64 else torch.float32, "dE")
    cce = lf.cce_forward(X, E, x)
    assert abs(float(cce.loss) - float(out.loss)) <= tol * max(1.0, abs(loss))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16])
def test_sampled_ce_matches_oracle_and_ccem(lf, dtype):
    # losses.cpp:142-221 (materialising) == ccem.cpp (fused) on the same candidates
    X, E, x, Eh, Ch, t = instance(0xCE2, 257, 64, 3000, dtype)
    inds_np = ob.sample_uniform(t, 63, 3000, 0xCE3)
    inds_np[:, 5] = inds_np[:, 4]  # a duplicated candidate column accumulates additively
    I = torch.from_numpy(inds_np).cuda()
    out = lf.ce_sampled_forward(X, E, I)
    g = lf.ce_sampled_backward(X, E, I, 1.0)
    loss, pos, lse = ob.ccem_forward(Eh, Ch, inds_np)
    dX, dC = ob.ccem_backward(Eh, Ch, inds_np, lse, 1.0)
    tol = {torch.float64: 1e-9, torch.float32: 1e-5, torch.bfloat16: 1e-2}[dtype]
    assert abs(float(out.loss) - loss) <= tol * max(1.0, abs(loss))
    check_grad(g.d_embeddings, dX, dtype if dtype != torch.float64 else torch.float32, "dX")
    check_grad(g.d_classifier, dC.T, dtype if dtype != torch.float64 else torch.float32, "dE")
    fused = lf.ccem_forward(X, E, I)
    assert abs(float(fused.loss) - float(out.loss)) <= tol * max(1.0, abs(loss))
