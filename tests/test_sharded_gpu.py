"""GPU: the device side of catalog sharding (lf_cce_forward_partial,
lf_cce_combine, lf_cce_backward_shard) on one GPU — P shards computed in
turn and exchanged in-process exactly as ShardedCce exchanges them across
ranks — equals the unsharded path and the oracle."""
import numpy as np
import pytest
import torch

import oracle_bind as ob
from gpu_util import check_grad, instance

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,d,P", [(torch.bfloat16, 64, 2), (torch.bfloat16, 128, 4),
                                       (torch.float32, 64, 3), (torch.float64, 8, 5)])
def test_sharded_equals_unsharded(cuda, dtype, d, P):
    import paper_2509_09682_b200 as lf
    from paper_2509_09682_b200.sharded import DeviceKernels, shard_bounds
    n, v, eps = 300, 5003, 1e-6
    X, E, x, Eh, Ch, t = instance(0xB2000004 + P, n, d, v, dtype)
    cfg = lf.CceConfig(filter_eps=eps)
    K = DeviceKernels()
    bounds = [shard_bounds(v, P, p) for p in range(P)]
    parts = torch.stack([K.forward_partial(X, E[b:e], x, b, cfg) for b, e in bounds])
    out = K.combine(parts)
    full = lf.cce_forward(X, E, x, cfg)
    assert ob.rel_err(float(out.loss), float(full.loss)) < 1e-6
    assert ob.rel_err(out.lse.cpu().numpy(), full.lse.cpu().numpy()).max() < 1e-6
    dX = None
    dE = []
    skipped = 0
    for b, e in bounds:
        dx, de, st = K.backward_shard(X, E[b:e], x, out.lse, 1.0, b, v, cfg, True)
        dX = dx if dX is None else dX + dx
        dE.append(de)
        skipped += st.skipped_elems
    dE = torch.cat(dE)
    _, _, lse = ob.cce_forward(Eh, Ch, t)
    dE_o, dC_o, frac, _ = ob.cce_backward(Eh, Ch, t, out.lse.cpu().numpy(), 1.0, eps)
    check_grad(dX, dE_o, dtype, "dX")
    check_grad(dE, dC_o.T, dtype, "dE")
    tol = 0.0 if dtype == torch.float64 else 2e-3
    assert abs(skipped / (n * (v - 1)) - frac) <= tol
