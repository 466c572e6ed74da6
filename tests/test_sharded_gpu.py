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


@pytest.mark.parametrize("d,P,v,n", [(128, 8, 262144, 512), (256, 8, 131072, 256)])
def test_sharded_config_shapes_reduced_catalog(cuda, d, P, v, n):
    """cfg4 (D=128) and cfg5 (D=256) geometry through the 8-way sharded code
    path at a reduced catalog (parity at reduced V), bf16,
    eps = 6e-8, production kernels (no stats): loss, lse and both gradients
    against the filtered oracle."""
    import paper_2509_09682_b200 as lf
    from paper_2509_09682_b200.sharded import DeviceKernels, shard_bounds
    X, E, x, Eh, Ch, t = instance(0xC0F4 + d, n, d, v, torch.bfloat16)
    cfg = lf.CceConfig(filter_eps=6e-8)
    K = DeviceKernels()
    bounds = [shard_bounds(v, P, p) for p in range(P)]
    parts = torch.stack([K.forward_partial(X, E[b:e], x, b, cfg) for b, e in bounds])
    out = K.combine(parts)
    loss, pos, lse = ob.cce_forward(Eh, Ch, t)
    assert ob.rel_err(float(out.loss), loss) < 1e-2
    assert ob.rel_err(out.lse.cpu().numpy(), lse).max() < 1e-3
    dX, dE = None, []
    for b, e in bounds:
        dx, de, _ = K.backward_shard(X, E[b:e], x, out.lse, 1.0, b, v, cfg, False)
        dX = dx if dX is None else dX + dx
        dE.append(de)
    dX_o, dC_o, _, _ = ob.cce_backward(Eh, Ch, t, lse, 1.0, 6e-8)
    check_grad(dX, dX_o, torch.bfloat16, "dX")
    check_grad(torch.cat(dE), dC_o.T, torch.bfloat16, "dE")


@pytest.mark.parametrize("d,P,v,n,eps", [(64, 2, 20011, 700, 6e-8), (64, 8, 100000, 512, 0.0),
                                         (128, 4, 30000, 300, 6e-8)])
def test_fused_sharded_phases_equal_oracle(cuda, d, P, v, n, eps):
    """The fused sharded step (lf_cce_fwdx_shard_begin on every shard, the
    ranks' (m, s, t) blocks gathered, lf_cce_fwdx_shard_end, dX partials
    summed) — the exchange ShardedCce.forward_backward runs across ranks —
    against the oracle; skip counts from the dE passes summed over shards."""
    from paper_2509_09682_b200.sharded import DeviceKernels, shard_bounds
    import paper_2509_09682_b200 as lf
    X, E, x, Eh, Ch, t = instance(0xF5ED + P + d, n, d, v, torch.bfloat16)
    cfg = lf.CceConfig(filter_eps=eps)
    K = DeviceKernels()
    assert K.fused_supported(X, cfg)
    bounds = [shard_bounds(v, P, p) for p in range(P)]
    begun = [K.fwdx_begin(X, E[b:e], x, b, cfg) for b, e in bounds]
    parts = torch.stack([p for p, _ in begun])
    dX, dE, skipped = None, [], 0
    for (b, e), (_, work) in zip(bounds, begun):
        out, dx, de, st = K.fwdx_end(work, parts, X, E[b:e], 1.0, v, True)
        dX = dx if dX is None else dX + dx
        dE.append(de)
        skipped += st.skipped_elems
    loss, pos, lse = ob.cce_forward(Eh, Ch, t)
    assert ob.rel_err(float(out.loss), loss) < 1e-2
    assert ob.rel_err(out.lse.cpu().numpy(), lse).max() < 1e-3
    dX_o, dC_o, frac, _ = ob.cce_backward(Eh, Ch, t, lse, 1.0, eps)
    check_grad(dX, dX_o, torch.bfloat16, "dX")
    check_grad(torch.cat(dE), dC_o.T, torch.bfloat16, "dE")
    assert abs(skipped / (n * (v - 1)) - frac) <= 2e-3
