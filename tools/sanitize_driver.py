"""Small-shape driver for compute-sanitizer: one call of every device kernel
family of liblseforge_b200.so — the tcgen05 modes (FWD, BWD_ROWS, BWD_ITEMS
with each FLAGS instantiation, FWDX fused, EVAL with each list class), the
fp32 / fp64 SIMT kernels, CCE- forward / backward (deterministic and atomic
dE), the samplers, the materialising CE / CE- baselines, Adam, the encoder,
the layout converters and the bounded peer barrier (world 1).

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_09682_b200 as lf  # noqa: E402
from paper_2509_09682_b200 import _capi, metrics  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)


def rnd(*shape, dtype=torch.float32):
    return ((torch.rand(*shape, device=dev, generator=g) * 2 - 1)).to(dtype)


def main():
    n, v, k = 200, 1000, 15
    cases = ((torch.bfloat16, 64), (torch.bfloat16, 128), (torch.bfloat16, 256), (torch.float32, 64),
             (torch.float64, 16))
    only = os.environ.get("LF_SANITIZE_D")  # developer filter, e.g. "256"
    if only:
        cases = tuple(c for c in cases if str(c[1]) == only)
    for dtype, d in cases:
        X, E = rnd(n, d, dtype=dtype), rnd(v, d, dtype=dtype)
        x = torch.randint(0, v, (n,), device=dev, generator=g)
        for eps in (0.0, 6e-8, 2.0 ** -8, 1.0):
            cfg = lf.CceConfig(filter_eps=eps)
            out = lf.cce_forward(X, E, x, cfg)
            for stats in (False, True):
                lf.cce_backward(X, E, x, out.lse, 1.0, cfg, stats=stats)
                lf.cce_forward_backward(X, E, x, 1.0, cfg, stats=stats)
        inds = lf.sample_uniform(x, k, v, 11)
        o = lf.ccem_forward(X, E, inds)
        lf.ccem_backward(X, E, inds, o.lse, 1.0)
        lf.ccem_backward(X, E, inds, o.lse, 1.0, lf.CceConfig(atomic_de=True))
        lf.ce_sampled_backward(X, E, inds)
        lf.ce_sampled_forward(X, E, inds)
        if dtype != torch.float64 or d <= 16:
            lf.ce_full_forward(X, E, x)
            lf.ce_full_backward(X, E, x)
        for kk in (3, 7, 10, 16):
            metrics.rank_topk(X, E, x, kk)
    # the fused step's rebase path: peaked rows (target ~80 nats above the rest)
    Eb = rnd(3000, 64, dtype=torch.float32) * 3
    t = torch.randint(0, 3000, (256,), device=dev, generator=g)
    Xb = (Eb[t] + Eb[(t + 1) % 3000]).to(torch.bfloat16) * 0.5
    lf.cce_forward_backward(Xb.contiguous(), Eb.to(torch.bfloat16), t, 1.0, lf.CceConfig())
    # popularity sampler (exponent 1 and not), Adam, layout converters
    counts = torch.randint(0, 50, (v,), device=dev, generator=g)
    x = torch.randint(0, v, (n,), device=dev, generator=g)
    lf.sample_popularity(x, 5, counts, 3)
    lf.sample_popularity(x, 5, counts, 3, exponent=0.75)
    P = rnd(4096)
    lf.DeviceAdam([P]).step([rnd(4096)])
    L = _capi.lib()
    st = torch.cuda.current_stream(dev).cuda_stream
    Cm = rnd(64, 333)
    Eo = torch.empty(333, 64, dtype=torch.bfloat16, device=dev)
    _capi.check(L.lf_classifier_to_items(Cm.data_ptr(), 64, 333, _capi.LF_BF16, Eo.data_ptr(), st))
    dC = torch.empty(64, 333, dtype=torch.float64, device=dev)
    dE = rnd(333, 64)
    _capi.check(L.lf_items_grad_to_classifier(dE.data_ptr(), _capi.LF_BF16, 333, 64, dC.data_ptr(), st))
    # bounded peer barrier, world 1 (signal + wait on its own flag)
    flags = torch.zeros(4, dtype=torch.int32, device=dev)
    table = torch.tensor([flags.data_ptr()], dtype=torch.int64, device=dev)
    _capi.check(L.lf_peer_barrier(table.data_ptr(), 1, 0, 1, st))
    torch.cuda.synchronize()
    _capi.check(L.lf_peer_status())
    print("sanitize driver: ok")


if __name__ == "__main__":
    main()
