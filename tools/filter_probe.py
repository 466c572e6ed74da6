"""Developer probe: the saturated-gradient filter on distribution B
(X_i = U(-1,1)^D + gamma E_(x_i)) at the cfg2 shape — per
kernel CUDA-event ms of lf_cce_forward_backward, the skip statistics, and
(--once) a single call for ncu."""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_09682_b200 as lf  # noqa: E402
from paper_2509_09682_b200 import _capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=51200)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--v", type=int, default=1000000)
ap.add_argument("--gamma", type=float, default=2.0)
ap.add_argument("--eps", type=float, nargs="+", default=[6e-8])
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--once", type=int, default=0)
a = ap.parse_args()

g = torch.Generator(device="cuda").manual_seed(0)
E = (torch.rand(a.v, a.d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
x = torch.randint(0, a.v, (a.n,), device="cuda", generator=g)
X = ((torch.rand(a.n, a.d, device="cuda", generator=g) * 2 - 1) + a.gamma * E[x].float()).to(torch.bfloat16)
L = _capi.lib()
for eps in a.eps:
    cfg = lf.CceConfig(filter_eps=eps)
    step = lambda: lf.cce_forward_backward(X, E, x, 1.0, cfg, validate=False)
    if a.once:
        step()
        torch.cuda.synchronize()
        continue
    step()
    torch.cuda.synchronize()
    L.lf_profile_reset()
    L.lf_profile_enable(1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.iters):
        step()
    e.record()
    torch.cuda.synchronize()
    L.lf_profile_enable(0)
    kern = {}
    for kind, name in enumerate(_capi.KERNEL_KINDS):
        cnt, ms = C.c_uint64(), C.c_double()
        L.lf_profile_read(kind, C.byref(cnt), C.byref(ms))
        if cnt.value:
            kern[name] = round(ms.value / a.iters, 3)
    o, r = lf.cce_forward_backward(X, E, x, 1.0, cfg, validate=False, stats=True)
    print(f"gamma={a.gamma} eps={eps:g}: {s.elapsed_time(e) / a.iters:.3f} ms/step {kern} "
          f"loss={float(o.loss):.6g} skipped={r.skipped_fraction:.6f} "
          f"subtiles={r.skipped_tiles}/{r.total_tiles}", flush=True)
