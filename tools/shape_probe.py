"""Developer probe: per-kernel CUDA-event ms of the 3-pass CCE (forward, dX
pass, dE pass) and of the fused call at a given shape (bf16, torch.rand
data), e.g. the per-GPU shards of configs 4 and 5."""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_09682_b200 as lf  # noqa: E402
from paper_2509_09682_b200 import _capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=7680)
ap.add_argument("--d", type=int, default=256)
ap.add_argument("--v", type=int, default=2000000)
ap.add_argument("--eps", type=float, default=6e-8)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
X = (torch.rand(a.n, a.d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
E = (torch.rand(a.v, a.d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
x = torch.randint(0, a.v, (a.n,), device="cuda", generator=g)
cfg = lf.CceConfig(filter_eps=a.eps)
L = _capi.lib()


def prof(fn, name):
    fn()
    torch.cuda.synchronize()
    L.lf_profile_reset()
    L.lf_profile_enable(1)
    for _ in range(a.iters):
        fn()
    torch.cuda.synchronize()
    L.lf_profile_enable(0)
    parts = {}
    for kind, kn in enumerate(_capi.KERNEL_KINDS):
        cnt, ms = C.c_uint64(), C.c_double()
        L.lf_profile_read(kind, C.byref(cnt), C.byref(ms))
        if cnt.value:
            parts[kn] = round(ms.value / a.iters, 3)
    print(f"{name} n={a.n} d={a.d} v={a.v} eps={a.eps}: {parts} total {sum(parts.values()):.3f} ms", flush=True)


def three_pass():
    o = lf.cce_forward(X, E, x, cfg, validate=False)
    lf.cce_backward(X, E, x, o.lse, 1.0, cfg, validate=False, stats=False)


prof(three_pass, "3-pass")
prof(lambda: lf.cce_forward_backward(X, E, x, 1.0, cfg, validate=False), "fused")
