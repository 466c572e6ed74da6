"""Developer timing probe: CUDA-event timing of the CCE forward / backward at a
given shape (default cfg2: n=51200, d=64, v=1M, bf16)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_09682_b200 as lf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=51200)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--v", type=int, default=1000000)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--eps", type=float, default=0.0)
ap.add_argument("--ccem", type=int, default=0)
ap.add_argument("--once", type=int, default=0)
ap.add_argument("--fused", type=int, default=0, help="time lf_cce_forward_backward")
a = ap.parse_args()

g = torch.Generator(device="cuda").manual_seed(0)
X = (torch.rand(a.n, a.d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
E = (torch.rand(a.v, a.d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
x = torch.randint(0, a.v, (a.n,), device="cuda", generator=g)
cfg = lf.CceConfig(filter_eps=a.eps)


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


if a.ccem:
    inds = torch.randint(0, a.v, (a.n, 1 + a.ccem), device="cuda", generator=g)
    inds[:, 0] = x
    out = lf.ccem_forward(X, E, inds, cfg, validate=False)
    tf = timed(lambda: lf.ccem_forward(X, E, inds, cfg, validate=False), a.iters)
    tb = timed(lambda: lf.ccem_backward(X, E, inds, out.lse, 1.0, cfg, validate=False), a.iters)
    cfg2 = lf.CceConfig(atomic_de=True)
    tba = timed(lambda: lf.ccem_backward(X, E, inds, out.lse, 1.0, cfg2, validate=False), a.iters)
    tfb = timed(lambda: lf.ccem_forward_backward(X, E, inds, 1.0, cfg, validate=False), a.iters)
    print(f"ccem n={a.n} d={a.d} v={a.v} K={a.ccem}: fwd {tf:.3f} ms  bwd(det) {tb:.3f} ms  "
          f"bwd(atomic) {tba:.3f} ms  pos/s={a.n/(tf+tb)*1e3:.3e}  fused fwd+bwd {tfb:.3f} ms "
          f"pos/s={a.n/tfb*1e3:.3e}")
elif a.fused:
    import ctypes as C
    from paper_2509_09682_b200 import _capi
    L = _capi.lib()
    step = lambda: lf.cce_forward_backward(X, E, x, 1.0, cfg, validate=False)
    if a.once:
        step()
        torch.cuda.synchronize()
        sys.exit(0)
    out, _ = step()
    print("loss", float(out.loss))
    t = timed(step, a.iters)
    L.lf_profile_reset()
    L.lf_profile_enable(1)
    step()
    torch.cuda.synchronize()
    L.lf_profile_enable(0)
    parts = []
    for kind, name in enumerate(_capi.KERNEL_KINDS):
        cnt, ms = C.c_uint64(), C.c_double()
        L.lf_profile_read(kind, C.byref(cnt), C.byref(ms))
        if cnt.value:
            parts.append(f"{name} {ms.value:.3f}")
    print(f"fused n={a.n} d={a.d} v={a.v} eps={a.eps}: {t:.3f} ms/step  pos/s={a.n/t*1e3:.3e}  "
          f"[{', '.join(parts)}]")
elif a.once:
    out = lf.cce_forward(X, E, x, cfg, validate=False)
    lf.cce_backward(X, E, x, out.lse, 1.0, cfg, validate=False, stats=False)
    torch.cuda.synchronize()
else:
    out = lf.cce_forward(X, E, x, cfg, validate=False)
    print("loss", float(out.loss))
    tf = timed(lambda: lf.cce_forward(X, E, x, cfg, validate=False), a.iters)
    tb = timed(lambda: lf.cce_backward(X, E, x, out.lse, 1.0, cfg, validate=False, stats=False),
               a.iters)
    L = a.n * a.v
    print(f"cce n={a.n} d={a.d} v={a.v}: fwd {tf:.3f} ms ({L/tf/1e9:.2f} Gelem/ms) bwd {tb:.3f} ms"
          f" total {tf+tb:.3f} ms  pos/s={a.n/(tf+tb)*1e3:.3e}  "
          f"fwd TFLOP/s={2*L*a.d/tf/1e9:.1f} bwd(exec 8LD) TFLOP/s={8*L*a.d/tb/1e9:.1f}")
