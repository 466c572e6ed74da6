"""Quick GPU-vs-oracle check of every path (developer tool; the real parity
suite is tests/test_*_gpu.py).  Prints one line per case."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_bind as ob  # noqa: E402
import paper_2509_09682_b200 as lf  # noqa: E402


def bf16_round(a):
    return torch.from_numpy(a).to(torch.bfloat16).float().numpy()


def run_cce(n, d, v, dtype, eps=0.0, seed=1):
    rng = ob.Rng(seed)
    inst = ob.make_instance(rng, n, d, v)
    Xh, Ch, t = inst.E, inst.C, inst.targets
    if dtype == torch.bfloat16:
        Xh = bf16_round(Xh)
        Ch = bf16_round(Ch)
    t0 = time.time()
    loss, pos, lse = ob.cce_forward(Xh, Ch, t)
    dE_o, dC_o, frac, _ = ob.cce_backward(Xh, Ch, t, lse, 1.0, eps)
    to = time.time() - t0
    dev = "cuda"
    X = torch.from_numpy(Xh).to(dev).to(dtype)
    E = torch.from_numpy(np.ascontiguousarray(Ch.T)).to(dev).to(dtype)
    x = torch.from_numpy(t).to(dev)
    cfg = lf.CceConfig(filter_eps=eps)
    out = lf.cce_forward(X, E, x, cfg)
    res = lf.cce_backward(X, E, x, out.lse, 1.0, cfg)
    torch.cuda.synchronize()
    gl = float(out.loss)
    lse_g = out.lse.cpu().numpy()
    pos_g = out.pos_logits.cpu().numpy()
    dX = res.grads.d_embeddings.double().cpu().numpy()
    dE = res.grads.d_classifier.double().cpu().numpy()
    rel = lambda a, b: float(np.max(np.abs(a - b) / np.maximum(1, np.abs(b))))
    nrm = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
    print(f"cce {str(dtype):15s} n={n} d={d} v={v} eps={eps}: loss {gl:.8f} vs {loss:.8f} "
          f"rel={abs(gl-loss)/max(1,abs(loss)):.2e} lse={rel(lse_g, lse):.2e} "
          f"pos_eq={bool((pos_g == pos).all())} pos={rel(pos_g, pos):.2e} "
          f"dX={nrm(dX, dE_o):.2e} dE={nrm(dE, dC_o.T):.2e} skip={res.skipped_fraction:.4f} "
          f"vs {frac:.4f} (oracle {to:.1f}s)", flush=True)


def run_ccem(n, d, v, ns, dtype, seed=3, atomic=False):
    rng = ob.Rng(seed)
    inst = ob.make_instance(rng, n, d, v)
    Xh, Ch, t = inst.E, inst.C, inst.targets
    inds = ob.sample_uniform(t, ns, v, seed + 7)
    if dtype == torch.bfloat16:
        Xh = bf16_round(Xh)
        Ch = bf16_round(Ch)
    loss, pos, lse = ob.ccem_forward(Xh, Ch, inds)
    dE_o, dC_o = ob.ccem_backward(Xh, Ch, inds, lse, 1.0)
    dev = "cuda"
    X = torch.from_numpy(Xh).to(dev).to(dtype)
    E = torch.from_numpy(np.ascontiguousarray(Ch.T)).to(dev).to(dtype)
    I = torch.from_numpy(inds).to(dev)
    cfg = lf.CceConfig(atomic_de=atomic)
    out = lf.ccem_forward(X, E, I, cfg)
    g = lf.ccem_backward(X, E, I, out.lse, 1.0, cfg)
    torch.cuda.synchronize()
    gl = float(out.loss)
    dX = g.d_embeddings.double().cpu().numpy()
    dE = g.d_classifier.double().cpu().numpy()
    pos_g = out.pos_logits.cpu().numpy()
    nrm = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
    print(f"ccem {str(dtype):15s} n={n} d={d} v={v} ns={ns} atomic={atomic}: loss {gl:.8f} vs "
          f"{loss:.8f} pos_eq={bool((pos_g == pos).all())} dX={nrm(dX, dE_o):.2e} "
          f"dE={nrm(dE, dC_o.T):.2e}", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "simt"):
        run_cce(37, 8, 53, torch.float64)
        run_cce(37, 8, 53, torch.float64, eps=1e-3)
        run_cce(300, 64, 5000, torch.float32)
        run_ccem(41, 8, 67, 9, torch.float64)
        run_ccem(300, 64, 5000, 63, torch.float32)
        run_ccem(300, 64, 5000, 63, torch.bfloat16)
        run_ccem(300, 64, 5000, 63, torch.bfloat16, atomic=True)
    if which in ("all", "tc"):
        run_cce(128, 64, 128, torch.bfloat16)
        run_cce(300, 64, 5000, torch.bfloat16)
        run_cce(300, 128, 3000, torch.bfloat16)
        run_cce(1000, 64, 20000, torch.bfloat16, eps=1e-6)
        run_cce(200, 256, 1000, torch.bfloat16)
