"""Normwise dX / dE error of the fused CCE call against the f64 oracle on
trained-like rows (X_i = U(-1,1)^D + gamma E_(x_i)), D = 64: how much the
read-out form's exact target handling buys as p_t -> 1.  Select the library
with LSEFORGE_B200_LIB (A/B of variants)."""
import argparse
import sys

import numpy as np
import torch

ROOT = __file__.rsplit("/", 2)[0] if "/" in __file__ else ".."
sys.path[:0] = [ROOT, ROOT + "/tests"]
import oracle_bind as ob  # noqa: E402
from gpu_util import prepare  # noqa: E402

import paper_2509_09682_b200 as lf  # noqa: E402


def nerr(got, want):
    g = got.double().cpu().numpy()
    return float(np.linalg.norm(g - want) / max(np.linalg.norm(want), 1e-300))


ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1500)
ap.add_argument("--v", type=int, default=30000)
ap.add_argument("--d", type=int, default=64)
a = ap.parse_args()
for gamma in (0.0, 0.5, 1.0, 1.5):
    for eps in (0.0, 6e-8):
        inst = ob.make_instance(ob.Rng(0xACC0 + int(gamma * 10)), a.n, a.d, a.v)
        Eref = (inst.E + gamma * inst.C.T[inst.targets]).astype(np.float32)
        X, E, Eh, Ch = prepare(Eref, inst.C, torch.bfloat16)
        x = torch.from_numpy(inst.targets).cuda()
        loss, _, lse = ob.cce_forward(Eh, Ch, inst.targets)
        dX, dC, _, _ = ob.cce_backward(Eh, Ch, inst.targets, lse, 1.0, eps)
        out, res = lf.cce_forward_backward(X, E, x, 1.0, lf.CceConfig(filter_eps=eps))
        print(f"gamma={gamma} eps={eps:g} loss={loss:.4g} dX {nerr(res.grads.d_embeddings, dX):.2e}"
              f" dE {nerr(res.grads.d_classifier, dC.T):.2e}", flush=True)
