"""Developer check: accuracy of the bf16 backward WITH filtering (eps = 6e-8)
against the CPU oracle, for the library selected by LSEFORGE_B200_LIB.
Prints normwise errors of dX and dE and the skipped fraction.

    LSEFORGE_B200_LIB=... python tools/filter_accuracy.py [--v 65536] [--gamma 0]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_bind as ob  # noqa: E402
import paper_2509_09682_b200 as lf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--v", type=int, default=65536)
ap.add_argument("--eps", type=float, default=6e-8)
ap.add_argument("--gamma", type=float, default=0.0)
a = ap.parse_args()

inst = ob.make_instance(ob.Rng(0xB2000002), a.n, a.d, a.v)
E = inst.E + a.gamma * inst.C.T[inst.targets]          # "trained-like" rows
Eh = torch.from_numpy(E.astype(np.float32)).to(torch.bfloat16)
Ch = torch.from_numpy(inst.C).to(torch.bfloat16)
Ef, Cf = Eh.float().numpy(), Ch.float().numpy()
X, Ed, x = Eh.cuda(), Ch.t().contiguous().cuda(), torch.from_numpy(inst.targets).cuda()
cfg = lf.CceConfig(filter_eps=a.eps)
out = lf.cce_forward(X, Ed, x, cfg)
res = lf.cce_backward(X, Ed, x, out.lse, 1.0, cfg)
loss, pos, lse = ob.cce_forward(Ef, Cf, inst.targets)
dX, dC, frac, _ = ob.cce_backward(Ef, Cf, inst.targets, lse, 1.0, a.eps)
gx = res.grads.d_embeddings.double().cpu().numpy()
ge = res.grads.d_classifier.double().cpu().numpy()
nx = np.linalg.norm(gx - dX) / np.linalg.norm(dX)
ne = np.linalg.norm(ge - dC.T) / np.linalg.norm(dC)
print(f"lib={os.path.basename(os.environ.get('LSEFORGE_B200_LIB', 'default'))} gamma={a.gamma} "
      f"loss={loss:.4f} dX_norm_err={nx:.3e} dE_norm_err={ne:.3e} skipped={res.skipped_fraction:.4f} "
      f"(oracle {frac:.4f})")
