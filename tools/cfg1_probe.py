"""Timing probe for BASELINE configs[0] (cfg1: fp32 CCE fwd + bwd, N = 2048,
D = 64, V = 32768, filtering off) through the public API: CUDA-event time
per step and the per-kernel split from the library's launch profiler.
Prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_09682_b200 as lf  # noqa: E402
from paper_2509_09682_b200 import synth  # noqa: E402

n, d, v = 2048, 64, 32768
Xh, Ch, t = synth.make_instance(0xB2000001, n, d, v)
X = torch.from_numpy(np.ascontiguousarray(Xh, np.float32)).cuda()
E = torch.from_numpy(np.ascontiguousarray(Ch.T, np.float32)).cuda()
x = torch.from_numpy(t).cuda()
cfg = lf.CceConfig()


def step_separate():
    o = lf.cce_forward(X, E, x, cfg, validate=False)
    return o, lf.cce_backward(X, E, x, o.lse, 1.0, cfg, validate=False, stats=False)


def step_fused():
    return lf.cce_forward_backward(X, E, x, 1.0, cfg, validate=False, stats=False)


step = step_fused if os.environ.get("CFG1_PATH", "fused") == "fused" else step_separate


for _ in range(3):
    step()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
iters = 20
s.record()
for _ in range(iters):
    step()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / iters
print(json.dumps({"probe": "cfg1", "path": os.environ.get("CFG1_PATH", "fused"), "ms_per_step": ms, "positions_per_s": n / ms * 1e3,
                  "tflops_fp32": 8 * n * v * d / ms * 1e-9}))
