"""Timing probe for the device Adam step (lf_adam_step) on the cfg2
classifier (V = 1M x D = 64 float params, f32 dE, double moments, fused bf16
shadow): CUDA events, bytes moved per element (read param 4 + grad 4 +
moments 16, write param 4 + moments 16 + shadow 2 = 46 B) against the
measured HBM copy bandwidth.  One JSON line."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_09682_b200 as lf  # noqa: E402

v, d, iters = 1_000_000, 64, 10
p = torch.randn(v, d, device="cuda") * 0.05
g = torch.randn(v, d, device="cuda")
sh = torch.empty(v, d, dtype=torch.bfloat16, device="cuda")
opt = lf.DeviceAdam([p])
for _ in range(3):
    opt.step([g], [sh])
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(iters):
    opt.step([g], [sh])
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / iters
bytes_ = 46 * v * d
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
print(json.dumps({"probe": "adam_step", "params": v * d, "ms": ms, "GB/s": bytes_ / ms / 1e6,
                  "hbm_peak_GB/s": peak, "frac": bytes_ / ms / 1e6 / peak,
                  "bytes_per_param": 46, "note": "f32 grad, f64 moments, fused bf16 shadow"}))
