"""Timing probe for the full-catalog evaluation kernels (lf_eval_rank_topk):
CUDA-event timing at a given shape (default cfg2: n=51200, d=64, v=1M, bf16,
k=10), plus the kernel-only time from the library's launch profiler.  Prints
one JSON line.  Roofline: 2 n v d flops on the tensor pipe (the scores),
measured bf16 peak from MEASURED_PEAKS.json."""
import argparse
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_09682_b200 import _capi, metrics  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=51200)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--v", type=int, default=1000000)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()

dt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[a.dtype]
g = torch.Generator(device="cuda").manual_seed(0)
X = (torch.rand(a.n, a.d, device="cuda", generator=g) * 2 - 1).to(dt)
E = (torch.rand(a.v, a.d, device="cuda", generator=g) * 2 - 1).to(dt)
x = torch.randint(0, a.v, (a.n,), device="cuda", generator=g)

fn = lambda: metrics.rank_topk(X, E, x, a.k)  # noqa: E731
fn()
torch.cuda.synchronize()
L = _capi.lib()
L.lf_profile_reset()
L.lf_profile_enable(1)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.iters):
    fn()
e.record()
torch.cuda.synchronize()
L.lf_profile_enable(0)
ms = s.elapsed_time(e) / a.iters
cnt, tot = C.c_uint64(), C.c_double()
L.lf_profile_read(7, C.byref(cnt), C.byref(tot))
k_ms = tot.value / a.iters  # the seeding launch and the main launch
flops = 2.0 * a.n * a.v * a.d
peak = None
try:
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
except OSError:
    pass
print(json.dumps({"probe": "eval_rank_topk", "n": a.n, "d": a.d, "v": a.v, "k": a.k, "dtype": a.dtype,
                  "ms_per_call": ms, "kernel_ms": k_ms, "launches_per_call": cnt.value / a.iters,
                  "seed_chunks": os.environ.get("LSEFORGE_EVAL_SEED_CHUNKS", "default"), "rows_per_s": a.n / ms * 1e3,
                  "tflops_kernel": flops / k_ms * 1e-9, "peaks": peak}))
