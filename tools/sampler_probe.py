"""Timing probe for the device negative samplers at the cfg3 shape (N = 51 200
rows, K = 512 negatives, V = 1M): uniform and popularity (Zipf-like counts),
CUDA events, one JSON line each."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_09682_b200 as lf  # noqa: E402

n, K, V = 51200, 512, 1_000_000
g = torch.Generator(device="cpu").manual_seed(0)
pos = torch.randint(0, V, (n,), generator=g).cuda()
counts = (1e6 / torch.arange(1, V + 1, dtype=torch.float64) ** 1.1).to(torch.int64) + 1


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


cu = counts.cuda()
for name, fn in (("sample_uniform", lambda: lf.sample_uniform(pos, K, V, 7)),
                 ("sample_popularity", lambda: lf.sample_popularity(pos, K, cu, 7))):
    ms = timed(fn)
    print(json.dumps({"probe": name, "n": n, "K": K, "v": V, "ms": ms, "draws_per_s": n * K / ms * 1e3,
                      "note": "includes the validation sync (and the cumulative weights for popularity)"}))
