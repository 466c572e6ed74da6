"""CE (materialising, cuBLAS) vs CCE (fused, this library) on one B200:
fwd+bwd time and peak device memory, the comparison behind the paper's
memory / speed claims.  bf16, no filtering.

    python tools/ce_vs_cce.py  -> one JSON line per shape
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_09682_b200 as lf  # noqa: E402
from paper_2509_09682_b200 import _capi  # noqa: E402


def peak_gb(fn):
    L = _capi.lib()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    L.lf_workspace_reset_peak()
    base_t = torch.cuda.memory_allocated()
    fn()
    torch.cuda.synchronize()
    cur, pk = C.c_uint64(), C.c_uint64()
    L.lf_workspace_stats(C.byref(cur), C.byref(pk))
    return (torch.cuda.max_memory_allocated() - base_t + pk.value) / 1e9


def timed(fn, iters=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


for n, d, v in [(51200, 64, 100_000), (51200, 64, 200_000), (51200, 64, 400_000), (8192, 64, 1_000_000)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    X = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    E = (torch.rand(v, d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    x = torch.randint(0, v, (n,), device="cuda", generator=g)

    def ce():
        lf.ce_full_forward(X, E, x, validate=False)
        lf.ce_full_backward(X, E, x, 1.0, validate=False)

    def cce():
        o = lf.cce_forward(X, E, x, validate=False)
        lf.cce_backward(X, E, x, o.lse, 1.0, validate=False, stats=False)

    row = {"n": n, "d": d, "v": v, "logits_gb_fp32": n * v * 4 / 1e9,
           "ce_ms": timed(ce), "cce_ms": timed(cce), "ce_peak_gb": peak_gb(ce),
           "cce_peak_gb": peak_gb(cce)}
    row["speedup"] = row["ce_ms"] / row["cce_ms"]
    row["memory_reduction"] = 1 - row["cce_peak_gb"] / row["ce_peak_gb"]
    print(json.dumps(row), flush=True)

# the sampled pair: materialising CE- (losses.cpp:142-221) vs fused CCE- at cfg3
for n, d, v, K in [(51200, 64, 1_000_000, 512), (51200, 64, 1_000_000, 2048)]:
    g = torch.Generator(device="cuda").manual_seed(2)
    X = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    E = (torch.rand(v, d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    I = torch.randint(0, v, (n, 1 + K), device="cuda", generator=g)

    def cem():
        lf.ce_sampled_forward(X, E, I)
        lf.ce_sampled_backward(X, E, I, 1.0)

    def ccem():
        o = lf.ccem_forward(X, E, I, validate=False)
        lf.ccem_backward(X, E, I, o.lse, 1.0, validate=False)

    row = {"sampled": True, "n": n, "d": d, "v": v, "K": K, "logits_gb_fp32": n * (1 + K) * 4 / 1e9,
           "cem_ms": timed(cem), "ccem_ms": timed(ccem), "cem_peak_gb": peak_gb(cem),
           "ccem_peak_gb": peak_gb(ccem)}
    row["speedup"] = row["cem_ms"] / row["ccem_ms"]
    row["memory_reduction"] = 1 - row["ccem_peak_gb"] / row["cem_peak_gb"]
    print(json.dumps(row), flush=True)
