#!/usr/bin/env python
"""bench.py — CCE fwd+bwd positions/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "cfg2"): SASRec-shaped CCE, bf16,
N = 51200 positions (batch 256 x seq 200), D = 64, V = 1,000,000 items,
saturated-gradient filtering ON (eps = kFp16MinPositive = 6e-8,
cce.hpp:15-30).  One step = cce_forward + cce_backward (loss, lse, pos, dX,
dE) over the whole batch.  For N > 1 the catalog is sharded over the ranks
(one process per GPU, NCCL): every rank owns V/N items, partial (m, s, t)
triples are all-gathered and dX is all-reduced (paper_2509_09682_b200/
sharded.py); total work is fixed, so scaling is "strong".

Timing: W untimed warm-up steps, then exactly K steps bracketed by a barrier
and torch.cuda.synchronize(); each step is timed with CUDA events on the
compute stream and an L2 flush (256 MB write) runs before every step outside
the events; the max over ranks is reported.  `e2e` times the same step
through the public API with the step's inputs copied from pinned host memory
and the loss read back, every step.

`--impl reference` times the reference's own CPU implementation (the
unmodified lseforge sources compiled in place into oracle/_ref) on the host
cores, on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CCE fwd+bwd positions/sec @V=1M,D=64 (1/2/4/8 GPU); % roofline; peak HBM GB"
N_ROWS, D, V = 51200, 64, 1_000_000
EPS = 6e-8  # CceConfig::Fp16SaturationPreset (cce.hpp:26-30)
SEED = 0xB2000002
WORKLOAD = ("cfg2: SASRec-shaped CCE bf16, N=51200 (batch 256 x seq 200), D=64, V=1M items, "
            "saturated-gradient filtering on (eps=6e-8)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", choices=["collective", "peer"], default="collective",
                    help="N>1: torch.distributed collectives (NCCL) or the peer-memory exchange "
                         "fused into the producing kernels (CUDA IPC)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return dict(hbm=float(j["hbm_gbs"]), tc=float(j["bf16_tflops"]),
                    tc_sustained=float(j.get("bf16_tflops_sustained", j["bf16_tflops"])),
                    source="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, tc=1590.0, tc_sustained=1400.0, source="fallback (B200_PROFILING.md)")


def mufu_peak():
    """Measured MUFU ex2 rate (profiles/*microbench_pipes.jsonl), exps/s."""
    import glob
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*microbench_pipes.jsonl")), reverse=True):
        for line in open(f):
            j = json.loads(line)
            if j["op"] == "ex2.approx.ftz.f32":
                return float(j["elems_per_s"]), os.path.relpath(f, ROOT)
    return 148 * 16 * 1.965e9, "assumed 16/clk/SM x 148 x 1.965 GHz"


def traffic_table():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        return json.load(open(p))
    return {}


# --------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md "clocks DURING the timed region")
# --------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:6], float(parts[6])))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return None
        load = [r for r in rows if r[3] > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(load)}


# --------------------------------------------------------------------------
# reference CPU timing (oracle/_ref = the unmodified reference sources)
# --------------------------------------------------------------------------
def reference_sample(rows_per_thread=16, steps=1, warmup=0, seed=SEED):
    import numpy as np
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_bind as ob
    threads = os.cpu_count() or 1
    rows = rows_per_thread * threads
    g = np.random.default_rng(seed)
    E = torch.from_numpy(g.uniform(-1, 1, (rows, D)).astype(np.float32)).to(torch.bfloat16).float().numpy()
    Cm = torch.from_numpy(g.uniform(-1, 1, (D, V)).astype(np.float32)).to(torch.bfloat16).float().numpy()
    t = g.integers(0, V, rows).astype(np.int64)
    times = []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        _, _, lse = ob.ref_cce_forward(E, Cm, t, rb=rows_per_thread, cb=256, workers=threads)
        ob.ref_cce_backward(E, Cm, t, lse, 1.0, EPS, rb=rows_per_thread, cb=256, workers=threads)
        if s >= warmup:
            times.append(time.perf_counter() - t0)
    per_step = sum(times) / len(times)
    sample = (f"reference lseforge cce_forward+cce_backward (oracle/_ref, -O3), {rows} rows x "
              f"V={V} x D={D}, eps={EPS}, row_block={rows_per_thread}, col_block=256, "
              f"workers={threads}, bf16-rounded fp32 inputs, {len(times)} step(s)")
    return rows / per_step, threads, sample, per_step


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    value, cores, sample, per_step = reference_sample(steps=args.steps, warmup=args.warmup)
    line = {"metric": METRIC, "value": value, "unit": "positions/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD, "sample_rows": int(round(value * per_step))},
            "cpu_baseline": {"value": value, "unit": "positions/s", "cores": cores,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "positions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# B200 arm
# --------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # LF_BENCH_SHARE_GPU=1 (test only): every rank uses cuda:0 and the gloo
    # backend, so the multi-rank code path can be exercised on one GPU.
    share = os.environ.get("LF_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    else:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        dist.init_process_group("gloo", rank=0, world_size=1)

    import paper_2509_09682_b200 as lf
    from paper_2509_09682_b200 import _capi
    from paper_2509_09682_b200.sharded import ShardedCce

    L = _capi.lib()
    sh = ShardedCce(V, exchange=args.exchange if world > 1 else "collective")
    v0, v1 = sh.v_begin, sh.v_end
    g = torch.Generator(device=dev).manual_seed(SEED)
    X = (torch.rand(N_ROWS, D, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    E_full = (torch.rand(V, D, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    E = E_full[v0:v1].contiguous()
    del E_full
    x = torch.randint(0, V, (N_ROWS,), device=dev, generator=g)
    cfg = lf.CceConfig(filter_eps=EPS)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(Xs, Es, xs):
        out = sh.forward(Xs, Es, xs, cfg)
        res = sh.backward(Xs, Es, xs, out.lse, 1.0, cfg, stats=False)
        return out, res

    _capi.check(L.lf_validate_targets(x.data_ptr(), N_ROWS, V, stream.cuda_stream))
    for _ in range(args.warmup):
        step(X, E, x)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    L.lf_workspace_reset_peak()

    # ---- timed region (device-resident inputs) ----
    L.lf_profile_reset()
    L.lf_profile_enable(1)
    launches0 = L.lf_launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    clocks = Clocks(local)
    dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(k & 0xFF)  # L2 flush, outside the events
        evs[k][0].record(stream)
        out, res = step(X, E, x)
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    launches = L.lf_launch_count() - launches0
    L.lf_profile_enable(0)
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    kern = {}
    for kind, name in enumerate(_capi.KERNEL_KINDS):
        cnt, ms = C.c_uint64(), C.c_double()
        L.lf_profile_read(kind, C.byref(cnt), C.byref(ms))
        if cnt.value:
            kern[name] = {"launches": int(cnt.value), "ms_total": ms.value,
                          "ms_per_launch": ms.value / cnt.value}
    t_max = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    total_ms = float(t_max)
    ms_step = total_ms / args.steps
    value = N_ROWS / (ms_step / 1e3)
    cur, wpk = C.c_uint64(), C.c_uint64()
    L.lf_workspace_stats(C.byref(cur), C.byref(wpk))
    peak_hbm = (torch.cuda.max_memory_allocated(dev) + wpk.value) / 1e9
    loss_val = float(out.loss)

    # ---- roofline of the dominant kernel (algorithmic work, live durations) ----
    peaks = load_peaks()
    mufu, mufu_src = mufu_peak()
    vs = v1 - v0
    Lsh = N_ROWS * vs
    alg = {"cce_fwd": 2 * Lsh * D,       # forward contraction (estimate_flops: N*D*V MACs)
           "cce_bwd_dx": 3 * Lsh * D,    # half of the backward's 6*L*D (3x forward MACs)
           "cce_bwd_de": 3 * Lsh * D}
    exps = {"cce_fwd": Lsh, "cce_bwd_dx": Lsh, "cce_bwd_de": Lsh}
    dom = max((k for k in kern if k in alg), key=lambda k: kern[k]["ms_total"], default=None)
    roof = None
    roof_exp = None
    if dom:
        dur = kern[dom]["ms_per_launch"] / 1e3
        ach = alg[dom] / dur / 1e12
        tr = traffic_table().get(dom)
        roof = {"kernel": dom, "bound": "tensor", "achieved": ach,
                "peak": peaks["tc_sustained"], "unit": "TFLOP/s",
                "frac": ach / peaks["tc_sustained"],
                "traffic": tr.get("dram_bytes_per_launch") if tr else None,
                "peak_source": peaks["source"] + ", bf16 sustained (kernel timed inside a long step)",
                "algorithmic_flops_per_launch": alg[dom], "ms_per_launch": dur * 1e3}
        roof_exp = {"kernel": dom, "achieved": exps[dom] / dur / 1e12, "peak": mufu / 1e12,
                    "unit": "Texp/s", "frac": exps[dom] / dur / mufu, "peak_source": mufu_src}
    # whole-step roofline (north star): T_roof = max(8LD/P_tc, 2L/P_exp) per GPU
    L_all = N_ROWS * V / world
    t_roof = max(8 * L_all * D / (peaks["tc_sustained"] * 1e12), 2 * L_all / mufu)
    step_roof = {"t_roof_ms": t_roof * 1e3, "ms_per_step": ms_step, "frac": t_roof * 1e3 / ms_step,
                 "binding": "exp (MUFU)" if 2 * L_all / mufu > 8 * L_all * D / (peaks["tc_sustained"] * 1e12) else "tensor",
                 "note": "algorithmic work 8*L*D flops and 2*L exps, L = N*V/P"}

    # ---- e2e through the public API with host buffers ----
    # Every step copies ITS inputs (X, the local E slice, targets) from pinned
    # host memory and reads its loss back on the host.  The copy of step k+1
    # runs on a side stream into the other half of a double buffer while step
    # k computes (the host->device link and the SMs work concurrently).
    e2e = None
    if not args.no_e2e:
        Xh = X.cpu().pin_memory()
        Eh = E.cpu().pin_memory()
        xh = x.cpu().pin_memory()
        loss_h = torch.empty((), dtype=torch.float64).pin_memory()
        bufs = [(torch.empty_like(X), torch.empty_like(E), torch.empty_like(x)) for _ in range(2)]
        cs = torch.cuda.Stream(dev)
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]

        def issue_copy(k):
            b = k % 2
            with torch.cuda.stream(cs):
                cs.wait_event(consumed[b])
                bufs[b][0].copy_(Xh, non_blocking=True)
                bufs[b][1].copy_(Eh, non_blocking=True)
                bufs[b][2].copy_(xh, non_blocking=True)
                copied[b].record(cs)

        def e2e_run(nsteps):
            for b in range(2):
                consumed[b].record(stream)
            issue_copy(0)
            for k in range(nsteps):
                b = k % 2
                stream.wait_event(copied[b])
                o, _ = step(*bufs[b])
                consumed[b].record(stream)
                if k + 1 < nsteps:
                    issue_copy(k + 1)
                loss_h.copy_(o.loss, non_blocking=True)
                stream.synchronize()  # the host reads the loss every step
                _ = float(loss_h)

        e2e_run(max(1, args.warmup))
        torch.cuda.synchronize()
        dist.barrier()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        e2e_run(args.steps)
        eb.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([ea.elapsed_time(eb) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        h2d = Xh.numel() * Xh.element_size() + Eh.numel() * Eh.element_size() + xh.numel() * 8
        e2e = {"value": N_ROWS / (float(e_ms) / 1e3), "unit": "positions/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 8,
               "ms_per_step": float(e_ms), "api": "ShardedCce.forward/backward (lf_cce_* C-ABI)",
               "overlap": "step k+1's host->device copy overlaps step k's compute (double buffer)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cv, cores, sample, _ = reference_sample(rows_per_thread=16, steps=1, warmup=0)
        cpu = {"value": cv, "unit": "positions/s", "cores": cores, "kind": "reference",
               "sample": sample}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "positions/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic",
                "config": {"workload": WORKLOAD, "n_positions": N_ROWS, "d": D, "v": V,
                           "filter_eps": EPS, "seed": SEED,
                           "parallelism": (f"catalog-sharded over {world} GPU(s), {args.exchange} exchange"
                                           if world > 1 else "single GPU"),
                           "l2": "inputs (134.6 MB) exceed L2 (126 MB) and a 256 MB L2 flush runs "
                                 "before every timed step (outside the events)"},
                "peak_hbm_gb": peak_hbm, "loss": loss_val,
                "roofline": roof, "roofline_exp": roof_exp, "step_roofline": step_roof,
                "kernels": kern, "gpu_launches": int(launches), "e2e": e2e,
                "cpu_baseline": cpu, "clocks": clk}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
