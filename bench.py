#!/usr/bin/env python
"""bench.py — CCE fwd+bwd positions/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "cfg2"): SASRec-shaped CCE, bf16,
N = 51200 positions (batch 256 x seq 200), D = 64, V = 1,000,000 items,
saturated-gradient filtering ON (eps = kFp16MinPositive = 6e-8,
cce.hpp:15-30).  Inputs are the reference's own instance: SplitMix64
make_instance (support.hpp:27-37, seed 0xB2000002; synth.py restates it bit
for bit), rounded to bf16.  One step = cce_forward + cce_backward (loss,
lse, pos, dX, dE) over the whole batch through lf_cce_forward_backward (the
fused forward + dX kernel, then the dE pass).  For N > 1 the catalog is
sharded over the ranks (one process per GPU, NCCL): every rank owns V/N
items, the (m, s, t) triples are all-gathered and dX is all-reduced
(ShardedCce.forward_backward); total work is fixed, so scaling is "strong".

Timing: W untimed warm-up steps, then exactly K steps bracketed by a barrier
and torch.cuda.synchronize(); each step is timed with CUDA events on the
compute stream, a 256 MB L2 flush runs before every step outside the events,
the max over ranks is reported.  `e2e` times the same step through the public
API with the step's inputs copied from pinned host memory and the loss read
back, every step (`e2e_grads` also reads dX and dE back).

The same line carries, at N = 1: `parity` (the reference run on the first
256 rows of the timed inputs vs the GPU), `cfg3` (CCE- K = 512, BASELINE
configs[2], with its own roofline, CPU baseline and full-N parity), and
`filter` (the saturated-gradient filtering protocol of SURVEY.md 8(d)).

`--impl reference` times the reference's own CPU implementation (the
unmodified lseforge sources compiled in place into oracle/_ref) on the host
cores, on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
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
SEED = 0xB2000002   # cfg2 (0xB2000000 + cfg#)
SEED3 = 0xB2000003  # cfg3
SEED1 = 0xB2000001  # cfg1
N1, V1 = 2048, 32768  # cfg1: fp32, batch 32 x seq 64, filtering off
K_NEG = 512
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
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the cfg3, filter and sharded-config sub-records")
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


def bf16_round(a):
    """Host copy of what the device sees: round-to-nearest-even to bf16, as float32."""
    import numpy as np
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).float().numpy()


# --------------------------------------------------------------------------
# reference CPU runs (oracle/_ref = the unmodified reference sources; the
# cpu_baseline leg and the checker of the GPU results — never the product)
# --------------------------------------------------------------------------
def reference_cfg2_sample(Xh, Ch, t, rows_per_thread=16):
    """cce_forward + cce_backward of the reference on the first rows of the
    instance (bf16-rounded float, full V and D), all host threads."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_bind as ob
    threads = os.cpu_count() or 1
    rows = rows_per_thread * threads
    E = Xh[:rows]
    ts = t[:rows]
    t0 = time.perf_counter()
    loss, pos, lse = ob.ref_cce_forward(E, Ch, ts, rb=rows_per_thread, cb=256, workers=threads)
    dE, dC, frac = ob.ref_cce_backward(E, Ch, ts, lse, 1.0, EPS, rb=rows_per_thread, cb=256,
                                       workers=threads)
    sec = time.perf_counter() - t0
    sample = (f"reference lseforge cce_forward+cce_backward (oracle/_ref, -O3), first {rows} rows of "
              f"the cfg2 instance (make_instance seed {SEED:#x}, bf16-rounded) x V={V} x D={D}, "
              f"eps={EPS}, row_block={rows_per_thread}, col_block=256, workers={threads}")
    return dict(rows=rows, threads=threads, sec=sec, sample=sample, loss=loss, pos=pos, lse=lse,
                dE=dE, dC=dC, frac=frac)


def cfg2_host_instance():
    from paper_2509_09682_b200 import synth
    Xr, Cr, t = synth.make_instance(SEED, N_ROWS, D, V)
    return bf16_round(Xr), bf16_round(Cr), t


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    Xh, Ch, t = cfg2_host_instance()
    secs = []
    last = None
    for s in range(args.warmup + args.steps):
        last = reference_cfg2_sample(Xh, Ch, t)
        if s >= args.warmup:
            secs.append(last["sec"])
    per_step = sum(secs) / len(secs)
    value = last["rows"] / per_step
    line = {"metric": METRIC, "value": value, "unit": "positions/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference make_instance)", "impl": "reference",
            "config": {"workload": WORKLOAD, "sample_rows": last["rows"], "seed": SEED},
            "cpu_baseline": {"value": value, "unit": "positions/s", "cores": last["threads"],
                             "kind": "reference", "sample": last["sample"]},
            "e2e": {"value": value, "unit": "positions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# B200 arm
# --------------------------------------------------------------------------
def rel(a, b):
    import numpy as np
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.maximum(1.0, np.abs(np.asarray(b)))))


def normwise(got, want):
    import numpy as np
    g = np.asarray(got, np.float64)
    w = np.asarray(want, np.float64)
    return float(np.linalg.norm(g - w) / max(np.linalg.norm(w), 1e-300))


def timed_steps(step, steps, warmup, stream, flush, kernels=None):
    """Device-timed loop (CUDA events on the compute stream, L2 flush outside).
    kernels: a dict to fill with the library's per-kernel ms per step
    (lf_profile_*), or None."""
    import torch
    from paper_2509_09682_b200 import _capi
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    L = _capi.lib()
    if kernels is not None:
        L.lf_profile_reset()
        L.lf_profile_enable(1)
    for k in range(steps):
        flush.fill_(k & 0xFF)
        evs[k][0].record(stream)
        step()
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    if kernels is not None:
        L.lf_profile_enable(0)
        for kind, name in enumerate(_capi.KERNEL_KINDS):
            cnt, ms = C.c_uint64(), C.c_double()
            L.lf_profile_read(kind, C.byref(cnt), C.byref(ms))
            if cnt.value:
                kernels[name] = round(ms.value / steps, 4)
    return sum(a.elapsed_time(b) for a, b in evs) / steps


def run_ours(args):
    import numpy as np
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
    vs = v1 - v0
    stream = torch.cuda.current_stream(dev)

    # ---- the reference's instance (make_instance, SplitMix64), bf16 ----
    Xh, Ch, t = cfg2_host_instance()
    X = torch.from_numpy(Xh).to(dev).to(torch.bfloat16)  # exact: already bf16 values
    C_dev = torch.from_numpy(np.ascontiguousarray(Ch[:, v0:v1])).to(dev)
    E = torch.empty((vs, D), dtype=torch.bfloat16, device=dev)
    # ref-C (D x V float) -> E (V x D bf16): the drop-in boundary's own converter
    _capi.check(L.lf_classifier_to_items(C_dev.data_ptr(), D, vs, _capi.LF_BF16, E.data_ptr(),
                                         stream.cuda_stream))
    del C_dev
    x = torch.from_numpy(t).to(dev)
    cfg = lf.CceConfig(filter_eps=EPS)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    _capi.check(L.lf_validate_targets(x.data_ptr(), N_ROWS, V, stream.cuda_stream))

    res_box = [None]

    def step(Xs=X, Es=E, xs=x):
        res_box[0] = None  # the previous step's outputs are released first
        res_box[0] = sh.forward_backward(Xs, Es, xs, 1.0, cfg, stats=False)
        return res_box[0]

    for _ in range(args.warmup):
        step()
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
        step()
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
    out, res = res_box[0]
    loss_val = float(out.loss)

    # ---- memory: the library's own footprint vs the harness's ----
    cur, wpk = C.c_uint64(), C.c_uint64()
    L.lf_workspace_stats(C.byref(cur), C.byref(wpk))
    inputs_b = X.numel() * 2 + E.numel() * 2 + x.numel() * 8
    outputs_b = (3 * N_ROWS + 1) * 8 + N_ROWS * D * 4 + vs * D * 4
    memory = {"library_peak_gb": (inputs_b + outputs_b + wpk.value) / 1e9,
              "inputs_gb": inputs_b / 1e9, "outputs_gb": outputs_b / 1e9,
              "workspace_peak_gb": wpk.value / 1e9,
              "harness_peak_gb": (torch.cuda.max_memory_allocated(dev) + wpk.value) / 1e9,
              "note": "library_peak = inputs (X, E, targets) + outputs (lse, pos, loss, dX, dE) + the "
                      "library's scratch high-water (lf_workspace_stats); harness_peak adds the 256 MB L2 "
                      "flush buffer and whatever torch holds"}

    # ---- roofline: the binding unit is the exp (MUFU ex2) ----
    peaks = load_peaks()
    mufu, mufu_src = mufu_peak()
    Lsh = N_ROWS * vs
    exps = {"cce_fwd_dx": Lsh, "cce_bwd_de": Lsh, "cce_fwd": Lsh, "cce_bwd_dx": Lsh}
    flops = {"cce_fwd_dx": 4 * Lsh * D,  # forward N*D*V MACs + the dX GEMM's N*D*V MACs
             "cce_bwd_de": 4 * Lsh * D,  # the logit recompute + the dE GEMM
             "cce_fwd": 2 * Lsh * D, "cce_bwd_dx": 3 * Lsh * D}
    dom = max((k for k in kern if k in exps), key=lambda k: kern[k]["ms_total"], default=None)
    roof = roof_tc = None
    if dom:
        dur = kern[dom]["ms_per_launch"] / 1e3
        tr = traffic_table().get(dom)
        roof = {"kernel": dom, "bound": "exp (MUFU ex2)", "achieved": exps[dom] / dur / 1e12,
                "peak": mufu / 1e12, "unit": "Texp/s", "frac": exps[dom] / dur / mufu,
                "traffic": tr.get("dram_bytes_per_launch") if tr else None,
                "peak_source": mufu_src,
                "algorithmic_exps_per_launch": exps[dom], "ms_per_launch": dur * 1e3,
                "note": "one exp per logit per launch (N*V_shard logits), whether MUFU ex2 or the "
                        "packed FMA-pipe polynomial computes it (a share of each 32-column chunk); peak = "
                        "the MUFU rate alone; traffic = dram read+write per launch from ncu --set full "
                        "(profiles/traffic.json)"}
        ach = flops[dom] / dur / 1e12
        roof_tc = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": peaks["tc_sustained"],
                   "unit": "TFLOP/s", "frac": ach / peaks["tc_sustained"],
                   "peak_source": peaks["source"] + ", bf16 sustained",
                   "algorithmic_flops_per_launch": flops[dom]}
    L_all = N_ROWS * V / world
    t_exp = 2 * L_all / mufu
    t_tc = 8 * L_all * D / (peaks["tc_sustained"] * 1e12)
    t_roof = max(t_exp, t_tc)
    step_roof = {"t_roof_ms": t_roof * 1e3, "ms_per_step": ms_step, "frac": t_roof * 1e3 / ms_step,
                 "binding": "exp (MUFU)" if t_exp > t_tc else "tensor",
                 "executed_over_algorithmic": {"exps": 1.0, "flops": 1.0},
                 "note": "algorithmic work 8*L*D flops and 2*L exps, L = N*V/P; the fused path executes "
                         "exactly that (forward+dX kernel: 1 exp, 4LD flops; dE pass: 1 exp, 4LD flops)"}

    # ---- e2e through the public API with host buffers ----
    e2e = e2e_grads = None
    if not args.no_e2e:
        e2e = run_e2e(step, X, E, x, stream, args, world, dev, grads=False)
        e2e_grads = run_e2e(step, X, E, x, stream, args, world, dev, grads=True)

    extras = {}

    def sub_record(name, fn):
        # a sub-record that fails is reported in the line, never fatal to it
        try:
            extras[name] = fn()
        except Exception as e:  # noqa: BLE001
            extras[name] = {"error": f"{type(e).__name__}: {e}"[:400]}
            torch.cuda.synchronize()

    if rank == 0 and world == 1 and not args.no_e2e:
        sub_record("e2e_dropin", dropin_e2e)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sub_record("cfg2_parity", lambda: cfg2_parity(lf, sh, X, E, x, out, res, Xh, Ch, t, cfg))
        cp = extras.pop("cfg2_parity")
        if isinstance(cp, tuple):
            extras["cpu_baseline"], extras["parity"] = cp
        else:
            extras["cpu_baseline"] = extras["parity"] = cp
    if rank == 0 and world == 1 and not args.no_extras:
        del res_box[0], out, res
        sub_record("filter", lambda: filter_protocol(lf, X, E, x, Xh, Ch, t, flush, stream, args))
        sub_record("cfg1", lambda: cfg1_record(lf, flush, stream, args, not args.no_cpu_baseline))
        sub_record("cfg3", lambda: cfg3_record(lf, flush, stream, args, peaks, not args.no_cpu_baseline))
        sub_record("sharded_configs", lambda: shard_record(lf, flush, stream, args, peaks))

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "positions/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic (the reference's make_instance, SplitMix64)",
                "config": {"workload": WORKLOAD, "n_positions": N_ROWS, "d": D, "v": V,
                           "filter_eps": EPS, "seed": SEED,
                           "path": "lf_cce_forward_backward (fused forward+dX kernel, then the dE pass)",
                           "parallelism": (f"catalog-sharded over {world} GPU(s), {args.exchange} exchange"
                                           if world > 1 else "single GPU"),
                           "l2": "inputs (134.6 MB) exceed L2 (126 MB) and a 256 MB L2 flush runs "
                                 "before every timed step (outside the events)"},
                "peak_hbm_gb": memory["library_peak_gb"], "memory": memory, "loss": loss_val,
                "roofline": roof, "roofline_tensor": roof_tc, "step_roofline": step_roof,
                "kernels": kern, "gpu_launches": int(launches), "e2e": e2e, "e2e_grads": e2e_grads,
                "e2e_dropin": extras.get("e2e_dropin"),
                "cpu_baseline": extras.get("cpu_baseline"), "parity": extras.get("parity"),
                "filter": extras.get("filter"), "cfg1": extras.get("cfg1"), "cfg3": extras.get("cfg3"),
                "sharded_configs": extras.get("sharded_configs"), "clocks": clk}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def run_e2e(step, X, E, x, stream, args, world, dev, grads):
    """The step through the public API with host buffers: every step copies
    ITS inputs (X, the local E slice, targets) from pinned host memory and
    reads its loss (grads=True: also dX and dE) back on the host.  The copy of
    step k+1 runs on a side stream into the other half of a double buffer
    while step k computes; the host reads step k's loss once step k+1 is
    enqueued (as a training loop logs it), so the GPU never waits for the
    host; with grads, step k's dX / dE go back on a third stream while step
    k+1 computes."""
    import torch
    import torch.distributed as dist
    Xh = X.cpu().pin_memory()
    Eh = E.cpu().pin_memory()
    xh = x.cpu().pin_memory()
    loss_h = [torch.empty((), dtype=torch.float64).pin_memory() for _ in range(2)]
    loss_ev = [torch.cuda.Event() for _ in range(2)]
    dXh = torch.empty((X.shape[0], X.shape[1]), dtype=torch.float32).pin_memory() if grads else None
    dEh = torch.empty((E.shape[0], E.shape[1]), dtype=torch.float32).pin_memory() if grads else None
    bufs = [(torch.empty_like(X), torch.empty_like(E), torch.empty_like(x)) for _ in range(2)]
    cs = torch.cuda.Stream(dev)
    ds = torch.cuda.Stream(dev)
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    keep = [None, None]

    def issue_copy(k):
        b = k % 2
        with torch.cuda.stream(cs):
            cs.wait_event(consumed[b])
            bufs[b][0].copy_(Xh, non_blocking=True)
            bufs[b][1].copy_(Eh, non_blocking=True)
            bufs[b][2].copy_(xh, non_blocking=True)
            copied[b].record(cs)

    def run(nsteps):
        for b in range(2):
            consumed[b].record(stream)
        issue_copy(0)
        pending = None
        for k in range(nsteps):
            b = k % 2
            stream.wait_event(copied[b])
            o, r = step(*bufs[b])
            consumed[b].record(stream)
            if k + 1 < nsteps:
                issue_copy(k + 1)
            loss_h[b].copy_(o.loss, non_blocking=True)
            loss_ev[b].record(stream)
            if grads:
                done = torch.cuda.Event()
                done.record(stream)
                if pending is not None:
                    ds.synchronize()  # the previous step's gradients have landed on the host
                with torch.cuda.stream(ds):
                    ds.wait_event(done)
                    dXh.copy_(r.grads.d_embeddings, non_blocking=True)
                    dEh.copy_(r.grads.d_classifier, non_blocking=True)
                keep[b] = r  # hold the device gradients until their copy is done
                pending = k
            if k > 0:  # the host reads the previous step's loss while this one runs
                loss_ev[1 - b].synchronize()
                _ = float(loss_h[1 - b])
        loss_ev[(nsteps - 1) % 2].synchronize()
        _ = float(loss_h[(nsteps - 1) % 2])
        if grads:
            ds.synchronize()

    run(max(1, args.warmup))
    torch.cuda.synchronize()
    dist.barrier()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    run(args.steps)
    eb.record(stream)
    torch.cuda.synchronize()
    e_ms = torch.tensor([ea.elapsed_time(eb) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    h2d = Xh.numel() * Xh.element_size() + Eh.numel() * Eh.element_size() + xh.numel() * 8
    d2h = 8 + ((dXh.numel() + dEh.numel()) * 4 if grads else 0)
    return {"value": N_ROWS / (float(e_ms) / 1e3), "unit": "positions/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": float(e_ms),
            "api": "ShardedCce.forward_backward -> lf_cce_forward_backward (C-ABI)",
            "overlap": "step k+1's host->device copy overlaps step k's compute (double buffer); the "
                       "host reads step k's loss while step k+1 runs"
                       + ("; step k's dX/dE device->host copy overlaps step k+1" if grads else "")}


def dropin_e2e():
    """cfg2 through the C++ drop-in exactly as a reference caller runs it:
    lseforge::cce_forward + cce_backward with host DenseMatrix inputs and
    host LossOutput / GradPair (double, d x v d_classifier) results
    (paper_2509_09682_b200/shim/build/dropin_check, wall clock, median of 3).
    Reported with the API's own floor — value-initialising the 512 MB d x v
    double the signature returns — and with LSEFORGE_B200_HOST_HEAP=keep."""
    exe = os.path.join(ROOT, "paper_2509_09682_b200", "shim", "build", "dropin_check")
    if not os.path.exists(exe):
        return None
    out = {}
    for tag, extra in (("default", {}), ("host_heap_keep", {"LSEFORGE_B200_HOST_HEAP": "keep"})):
        env = dict(os.environ, LSEFORGE_B200_DTYPE="bf16", **extra)
        try:
            p = subprocess.run([exe, "bench", "3"], capture_output=True, text=True, timeout=600, env=env)
            out[tag] = json.loads(p.stdout.strip().splitlines()[-1])
        except Exception as e:  # reported, not fatal: the device-side bench stands on its own
            out[tag] = {"error": repr(e)[:200]}
    out["api"] = ("lseforge::cce_forward + cce_backward (the reference signatures) through "
                  "shim/lseforge_shim.cpp + liblseforge_b200.so, LSEFORGE_B200_DTYPE=bf16")
    return out


def cfg2_parity(lf, sh, X, E, x, out, res, Xh, Ch, t, cfg):
    """The reference (oracle/_ref) on the first rows of the SAME inputs the
    bench timed, and the GPU on the same rows: the full-N run's per-row lse /
    pos / dX (dX_i scales as 1/N) and a GPU run on the sample alone for the
    loss, dE (the sample's contribution) and the skip fraction."""
    import numpy as np
    import torch
    r = reference_cfg2_sample(Xh, Ch, t)
    ns = r["rows"]
    cpu = {"value": ns / r["sec"], "unit": "positions/s", "cores": r["threads"], "kind": "reference",
           "sample": r["sample"]}
    lse_g = out.lse[:ns].cpu().numpy()
    pos_g = out.pos_logits[:ns].cpu().numpy()
    dX_g = res.grads.d_embeddings[:ns].double().cpu().numpy() * N_ROWS
    so, sr = lf.cce_forward_backward(X[:ns].contiguous(), E, x[:ns].contiguous(), 1.0, cfg,
                                     stats=True)
    dE_g = sr.grads.d_classifier.double().cpu().numpy()
    tol = {"loss_rel": 1e-2, "lse_max_rel": 1e-3, "pos_max_rel": 1e-3, "dX_normwise": 1e-2,
           "dE_normwise": 1e-2, "skipped_fraction_abs": 2e-3}
    p = {"rows": ns, "inputs": "the timed cfg2 instance (first rows), reference fed the same bf16 values",
         "loss_rel": abs(float(so.loss) - r["loss"]) / max(1.0, abs(r["loss"])),
         "lse_max_rel": rel(lse_g, r["lse"]), "pos_max_rel": rel(pos_g, r["pos"]),
         "dX_normwise": normwise(dX_g, r["dE"] * ns),
         "dE_normwise": normwise(dE_g, r["dC"].T),
         "skipped_fraction": sr.skipped_fraction, "skipped_fraction_ref": r["frac"],
         "tolerance": tol}
    p["pass"] = bool(p["loss_rel"] < tol["loss_rel"] and p["lse_max_rel"] < tol["lse_max_rel"]
                     and p["pos_max_rel"] < tol["pos_max_rel"] and p["dX_normwise"] < tol["dX_normwise"]
                     and p["dE_normwise"] < tol["dE_normwise"]
                     and abs(p["skipped_fraction"] - p["skipped_fraction_ref"]) <= tol["skipped_fraction_abs"])
    p["note"] = ("dX from the fused kernel is the unfiltered gradient (each entry the eps filter drops "
                 "is < eps); dE and the skip fraction follow the filter exactly")
    del so, sr
    torch.cuda.synchronize()
    return cpu, p


def filter_protocol(lf, X, E, x, Xh, Ch, t, flush, stream, args):
    """SURVEY.md 8(d) "Recommended protocol": the headline data (distribution
    A, uniform) at the reference preset, and distribution B, X_i = U(-1,1)^D
    + gamma E_(x_i), for gamma in {1, 2} and eps in {6e-8, 1e-6, 2^-12,
    2^-8}: per-element skipped_fraction (reference definition,
    cce.cpp:264-268), skipped / total 32 x 32 sub-tiles at the kernel's skip
    granularity, and positions/s of the production step (stats off)."""
    import numpy as np
    import torch
    rows = []
    steps = max(3, min(args.steps, 5))

    def measure(Xd, dist_name, gamma, eps):
        cfg = lf.CceConfig(filter_eps=eps)
        fb = lambda: lf.cce_forward_backward(Xd, E, x, 1.0, cfg, validate=False)
        kern = {}
        ms = timed_steps(fb, steps, 1, stream, flush, kern)
        o, r = lf.cce_forward_backward(Xd, E, x, 1.0, cfg, validate=False, stats=True)
        fused = bool(lf._capi.lib().lf_cce_fused_supported(C.byref(cfg.to_c(lf._capi.LF_BF16)), D))
        rows.append({"dist": dist_name, "gamma": gamma, "eps": eps, "loss": float(o.loss),
                     "skipped_fraction": r.skipped_fraction, "skipped_subtiles": r.skipped_tiles,
                     "total_subtiles": r.total_tiles,
                     "subtile_skip_frac": (r.skipped_tiles / r.total_tiles) if r.total_tiles else 0.0,
                     "ms_per_step": ms, "kernel_ms_per_step": kern,
                     "positions_per_s": N_ROWS / (ms / 1e3),
                     "path": "fused forward+dX, filtered dE pass" if fused
                             else "3 passes (forward, filtered dX pass with sub-tile skipping, filtered dE pass)"})
        del o, r

    measure(X, "A (uniform, headline)", 0.0, EPS)
    tgt_rows = np.ascontiguousarray(Ch[:, t].T)  # E_(x_i), already bf16 values
    Xr = Xh.astype(np.float32)
    for gamma in (1.0, 2.0):
        XB = torch.from_numpy(Xr + gamma * tgt_rows).to(X.device).to(torch.bfloat16)
        for eps in (6e-8, 1e-6, 2.0 ** -12, 2.0 ** -8):
            measure(XB, "B (trained-like)", gamma, eps)
        del XB
    torch.cuda.synchronize()
    return {"runs": rows, "steps_per_run": steps,
            "skip_granularity": "32 rows x 32 items (dE pass in the fused path; dX pass in the 3-pass path)",
            "note": "distribution B at coarse eps (>= 2^-12) runs the 3-pass path whose dX pass skips "
                    "sub-tiles below eps; positions/s is the production step (stats off)"}


def cfg3_record(lf, flush, stream, args, peaks, cpu):
    """BASELINE configs[2]: CCE- bf16, N = 51200, D = 64, V = 1M, K = 512
    uniform negatives from the reference's sample_uniform stream (the GPU
    sampler, index-for-index the reference's), fwd + bwd (deterministic dE)."""
    import numpy as np
    import torch
    from paper_2509_09682_b200 import synth
    dev = torch.device("cuda", torch.cuda.current_device())
    Xr, Cr, t3 = synth.make_instance(SEED3, N_ROWS, D, V)
    Xh, Ch = bf16_round(Xr), bf16_round(Cr)
    del Xr, Cr
    X3 = torch.from_numpy(Xh).to(dev).to(torch.bfloat16)
    E3 = torch.from_numpy(np.ascontiguousarray(Ch.T)).to(dev).to(torch.bfloat16)
    x3 = torch.from_numpy(t3).to(dev)
    sseed = synth.derived_seed(SEED3, 7)
    inds = lf.sample_uniform(x3, K_NEG, V, sseed)
    cfg = lf.CceConfig()
    box = [None]

    def step_unfused():
        box[0] = None
        o = lf.ccem_forward(X3, E3, inds, cfg, validate=False)
        g = lf.ccem_backward(X3, E3, inds, o.lse, 1.0, cfg, validate=False)
        box[0] = (o, g)

    def step():
        box[0] = None
        box[0] = lf.ccem_forward_backward(X3, E3, inds, 1.0, cfg, validate=False)

    kern_u = {}
    ms_u = timed_steps(step_unfused, args.steps, max(3, args.warmup), stream, flush, kern_u)
    kern = {}
    ms = timed_steps(step, args.steps, max(3, args.warmup), stream, flush, kern)
    S = N_ROWS * (1 + K_NEG)
    alg_bytes = 2 * S * (2 * D + 8) + S * 4 * D + V * D * 4 + N_ROWS * (6 * D + 16)
    ach = alg_bytes / (ms / 1e3) / 1e9
    rec = {"workload": "cfg3: CCE- bf16, N=51200, D=64, V=1M, K=512 uniform negatives "
                       f"(make_instance seed {SEED3:#x}, sample_uniform SplitMix64(seed).derived(7))",
           "value": N_ROWS / (ms / 1e3), "unit": "positions/s", "ms_per_step": ms, "steps": args.steps,
           "path": "lf_ccem_forward_backward (one gather pass: lse, pos, dX, logits; then the ordered dE)",
           "kernel_ms_per_step": kern,
           "unfused": {"path": "lf_ccem_forward + lf_ccem_backward", "ms_per_step": ms_u,
                       "value": N_ROWS / (ms_u / 1e3), "kernel_ms_per_step": kern_u},
           "roofline": {"bound": "hbm", "achieved": ach, "peak": peaks["hbm"], "unit": "GB/s",
                        "frac": ach / peaks["hbm"], "traffic": None,
                        "algorithmic_bytes_per_step": alg_bytes,
                        "note": "SURVEY.md 8(d): 2 S (2D+8) gathers + index reads (fwd, bwd) + S 4D dE "
                                "contributions + V D 4 dE write + N (6D+16), S = N (1+K); whole step. "
                                "The fused path gathers the candidates' rows once, so it can exceed this "
                                "two-pass algorithmic count's bound"},
           "bar_pos_per_s": 11.8e6}
    o, g = box[0]
    if cpu:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle_bind as ob
        threads = os.cpu_count() or 1
        ih = inds.cpu().numpy()
        t0 = time.perf_counter()
        loss, pos, lse = ob.ref_ccem_forward(Xh, Ch, ih, rb=128, workers=threads)
        rdE, rdC = ob.ref_ccem_backward_rows(Xh, Ch, ih, lse, np.full(N_ROWS, 1.0 / N_ROWS), rb=128,
                                             workers=threads)
        sec = time.perf_counter() - t0
        rec["cpu_baseline"] = {"value": N_ROWS / sec, "unit": "positions/s", "cores": threads,
                               "kind": "reference",
                               "sample": f"reference ccem_forward + ccem_backward_rows (oracle/_ref) at full "
                                         f"N={N_ROWS}, K={K_NEG}, V={V}, D={D}, workers={threads}"}
        dEg = g.d_classifier.float().cpu().numpy()
        num = den = 0.0
        for a in range(0, V, 1 << 17):  # column blocks: bounded host memory
            b = min(V, a + (1 << 17))
            w = rdC[:, a:b].T
            num += float(np.sum((dEg[a:b] - w) ** 2))
            den += float(np.sum(w * w))
        tol = {"loss_rel": 1e-2, "lse_max_rel": 1e-3, "dX_normwise": 1e-2, "dE_normwise": 1e-2}
        p = {"rows": N_ROWS, "loss_rel": abs(float(o.loss) - loss) / max(1.0, abs(loss)),
             "lse_max_rel": rel(o.lse.cpu().numpy(), lse),
             "pos_max_rel": rel(o.pos_logits.cpu().numpy(), pos),
             "dX_normwise": normwise(g.d_embeddings.double().cpu().numpy(), rdE),
             "dE_normwise": (num / den) ** 0.5 if den else 0.0, "tolerance": tol}
        p["pass"] = bool(p["loss_rel"] < tol["loss_rel"] and p["lse_max_rel"] < tol["lse_max_rel"]
                         and p["dX_normwise"] < tol["dX_normwise"] and p["dE_normwise"] < tol["dE_normwise"])
        rec["parity"] = p
    del box[0], o, g, X3, E3, x3, inds
    torch.cuda.synchronize()
    return rec


def cfg1_record(lf, flush, stream, args, cpu):
    """BASELINE configs[0]: CCE fwd + bwd fp32, N = 2048 (batch 32 x seq 64),
    D = 64, V = 32768, filtering off — "bit-for-tolerance vs the CPU oracle".
    The reference itself (oracle/_ref, all host threads) runs the same
    make_instance inputs at full size; the GPU path is the public
    cce_forward_backward (the trainer's pairing, as for cfg2; fp32: the fused
    SIMT forward + dX, then the dE pass, exact exp)."""
    import numpy as np
    import torch
    from paper_2509_09682_b200 import synth
    dev = torch.device("cuda", torch.cuda.current_device())
    Xh, Ch, t1 = synth.make_instance(SEED1, N1, D, V1)
    X1 = torch.from_numpy(np.ascontiguousarray(Xh, np.float32)).to(dev)
    E1 = torch.from_numpy(np.ascontiguousarray(Ch.T, np.float32)).to(dev)
    x1 = torch.from_numpy(t1).to(dev)
    cfg = lf.CceConfig()
    box = [None]

    def step():
        box[0] = None
        box[0] = lf.cce_forward_backward(X1, E1, x1, 1.0, cfg, validate=False, stats=False)

    kern = {}
    ms = timed_steps(step, args.steps, max(3, args.warmup), stream, flush, kern)
    rec = {"workload": f"cfg1: CCE fp32, N={N1} (batch 32 x seq 64), D={D}, V={V1}, filtering off "
                       f"(make_instance seed {SEED1:#x})",
           "value": N1 / (ms / 1e3), "unit": "positions/s", "ms_per_step": ms, "steps": args.steps,
           "path": "lf_cce_forward_backward (fp32 SIMT: fused forward + dX, then the dE pass)",
           "kernel_ms_per_step": kern}
    # fp32 FMA roofline: algorithmic 8 N V D flops (logits 2 + dX 2 in the
    # fused pass, logits 2 + dE 2 in the dE pass; executed = algorithmic) against
    # the nominal CUDA-core fp32 rate (148 SMs x 128 lanes x 2 flop x max clock)
    peak32 = 148 * 128 * 2 * 1.965e9 / 1e12
    ach32 = 8.0 * N1 * V1 * D / (ms / 1e3) / 1e12
    rec["roofline"] = {"bound": "fp32 FMA (CUDA cores)", "achieved": ach32, "peak": peak32, "unit": "TFLOP/s",
                       "frac": ach32 / peak32, "traffic": None,
                       "peak_source": "nominal: 148 SMs x 128 FP32 lanes x 2 x 1.965 GHz (no measured fp32 peak)"}
    o, r = box[0]
    if cpu:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle_bind as ob
        threads = os.cpu_count() or 1
        t0 = time.perf_counter()
        loss, pos, lse = ob.ref_cce_forward(Xh, Ch, t1, workers=threads)
        rdE, rdC, _ = ob.ref_cce_backward(Xh, Ch, t1, lse, 1.0, 0.0, workers=threads)
        sec = time.perf_counter() - t0
        rec["cpu_baseline"] = {"value": N1 / sec, "unit": "positions/s", "cores": threads, "kind": "reference",
                               "sample": f"reference cce_forward + cce_backward (oracle/_ref) at full cfg1 size, "
                                         f"workers={threads}"}
        dXg = r.grads.d_embeddings.double().cpu().numpy()
        dEg = r.grads.d_classifier.double().cpu().numpy()
        tol = {"loss_rel": 1e-5, "lse_max_rel": 1e-5, "pos_max_rel": 1e-5, "dX_normwise": 1e-5,
               "dE_normwise": 1e-5}
        p = {"rows": N1, "loss_rel": abs(float(o.loss) - loss) / max(1.0, abs(loss)),
             "lse_max_rel": rel(o.lse.cpu().numpy(), lse), "pos_max_rel": rel(o.pos_logits.cpu().numpy(), pos),
             "dX_normwise": normwise(dXg, rdE), "dE_normwise": normwise(dEg, rdC.T), "tolerance": tol,
             "note": "fp32 tolerance of the north star (1e-5 relative); reference accumulates in double"}
        p["pass"] = all(p[k] < tol[k] for k in tol)
        rec["parity"] = p
    del box[0], o, r, X1, E1, x1
    torch.cuda.synchronize()
    return rec


def shard_record(lf, flush, stream, args, peaks):
    """Per-GPU work of the catalog-sharded configs (BASELINE configs[3],
    configs[4]) at P = 8, timed on this one GPU: the fused step over one
    rank's catalog slice (the exchange is not included — one all-gather of
    N*16 B and one all-reduce of N*D*4 B per step).  Synthetic
    torch.rand data of the shard's shape, bf16, eps = 6e-8."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev).manual_seed(0)
    out = []
    for name, n, d, v_total, P in (("cfg4: N=131072, D=128, V=4M over 8 GPUs", 131072, 128, 4_000_000, 8),
                                   ("cfg5: N=7680 (15% of 256x200), D=256, V=16M over 8 GPUs", 7680, 256,
                                    16_000_000, 8)):
        vs = v_total // P
        X = (torch.rand(n, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
        E = (torch.rand(vs, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
        x = torch.randint(0, vs, (n,), device=dev, generator=g)
        cfg = lf.CceConfig(filter_eps=EPS)
        box = [None]

        def step():
            box[0] = None
            box[0] = lf.cce_forward_backward(X, E, x, 1.0, cfg, validate=False)

        kern = {}
        ms = timed_steps(step, max(3, min(args.steps, 5)), 2, stream, flush, kern)
        flops = 8.0 * n * vs * d
        tc = flops / (ms / 1e3) / 1e12
        out.append({"config": name, "shard": {"n": n, "d": d, "v_shard": vs}, "ms_per_step": ms,
                    "kernel_ms_per_step": kern,
                    "compute_bound_job_positions_per_s": n / (ms / 1e3),
                    "roofline": {"bound": "tensor", "achieved": tc, "peak": peaks["tc_sustained"],
                                 "unit": "TFLOP/s", "frac": tc / peaks["tc_sustained"],
                                 "algorithmic_flops_per_step": flops}})
        del box[0], X, E, x
        torch.cuda.synchronize()
    return {"shards": out,
            "note": "one rank's fused CCE step at P = 8 on one B200 (no NVLink exchange: no multi-GPU "
                    "box in this round); compute_bound_job_positions_per_s = N / t_shard, the 8-GPU "
                    "job's rate if the two exchanges were free"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
