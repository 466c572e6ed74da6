"""GPU: bench.py keeps its JSON contract — one line with the required keys,
for one rank and for two ranks (the catalog-sharded path; on a single-GPU box
both ranks share cuda:0 over gloo via LF_BENCH_SHARE_GPU=1)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "e2e",
        "clocks"}


def last_json(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_one_rank(cuda):
    p = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    j = last_json(p.stdout)
    assert KEYS <= set(j), KEYS - set(j)
    assert j["n_gpus"] == 1 and j["value"] > 0 and j["gpu_launches"] > 0
    assert j["roofline"]["frac"] > 0 and j["e2e"]["h2d_bytes_per_step"] > 0
    assert abs(j["loss"] - 17.3) < 0.1  # uniform logits: lse ~ ln(V) + var/2


@pytest.mark.parametrize("exchange,port", [("collective", 29571), ("peer", 29573)])
def test_bench_two_ranks_sharded(cuda, exchange, port):
    env = dict(os.environ, LF_BENCH_SHARE_GPU="1")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3",
                        "--exchange", exchange],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-2000:])
    j = last_json(p.stdout)
    assert j["n_gpus"] == 2 and "sharded" in j["config"]["parallelism"]
    assert exchange in j["config"]["parallelism"]
    assert abs(j["loss"] - 17.3) < 0.1  # the combined sharded loss equals the unsharded one
