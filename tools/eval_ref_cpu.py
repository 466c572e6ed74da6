"""CPU baseline for full-catalog evaluation: the reference's own evaluate()
(metrics.cpp:13-103, oracle/_ref — the unmodified sources compiled in place)
on a bounded sample of the cfg2 shape (V = 1M items, D = 64), all host
threads.  Prints one JSON line with rows/s.  Test/measurement infrastructure."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_bind as ob  # noqa: E402

n = int(os.environ.get("ROWS", "256"))
v, d, k = 1_000_000, 64, 10
workers = os.cpu_count() or 1
g = np.random.default_rng(0)
pre = g.integers(0, v, (n, 4))
tg = g.integers(0, v, n)
counts = g.integers(0, 40, v)


def timed(rows):
    t = time.perf_counter()
    ob.ref_eval_instance(v, d, 1, pre[:rows], tg[:rows], k, counts, workers, extras=False)
    return time.perf_counter() - t


t_small = timed(workers)  # parameter init + one row per thread
t_big = timed(n)
per_row = (t_big - t_small) / (n - workers)
print(json.dumps({"probe": "reference evaluate() (oracle/_ref)", "rows": n, "v": v, "d": d, "k": k,
                  "threads": workers, "seconds": t_big, "rows_per_s": 1.0 / per_row,
                  "note": "per-row cost = (T(rows) - T(threads)) / (rows - threads): excludes the "
                          "ToyEncoderParams::Init of the 1M-item tables that every call pays"}))
