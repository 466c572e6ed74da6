#!/bin/bash
# One GPU-box pass: parity tests, a bench line, and ncu captures of the
# tensor-core kernels.  Outputs land in gpurun_out/ (merged back by gpurun).
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-run}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ "${TESTS:-1}" = 1 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  tail -3 $O/pytest_gpu.log
fi
if [ "${BENCH:-1}" = 1 ]; then
  timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:-} > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
  cat $O/bench.json
fi
if [ "${LAUNCHES:-0}" = 1 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_under_ncu.log 2>&1; echo "launches rc=$?"
fi
if [ "${NCU:-0}" = 1 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-cce_tc_kernel} -c ${NCU_C:-3} \
    -o $O/full -f python tools/time_probe.py --once 1 --eps ${EPS:-6e-8} ${PROBE_ARGS:-} > $O/ncu_full.log 2>&1; echo "ncu rc=$?"
  tail -5 $O/ncu_full.log
fi
if [ -n "${EXTRA:-}" ]; then bash -c "$EXTRA" > $O/extra.log 2>&1; echo "extra rc=$?"; tail -30 $O/extra.log; fi
