#!/bin/bash
# Time (and optionally check filtered accuracy of) every tuning variant under
# build/variants (cfg2 shape).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for so in paper_2509_09682_b200/liblseforge_b200.so paper_2509_09682_b200/build/variants/*.so; do
  echo "== $so"
  LSEFORGE_B200_LIB=$PWD/$so timeout 300 python tools/time_probe.py --eps ${EPS:-6e-8} --iters 5 2>&1 | tail -1
  if [ "${ACC:-0}" = 1 ]; then
    for g in 0 1; do LSEFORGE_B200_LIB=$PWD/$so timeout 300 python tools/filter_accuracy.py --gamma $g 2>&1 | tail -1; done
  fi
done
