#!/bin/bash
# Runs the reference's own test programs linked against the B200 drop-in
# (built by `make -C oracle dropin`), once per device dtype.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-dropin}; mkdir -p $O
for dt in ${DTYPES:-f64}; do
  for t in test_cce test_ccem test_memory test_oracles test_harness test_sampler acceptance; do
    LSEFORGE_B200_DTYPE=$dt LSEFORGE_THREADS=8 timeout 900 oracle/_ref/dropin/$t > $O/${t}_$dt.log 2>&1
    echo "$dt $t rc=$?"; tail -1 $O/${t}_$dt.log
  done
done
