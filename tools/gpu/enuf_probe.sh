#!/bin/bash
# ENUF reciprocal energy at 45^3 / 64^3 cells against library variants and spread methods
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "${PYK:-sort or ewald or rank_group}" > gpurun_out/ep_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ep_pytest.log
for v in ${VARIANTS:-libhpnfft.so}; do
  for meth in ${METHODS:-auto}; do
    echo "== $v $meth"
    HPNFFT_LIB=$PWD/paper_2001_01583_b200/$v ENUF_METHOD=$meth ENUF_CELLS=${CELLS:-45,64} timeout 600 python tools/enuf_bench.py 2>&1 | cut -c1-420
  done
done
