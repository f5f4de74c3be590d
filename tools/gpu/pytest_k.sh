#!/bin/bash
# GPU box: a subset of the GPU tests (K = pytest -k expression)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout ${TMO:-1800} python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$K" -s > gpurun_out/pytest_${TAG:-k}.log 2>&1
echo "rc=$?"; tail -${TAILN:-25} gpurun_out/pytest_${TAG:-k}.log
