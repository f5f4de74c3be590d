#!/bin/bash
# GPU box: one compute-sanitizer tool (TOOL=memcheck|racecheck|synccheck|initcheck) on the small
# cases of tools/sanitize_case.py, after a plain run of the same command has exited 0
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TOOL=${TOOL:-memcheck}
timeout 600 python tools/sanitize_case.py > gpurun_out/san_plain_${TOOL}.log 2>&1 && \
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool ${TOOL} ${SAN_ARGS} --print-limit 50 \
    python tools/sanitize_case.py > gpurun_out/san_${TOOL}.log 2>&1
echo "sanitizer ${TOOL} rc=$?"
tail -8 gpurun_out/san_${TOOL}.log
