#!/bin/bash
# GPU box with NG GPUs: bench.py at config 4 (uniform, clustered equal-cost) and config 5 on all GPUs
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
TAG=${TAG:-sc}
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $NG"
[ "$NG" -eq 1 ] && RUN="python bench.py"
timeout 900 $RUN --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_c4_n$NG.json 2> gpurun_out/${TAG}_c4_n$NG.err; echo "c4 rc=$?"
timeout 900 $RUN --steps 10 --warmup 3 --no-cpu-baseline --dist clustered --partition equal_count > gpurun_out/${TAG}_c4cl_n$NG.json 2> gpurun_out/${TAG}_c4cl_n$NG.err; echo "c4cl rc=$?"
timeout 1500 $RUN --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_c5_n$NG.json 2> gpurun_out/${TAG}_c5_n$NG.err; echo "c5 rc=$?"
for f in gpurun_out/${TAG}_*_n$NG.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], "value %.4g ms %.3f e2e %s" % (d["value"], d["ms_per_step"], (d.get("e2e") or {}).get("value")))
except Exception as e:
    print(sys.argv[1], "no line", e)
PY
done
