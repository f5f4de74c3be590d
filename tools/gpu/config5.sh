#!/bin/bash
# GPU box: BASELINE config 5 (N = 512^3, M = 1e9) on the visible GPUs (1, 2 or 4)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
TAG=${TAG:-c5}
if [ "$NG" -gt 1 ]; then
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $NG --config 5 --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_n$NG.json 2> gpurun_out/${TAG}_n$NG.err
else
  timeout 1500 python bench.py --config 5 --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_n1.json 2> gpurun_out/${TAG}_n1.err
fi
echo "rc=$?"
python - "$TAG" "$NG" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/{sys.argv[1]}_n{sys.argv[2]}.json").read().strip().splitlines()[-1])
    print("value %.4g ms %.2f" % (d["value"], d["ms_per_step"]), d["detail"]["stages_ms"], d["config"]["exchange"][:40], d["detail"].get("record_group"))
except Exception as e:
    print("no line", e)
PY
tail -3 gpurun_out/${TAG}_n$NG.err
