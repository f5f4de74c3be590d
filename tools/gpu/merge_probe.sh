#!/bin/bash
# clustered points: the sweep's merged-chunk list path forced on / off (HPNFFT_SWEEP_MERGE)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $NG"
[ "$NG" -eq 1 ] && RUN="python bench.py"
for mg in auto 1; do
  for dist in uniform clustered; do
    if [ $mg = auto ]; then unset HPNFFT_SWEEP_MERGE; else export HPNFFT_SWEEP_MERGE=$mg; fi
    HPNFFT_BENCH_RANK_STAGES=1 timeout 600 $RUN --steps 10 --warmup 3 --no-cpu-baseline --dist $dist --partition equal_count > gpurun_out/mp_${dist}_${mg}_n$NG.json 2> gpurun_out/mp_${dist}_${mg}_n$NG.err
    python - gpurun_out/mp_${dist}_${mg}_n$NG.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], "value %.4g ms %.3f" % (d["value"], d["ms_per_step"]))
    for ln in open(sys.argv[1][:-5] + ".err"):
        if ln.startswith('{"rank"'):
            r = json.loads(ln); st = r["stages"]
            print("  rank", r["rank"], "M", r["M_local"], "planes", r["info"], "spread", st.get("spread"), "records", st.get("records"))
except Exception as e:
    print(sys.argv[1], "no line", e)
PY
  done
done
