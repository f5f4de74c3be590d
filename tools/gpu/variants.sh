#!/bin/bash
# GPU box: bench.py (config 4, no CPU baseline) against several library variants: VARIANTS="a.so b.so"
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in $VARIANTS; do
  for dist in ${DISTS:-uniform}; do
    HPNFFT_LIB=$PWD/paper_2001_01583_b200/$v timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --dist $dist ${BENCH_ARGS} > gpurun_out/var_${v%.so}_$dist.json 2>&1
    python - "$v" "$dist" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/var_{sys.argv[1][:-3]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
st = d["detail"]["stages_ms"]
print(sys.argv[1], sys.argv[2], "value %.4g" % d["value"], "ms %.3f" % d["ms_per_step"], "spread %.3f records %.3f sweep %.3f" % (st["spread"], st["records"], st["spread"] - st["records"]))
PY
  done
done
