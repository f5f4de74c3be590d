#!/bin/bash
# GPU box: the round's 1-GPU evidence lines (bench.py as the driver runs it, plus the variants)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${TAG:-r2f}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_n1.json 2> gpurun_out/${T}_n1.err; echo "default rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 --dist clustered --partition equal_count --no-cpu-baseline > gpurun_out/${T}_n1_cl.json 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --direction inverse --no-cpu-baseline > gpurun_out/${T}_n1_inv.json 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --precision f32 --m 3 > gpurun_out/${T}_n1_f32.json 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; echo "ref rc=$?"
timeout 600 python tools/enuf_bench.py > gpurun_out/${T}_enuf.txt 2>&1
for f in gpurun_out/${T}_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], "value %.4g ms %.3f" % (d["value"], d["ms_per_step"]), "frac", (d.get("roofline") or {}).get("frac"), "clocks", d.get("clocks", {}).get("sm_mhz"), d.get("clocks", {}).get("reasons"))
except Exception as e:
    print(sys.argv[1], "no line", e)
PY
done
