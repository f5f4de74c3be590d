#!/bin/bash
# GPU box: 1-GPU bench line (default config 4), the reference arm, and a clustered line
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TAG=${TAG:-b}
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_n1.json 2> gpurun_out/${TAG}_n1.err; echo "bench rc=$?"
tail -c 600 gpurun_out/${TAG}_n1.json
timeout 900 python bench.py --steps 10 --warmup 3 --dist clustered --no-cpu-baseline > gpurun_out/${TAG}_n1_cl.json 2>&1
timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-5} --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
tail -c 300 gpurun_out/${TAG}_ref.json
