#!/bin/bash
# GPU box: (1) the launch list of bench.py (gpu__time_duration, cold-cache serialised launches) and
# (2) one --set full capture of the hot-path kernels of a config-4 pass; each ncu command only after
# the same command exited 0 without ncu.  TAG names the outputs.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r2}
NCU=/usr/local/cuda/bin/ncu
CMD1="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD1 > gpurun_out/${TAG}_bench_plain.json 2>&1 && \
$NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD1 > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
CMD2="python tools/profile_step.py --config 4 --dist ${DIST:-uniform}"
$CMD2 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
$NCU --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_spread_sweep|k_point_records|k_fft_pass|k_keys|k_scatter|k_gather}" -s ${SKIP:-8} -c ${COUNT:-8} -o gpurun_out/${TAG}_prof $CMD2 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full capture rc=$?"
tail -3 gpurun_out/${TAG}_ncu_full.log
