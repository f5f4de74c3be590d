cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c5_n1.json 2> gpurun_out/c5_n1.err; tail -c 1800 gpurun_out/c5_n1.json; tail -3 gpurun_out/c5_n1.err
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -c 400
