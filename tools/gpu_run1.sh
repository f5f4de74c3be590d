cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 5 --warmup 3 --direction inverse 2>/dev/null | tail -1 > gpurun_out/inv_n1.json; cut -c1-200 gpurun_out/inv_n1.json
