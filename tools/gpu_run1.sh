cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 5 --warmup 3 --direction inverse 2>&1 | tail -1 | cut -c1-900
