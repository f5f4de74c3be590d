cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
timeout 300 python tools/enuf_bench.py 2>&1 | tail -4 | cut -c1-330
timeout 120 python tools/profile_step.py --config 4 --timing --reps 4 | cut -c1-250
timeout 120 python tools/profile_step.py --config 3 --timing --reps 4 | cut -c1-250
