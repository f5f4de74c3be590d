cd $GRAFT_REPO_ROOT
timeout 120 python tools/profile_step.py --config 4 --timing --reps 3 2>&1 | tail -1 | cut -c1-400
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
