cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -x -q -m gpu -k "config3 or ragged or inverse_config or ewald or tiny or cutoffs" 2>&1 | tail -1
ENUF_CELLS=32,45 timeout 300 python tools/enuf_bench.py 2>&1 | tail -2 | cut -c1-400
timeout 120 python tools/profile_step.py --config 4 --timing --reps 4
timeout 120 python tools/profile_step.py --config 4 --timing --reps 4 --inverse
