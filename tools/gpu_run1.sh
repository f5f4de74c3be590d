cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "inverse" 2>&1 | tail -1
timeout 120 python tools/profile_step.py --config 4 --timing --reps 3 --inverse 2>&1 | tail -1 | grep -o "'inv_fft': [0-9.]*\|'interp': [0-9.]*"
