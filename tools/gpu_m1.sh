cd $GRAFT_REPO_ROOT
timeout 800 python -m pytest tests/test_gpu_parity.py -x -q -s -m gpu -k "cutoffs or windows_bspline or fig12" 2>&1 | grep -E "^E |FAILED|passed|failed|\(a\)" | head -12
