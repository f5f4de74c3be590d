cd $GRAFT_REPO_ROOT
NG=${NG:-4}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
NG=$NG bash tools/gpu_run_dist2.sh
