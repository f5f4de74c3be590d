cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -v "^\s*$" | grep -A30 "FAILURES\|Error" | head -50
