cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "n1024 or ewald or ragged or inverse_config3" 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
timeout 300 python tools/enuf_bench.py 2>&1 | tail -4 | cut -c1-330
