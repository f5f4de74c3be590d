cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "n1024 or config3 or ewald" 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
ENUF_CELLS=45 timeout 300 python tools/enuf_bench.py 2>&1 | tail -1 | cut -c1-330
HPNFFT_FFT1024=0 ENUF_CELLS=45 timeout 300 python tools/enuf_bench.py 2>&1 | tail -1 | cut -c1-330
