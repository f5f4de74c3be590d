cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "sweep or config3 or ragged or clustered or thin or cutoffs" 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
for i in 1 2; do for L in libhpnfft.so ${ALT:-libhpnfft_noleanf.so}; do HPNFFT_LIB=paper_2001_01583_b200/$L timeout 120 python tools/profile_step.py --config 4 --timing --reps 4 | python -c "import sys,ast; s=sys.stdin.read(); d=ast.literal_eval(s[s.index('{'):]); print('$L', round(d['spread'],3), round(d['records'],3))"; done; done
for L in libhpnfft.so ${ALT:-libhpnfft_noleanf.so}; do HPNFFT_LIB=paper_2001_01583_b200/$L ENUF_CELLS=32,45 timeout 300 python tools/enuf_bench.py 2>&1 | tail -2 | cut -c1-140; done
