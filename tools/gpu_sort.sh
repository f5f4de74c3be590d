cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config3 or ragged or clustered or thin or partition or async" 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
for F in 1 0 1 0; do HPNFFT_SORT_FUSED=$F timeout 120 python tools/profile_step.py --config 4 --timing --reps 4 | python -c "import sys,ast; s=sys.stdin.read(); d=ast.literal_eval(s[s.index('{'):]); print('fused=$F', round(d['keys'],3), round(d['scan'],3), round(d['scatter'],3), round(d['spread'],3))"; done
