cd $GRAFT_REPO_ROOT
for L in paper_2001_01583_b200/libhpnfft.so build_var/sub2.so; do for P in 8x32 16x16 12x16; do
HPNFFT_LIB=$L HPNFFT_SWEEP_PATCH=$P timeout 120 python tools/profile_step.py --config 4 --timing --reps 3 2>&1 | tail -1 | grep -o "ok [0-9.]*\|'patch': '[0-9x]*'\|'spread': [0-9.]*" | tr '\n' ' '; echo $L
done; done
HPNFFT_LIB=build_var/sub2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
