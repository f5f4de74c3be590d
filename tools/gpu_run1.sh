cd $GRAFT_REPO_ROOT
for L in paper_2001_01583_b200/libhpnfft.so build_var/ntskip.so; do
HPNFFT_LIB=$L timeout 120 python tools/profile_step.py --config 4 --timing --reps 3 2>&1 | tail -1 | cut -c1-240
done
HPNFFT_LIB=build_var/ntskip.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
