cd $GRAFT_REPO_ROOT
for L in paper_2001_01583_b200/libhpnfft.so build_var/tw1.so build_var/fftc4.so build_var/fftc8.so; do
HPNFFT_LIB=$L timeout 120 python tools/profile_step.py --config 4 --timing --reps 3 2>&1 | tail -1 | grep -o "'fft_[a-z_]*': [0-9.]*" | tr '\n' ' '; echo
done
HPNFFT_LIB=build_var/tw1.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
