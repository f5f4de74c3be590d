cd $GRAFT_REPO_ROOT
for P in 8x32 12x16; do
  HPNFFT_SWEEP_PATCH=$P timeout 120 python tools/profile_step.py --config 4 --timing --reps 3 2>&1 | tail -1 | cut -c1-250
  HPNFFT_SWEEP_PATCH=$P HPNFFT_SWEEP_PROF=1 timeout 120 python tools/profile_step.py --config 4 --reps 1 2>&1 | grep "sweep prof"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
