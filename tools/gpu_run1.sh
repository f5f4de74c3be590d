cd $GRAFT_REPO_ROOT
for D in uniform clustered; do for P in 12x16 8x32; do
  HPNFFT_SWEEP_PATCH=$P timeout 120 python tools/profile_step.py --config 4 --dist $D --timing --reps 3 2>&1 | tail -1 | cut -c1-200
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
