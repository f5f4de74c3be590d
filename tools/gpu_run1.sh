cd $GRAFT_REPO_ROOT
for D in uniform clustered; do
  timeout 120 python tools/profile_step.py --config 4 --dist $D --timing --reps 3 2>&1 | tail -1 | cut -c1-200
  HPNFFT_SWEEP_PROF=1 timeout 120 python tools/profile_step.py --config 4 --dist $D --reps 1 2>&1 | grep "sweep prof"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
