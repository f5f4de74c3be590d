cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
for L in paper_2001_01583_b200/libhpnfft.so build_var/dbg1.so; do
for P in 8x32 12x32; do
  echo "== $L $P"
  HPNFFT_LIB=$L HPNFFT_SWEEP_PATCH=$P timeout 120 python tools/profile_step.py --config 4 --timing --reps 3 2>&1 | tail -1 | cut -c1-400
  HPNFFT_LIB=$L HPNFFT_SWEEP_PROF=1 HPNFFT_SWEEP_PATCH=$P timeout 120 python tools/profile_step.py --config 4 --reps 1 2>&1 | grep "sweep prof"
done; done
HPNFFT_SWEEP_PATCH=8x32 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spread_sweep -c 1 -o gpurun_out/prof_sweep_c2 -f python tools/profile_step.py --config 4 --reps 1 > gpurun_out/ncu_c2.log 2>&1; tail -1 gpurun_out/ncu_c2.log
