cd $GRAFT_REPO_ROOT
for L in build_var/prof.so build_var/lw3.so build_var/lw2ns4.so; do
for D in uniform clustered; do
HPNFFT_LIB=$L timeout 120 python tools/profile_step.py --config 4 --dist $D --timing --reps 3 2>&1 | tail -1 | grep -o "'spread': [0-9.]*\|ok [0-9.]*" | tr '\n' ' '; echo $L $D
HPNFFT_LIB=$L HPNFFT_SWEEP_PROF=1 timeout 120 python tools/profile_step.py --config 4 --dist $D --reps 1 2>&1 | grep "sweep prof"
done; done
