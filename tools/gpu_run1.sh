cd $GRAFT_REPO_ROOT
for D in clustered uniform; do for P in 12x16 16x16 8x32; do
HPNFFT_SWEEP_PATCH=$P timeout 120 python tools/profile_step.py --config 4 --dist $D --timing --reps 4 2>&1 | tail -1 | grep -o "'dist': '[a-z]*'\|'patch': '[0-9x]*'\|'spread': [0-9.]*" | tr '\n' ' '; echo
done; done
