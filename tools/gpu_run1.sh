cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_point_records|k_fft_pass|k_keys|k_gather_x|k_scatter" -c 7 -o gpurun_out/prof_rec_fft2 -f python tools/profile_step.py --config 4 --reps 1 > gpurun_out/ncu_rf2.log 2>&1; tail -1 gpurun_out/ncu_rf2.log
