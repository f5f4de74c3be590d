cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; tail -c 600 gpurun_out/final_n1.json
timeout 600 python bench.py --steps 10 --warmup 3 --dist clustered > gpurun_out/final_n1_cl.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; tail -c 300 gpurun_out/final_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_launch.log 2>&1; tail -1 gpurun_out/final_ncu_launch.log
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_spread_sweep|k_point_records|k_fft_pass" -c 5 -o gpurun_out/prof_final -f python tools/profile_step.py --config 4 --reps 1 > gpurun_out/ncu_final.log 2>&1; tail -1 gpurun_out/ncu_final.log
