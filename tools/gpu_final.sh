cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; tail -c 400 gpurun_out/final_n1.json
timeout 600 python bench.py --steps 10 --warmup 3 --dist clustered --no-cpu-baseline > gpurun_out/final_n1_cl.json 2>/dev/null
timeout 600 python bench.py --steps 5 --warmup 3 --direction inverse > gpurun_out/final_inv.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_launch.log 2>&1; tail -1 gpurun_out/final_ncu_launch.log
timeout 300 python tools/enuf_bench.py > gpurun_out/final_enuf.txt 2>&1; tail -4 gpurun_out/final_enuf.txt | cut -c1-120
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
