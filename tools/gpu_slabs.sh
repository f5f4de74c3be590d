cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=${NG:-4}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 tools/dist_check.py 2>&1 | grep -v "^W1\|OMP_NUM" | tail -14
HPNFFT_DIST_P2P=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29512 tools/dist_check.py 2>&1 | grep -v "^W1\|OMP_NUM" | grep "grid_slab\|ALL\|FAIL\|rror" | tail -8
for PART in equal_size equal_count; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus $NG --steps 10 --warmup 3 --exchange grid_slab --dist clustered --partition $PART > gpurun_out/scale_n${NG}_grid_slab_cl_$PART.json 2> gpurun_out/scale_n${NG}_cl_$PART.err
  tail -1 gpurun_out/scale_n${NG}_grid_slab_cl_$PART.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('clustered grid_slab $PART', d['n_gpus'], '%.3e'%d['value'], '%.2f ms'%d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'])" || tail -5 gpurun_out/scale_n${NG}_cl_$PART.err
done
