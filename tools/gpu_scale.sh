cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=${NG:-2}
for EX in grid_slab allreduce; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $NG --steps 10 --warmup 3 --exchange $EX > gpurun_out/scale_n${NG}_$EX.json 2> gpurun_out/scale_n${NG}_$EX.err
  tail -1 gpurun_out/scale_n${NG}_$EX.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$EX', d['n_gpus'], '%.3e'%d['value'], '%.2f ms'%d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], {k: round(v,3) for k,v in d['detail']['stages_ms'].items() if v})" || tail -5 gpurun_out/scale_n${NG}_$EX.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus $NG --steps 10 --warmup 3 --exchange grid_slab --dist clustered > gpurun_out/scale_n${NG}_grid_slab_cl.json 2>/dev/null
tail -1 gpurun_out/scale_n${NG}_grid_slab_cl.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('clustered grid_slab', d['n_gpus'], '%.3e'%d['value'])"
