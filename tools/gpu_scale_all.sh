cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for NG in 2 4; do
  for EX in grid_slab allreduce; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2952$NG bench.py --gpus $NG --steps 10 --warmup 3 --exchange $EX > gpurun_out/scale_n${NG}_$EX.json 2> gpurun_out/scale_n${NG}_$EX.err
    tail -1 gpurun_out/scale_n${NG}_$EX.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$EX', d['n_gpus'], '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'])" || tail -3 gpurun_out/scale_n${NG}_$EX.err
  done
  for PART in equal_size equal_count; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2953$NG bench.py --gpus $NG --steps 10 --warmup 3 --exchange grid_slab --dist clustered --partition $PART > gpurun_out/scale_n${NG}_grid_slab_cl_$PART.json 2>/dev/null
    tail -1 gpurun_out/scale_n${NG}_grid_slab_cl_$PART.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('clustered $PART', d['n_gpus'], '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'])"
  done
done
