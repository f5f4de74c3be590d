cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "async or pipeline or errors or timing" 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/async_n1.json 2> gpurun_out/async_n1.err
tail -1 gpurun_out/async_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n1', '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], d['e2e']['ms_per_step'])" || tail -5 gpurun_out/async_n1.err
for NG in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2951$NG bench.py --gpus $NG --steps 10 --warmup 3 > gpurun_out/async_n$NG.json 2> gpurun_out/async_n$NG.err
  tail -1 gpurun_out/async_n$NG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n$NG', '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], d['e2e']['ms_per_step'])" || tail -5 gpurun_out/async_n$NG.err
done
