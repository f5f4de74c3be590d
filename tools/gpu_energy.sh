cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "ewald" 2>&1 | grep -E "^E |FAILED|passed|failed|Error" | head -20
NG=${NG:-2}
if [ "$NG" -gt 1 ]; then
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 tools/dist_check.py 2>&1 | grep -v "^W1\|OMP_NUM" | grep "ewald\|rror\|FAIL" | tail -8
fi
