cd $GRAFT_REPO_ROOT
NG=${NG:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 tools/dist_check.py 2>&1 | grep -v "^W1\|OMP_NUM" | tail -12
