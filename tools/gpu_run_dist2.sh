cd $GRAFT_REPO_ROOT
bash tools/gpu_run_dist.sh
bash tools/gpu_scale.sh
