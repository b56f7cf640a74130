cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./scripts/micro_tile > gpurun_out/micro_tile.txt 2>&1
