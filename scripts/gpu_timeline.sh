cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for np in 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) scripts/timeline.py --gpus $np > gpurun_out/tl_$np.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) scripts/timeline.py --gpus 4 --strategy 2d > gpurun_out/tl_2d.log 2>&1
timeout 600 python scripts/timeline.py --gpus 1 > gpurun_out/tl_1.log 2>&1
tail -3 gpurun_out/tl_*.log
