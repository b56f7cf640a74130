cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pu2
timeout 900 python -m pytest tests/test_gpu_training.py -m "gpu" -q --timeout 300 -p no:cacheprovider -rf -x -k "exchange or odd or distributed" > gpurun_out/pu2/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pu2/pytest.log
tail -2 gpurun_out/pu2/pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --steps 10 --warmup 3 --no-alt > gpurun_out/pu2/b4.log 2>&1
grep "^{" gpurun_out/pu2/b4.log | cut -c1-200
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) scripts/timeline.py --gpus 4 > gpurun_out/pu2/tl.log 2>&1
mv gpurun_out/timeline_1d_n4_r0.txt gpurun_out/pu2/; rm -f gpurun_out/timeline_*
