cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t4
timeout 1500 python -m pytest tests -m "gpu" -q --timeout 300 -p no:cacheprovider -rf > gpurun_out/t4/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t4/pytest.log
tail -5 gpurun_out/t4/pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --steps 10 --warmup 3 --no-alt > gpurun_out/t4/1d_n4.log 2>&1
grep "^{" gpurun_out/t4/1d_n4.log | cut -c1-300
