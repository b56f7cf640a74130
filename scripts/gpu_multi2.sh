cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_training.py -m "gpu" -k "distributed" -q --timeout 240 -p no:cacheprovider -rf > gpurun_out/pytest_multi.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi.log
python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/m_1d_n1.log 2>&1
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 5 --warmup 2 > gpurun_out/m_1d_n$N.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --strategy 1.5d --steps 5 --warmup 2 > gpurun_out/m_15d_n4.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --strategy 2d --steps 5 --warmup 2 > gpurun_out/m_2d_n4.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/m_ref.log 2>&1
