cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 900 python -m pytest tests -m "gpu" -q --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest_multi.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi.log
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bench_1d_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_1d_n$N.log
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --strategy 1.5d --steps 5 --warmup 3 > gpurun_out/bench_15d_n4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_15d_n4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --strategy 2d --steps 5 --warmup 3 > gpurun_out/bench_2d_n4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_2d_n4.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
