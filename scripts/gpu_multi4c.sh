cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_training.py tests/test_harness.py -m "gpu" -q --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest_multi4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi4.log
run() { # name nproc args...
  name=$1; np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > gpurun_out/s4_$name.log 2>&1; echo "rc=$?" >> gpurun_out/s4_$name.log
}
run 1d_n2 2 --steps 10 --warmup 3 --no-alt
run 1d_n4 4 --steps 10 --warmup 3 --no-alt
