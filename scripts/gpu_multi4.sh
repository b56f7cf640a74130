cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/m4
timeout 1200 python -m pytest tests -m "gpu" -q --timeout 300 -p no:cacheprovider -rf > gpurun_out/m4/pytest_multi4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/m4/pytest_multi4.log
run() { # name nproc args...
  name=$1; np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > gpurun_out/m4/$name.log 2>&1; echo "rc=$?" >> gpurun_out/m4/$name.log
}
run 1d_n2 2 --steps 10 --warmup 3 --no-alt
run 1d_n4 4 --steps 10 --warmup 3 --no-alt
run 15d_n4 4 --strategy 1.5d --steps 10 --warmup 3 --no-alt
run 2d_n4 4 --strategy 2d --steps 10 --warmup 3 --no-alt
run 15d_n2 2 --strategy 1.5d --steps 10 --warmup 3 --no-alt
