cd $GRAFT_REPO_ROOT
run() { # name nproc args...
  name=$1; np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > gpurun_out/s4b_$name.log 2>&1; echo "rc=$?" >> gpurun_out/s4b_$name.log
}
run 1d_n4_a 4 --steps 10 --warmup 3 --no-alt --no-cpu-baseline
run 1d_n4_f0 4 --steps 10 --warmup 3 --no-alt --fuse 0
run 1d_n4_b 4 --steps 10 --warmup 3 --no-alt
run 1d_n2 2 --steps 10 --warmup 3 --no-alt
