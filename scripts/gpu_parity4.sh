# 4-GPU bench lines with the in-bench parity check (rank 0 re-trains at P = 1 and compares losses).
cd $GRAFT_REPO_ROOT
O=gpurun_out/${ROUND_TAG:-r02}_p4
mkdir -p $O
run() { # name nproc args...
  name=$1; np=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > $O/$name.log 2>&1; echo "rc=$?" >> $O/$name.log
}
run reddit_1d_n4 4 --steps 20 --warmup 5 --no-alt
run reddit_15d_n4 4 --strategy 1.5d --steps 20 --warmup 5 --no-alt
run reddit_2d_n4 4 --strategy 2d --steps 20 --warmup 5 --no-alt
run reddit_1d_n2 2 --steps 20 --warmup 5 --no-alt
run amazon_1d_n4 4 --config amazon --steps 3 --warmup 3 --no-alt
grep -h '^{' $O/*.log > $O/bench_multi.jsonl
