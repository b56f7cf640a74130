# 2- and 4-GPU Reddit bench lines only (torchrun, one process per GPU).
cd $GRAFT_REPO_ROOT
O=gpurun_out/${ROUND_TAG:-r02}_m4b
mkdir -p $O
run() { # name nproc args...
  name=$1; np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > $O/$name.log 2>&1; echo "rc=$?" >> $O/$name.log
}
run reddit_1d_n2 2 --steps 20 --warmup 5 --no-alt
run reddit_1d_n4 4 --steps 20 --warmup 5 --no-alt
run reddit_15d_n4 4 --strategy 1.5d --steps 20 --warmup 5 --no-alt
run reddit_2d_n4 4 --strategy 2d --steps 20 --warmup 5 --no-alt
grep -h '^{' $O/*.log > $O/bench_multi.jsonl
python -c "
import json
for l in open('$O/bench_multi.jsonl'):
  d=json.loads(l); print(d['n_gpus'], d['config']['strategy'], d['value'], d['e2e']['value'], d['e2e']['sync_ms'])"
