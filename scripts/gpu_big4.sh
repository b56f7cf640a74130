cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/big4
run() { # name nproc args...
  name=$1; np=$2; shift 2
  if [ $np = 1 ]; then
    timeout 900 python bench.py --gpus 1 "$@" > gpurun_out/big4/$name.log 2>&1; echo "rc=$?" >> gpurun_out/big4/$name.log
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > gpurun_out/big4/$name.log 2>&1; echo "rc=$?" >> gpurun_out/big4/$name.log
  fi
  python - gpurun_out/big4/$name.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[1], "NO JSON", open(sys.argv[1]).read()[-800:]); sys.exit()
d=json.loads(l[-1]); print(sys.argv[1], d["value"], "eager", d.get("eager_ms_per_step"), "e2e", d["e2e"]["value"], d["config"].get("workload"), {k:(v["launches"],v["ms_per_launch"]) for k,v in d["kernels"].items()})
PY
}
run amazon_1d_n1 1 --config amazon --steps 3 --warmup 3 --no-alt --no-cpu-baseline
run amazon_2d_n4 4 --config amazon --strategy 2d --steps 3 --warmup 3 --no-alt
run amazon_1d_n4 4 --config amazon --steps 3 --warmup 3 --no-alt
run protein_1d_n1 1 --config protein --steps 3 --warmup 3 --no-alt --no-cpu-baseline
run protein_15d_n4 4 --config protein --strategy 1.5d --steps 3 --warmup 3 --no-alt
run protein_1d_n4 4 --config protein --steps 3 --warmup 3 --no-alt
run reddit_1d_n4 4 --steps 10 --warmup 3 --no-alt
run reddit_15d_n4 4 --strategy 1.5d --steps 10 --warmup 3 --no-alt
run reddit_2d_n4 4 --strategy 2d --steps 10 --warmup 3 --no-alt
run reddit_1d_n2 2 --steps 10 --warmup 3 --no-alt
run reddit_15d_n2 2 --strategy 1.5d --steps 10 --warmup 3 --no-alt
