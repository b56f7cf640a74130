cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pp
run() { # name nproc args...
  name=$1; np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > gpurun_out/pp/$name.log 2>&1; echo "rc=$?" >> gpurun_out/pp/$name.log
  python - gpurun_out/pp/$name.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[1], "NO JSON", open(sys.argv[1]).read()[-800:]); sys.exit()
d=json.loads(l[-1]); print(sys.argv[1], d["value"], "eager", d.get("eager_ms_per_step"))
PY
}
for proto in default Simple LL128 "^LL"; do
  if [ "$proto" = default ]; then unset NCCL_PROTO; else export NCCL_PROTO="$proto"; fi
  tag=$(echo $proto | tr -d '^')
  run 15d_n4_$tag 4 --strategy 1.5d --steps 10 --warmup 3 --no-alt
  run 2d_n4_$tag 4 --strategy 2d --steps 10 --warmup 3 --no-alt
  run 15d_n2_$tag 2 --strategy 1.5d --steps 10 --warmup 3 --no-alt
done
unset NCCL_PROTO
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=TUNING timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 --strategy 1.5d --steps 2 --warmup 3 --no-alt > gpurun_out/pp/nccl_debug.log 2>&1
grep -i "nvls\|algo\|proto" gpurun_out/pp/nccl_debug.log | head -30
