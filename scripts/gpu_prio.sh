cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pr
run() { # name nproc args...
  name=$1; np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > gpurun_out/pr/$name.log 2>&1; echo "rc=$?" >> gpurun_out/pr/$name.log
  python - gpurun_out/pr/$name.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[1], "NO JSON", open(sys.argv[1]).read()[-800:]); sys.exit()
d=json.loads(l[-1]); print(sys.argv[1], d["value"], "eager", d.get("eager_ms_per_step"), {k:(v["launches"],v["ms_per_launch"]) for k,v in d["kernels"].items()})
PY
}
run 2d_n4 4 --strategy 2d --steps 10 --warmup 3 --no-alt
run 15d_n4 4 --strategy 1.5d --steps 10 --warmup 3 --no-alt
run 1d_n4 4 --steps 10 --warmup 3 --no-alt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) scripts/timeline.py --gpus 4 --strategy 2d > gpurun_out/pr/tl.log 2>&1
mv gpurun_out/timeline_2d_n4_r0.txt gpurun_out/pr/
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) scripts/timeline.py --gpus 4 --strategy 1.5d > gpurun_out/pr/tl15.log 2>&1
mv gpurun_out/timeline_1.5d_n4_r0.txt gpurun_out/pr/
rm -f gpurun_out/timeline_*
