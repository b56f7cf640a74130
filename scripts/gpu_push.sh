cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pu
timeout 1500 python -m pytest tests -m "gpu" -q --timeout 300 -p no:cacheprovider -rf -x > gpurun_out/pu/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pu/pytest.log
tail -4 gpurun_out/pu/pytest.log
run() { # name nproc args...
  name=$1; np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > gpurun_out/pu/$name.log 2>&1; echo "rc=$?" >> gpurun_out/pu/$name.log
  python - gpurun_out/pu/$name.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[1], "NO JSON", open(sys.argv[1]).read()[-1500:]); sys.exit()
d=json.loads(l[-1]); print(sys.argv[1], d["value"], "eager", d.get("eager_ms_per_step"), "loss", d.get("loss_last"))
PY
}
run 1d_n2 2 --steps 10 --warmup 3 --no-alt
run 1d_n4 4 --steps 10 --warmup 3 --no-alt
run 1d_n4b 4 --steps 20 --warmup 3 --no-alt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) scripts/timeline.py --gpus 4 > gpurun_out/pu/tl.log 2>&1
mv gpurun_out/timeline_1d_n4_r0.txt gpurun_out/pu/; rm -f gpurun_out/timeline_*
