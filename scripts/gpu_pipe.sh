cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pp2
timeout 900 python -m pytest tests/test_gpu_training.py -m "gpu" -q --timeout 300 -p no:cacheprovider -rf -x -k "exchange or distributed" > gpurun_out/pp2/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pp2/pytest.log
tail -3 gpurun_out/pp2/pytest.log
run() { # name nproc args...
  name=$1; np=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > gpurun_out/pp2/$name.log 2>&1; echo "rc=$?" >> gpurun_out/pp2/$name.log
  python - gpurun_out/pp2/$name.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[1], "NO JSON", open(sys.argv[1]).read()[-1500:]); sys.exit()
d=json.loads(l[-1]); print(sys.argv[1], d["value"], "eager", d.get("eager_ms_per_step"), "e2e", d["e2e"]["value"], d["epoch_roofline"]["bound"], d["epoch_roofline"]["t_link_ms"], {k:(v["launches"],v["ms_per_launch"]) for k,v in d["kernels"].items()})
PY
}
run amazon_1d_n4 4 --config amazon --steps 3 --warmup 3 --no-alt
run protein_1d_n4 4 --config protein --steps 3 --warmup 3 --no-alt
run amazon_1d_n2 2 --config amazon --steps 3 --warmup 3 --no-alt
run reddit_1d_n4 4 --steps 10 --warmup 3 --no-alt
