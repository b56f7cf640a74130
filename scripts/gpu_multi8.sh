cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/m8
nvidia-smi -L > gpurun_out/m8/gpus.txt 2>&1
timeout 1200 python -m pytest tests -m "gpu" -q --timeout 300 -p no:cacheprovider -rf -k "distributed or resident or exchange or ledger or multigpu" > gpurun_out/m8/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/m8/pytest.log
tail -5 gpurun_out/m8/pytest.log
run() { # name nproc args...
  name=$1; np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np "$@" > gpurun_out/m8/$name.log 2>&1; echo "rc=$?" >> gpurun_out/m8/$name.log
  python - gpurun_out/m8/$name.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[1], "NO JSON", open(sys.argv[1]).read()[-800:]); sys.exit()
d=json.loads(l[-1]); print(sys.argv[1], d["value"], "eager", d.get("eager_ms_per_step"), "e2e", d["e2e"]["value"], {k:(v["launches"],v["ms_per_launch"]) for k,v in d["kernels"].items()})
PY
}
run reddit_1d_n8 8 --steps 10 --warmup 3 --no-alt
run reddit_15d_n8 8 --strategy 1.5d --steps 10 --warmup 3 --no-alt
run reddit_3d_n8 8 --strategy 3d --steps 10 --warmup 3 --no-alt
run amazon_3d_n8 8 --config amazon --strategy 3d --steps 3 --warmup 3 --no-alt
run amazon_2d_n8 8 --config amazon --strategy 1d --steps 3 --warmup 3 --no-alt
run protein_15d_n8 8 --config protein --strategy 1.5d --steps 3 --warmup 3 --no-alt
run protein_3d_n8 8 --config protein --strategy 3d --steps 3 --warmup 3 --no-alt
