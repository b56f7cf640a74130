cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sg
timeout 900 python -m pytest tests -m gpu -q --timeout 240 -p no:cacheprovider -rf -x > gpurun_out/sg/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sg/pytest.log
tail -4 gpurun_out/sg/pytest.log
for cfg in reddit amazon protein; do
timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-alt --no-cpu-baseline > gpurun_out/sg/$cfg.log 2>&1
python - gpurun_out/sg/$cfg.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[1], "NO JSON", open(sys.argv[1]).read()[-1500:]); sys.exit()
d=json.loads(l[-1]); print(sys.argv[1], d["value"], "e2e", d["e2e"]["value"], json.dumps(d.get("epoch_roofline")), {k:(v["launches"],v["ms_per_launch"],v["GBps"]) for k,v in d["kernels"].items()})
PY
done
