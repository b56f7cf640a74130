cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/cv
timeout 900 python -m pytest tests -m gpu -q --timeout 240 -p no:cacheprovider -rf -x > gpurun_out/cv/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/cv/pytest.log
tail -3 gpurun_out/cv/pytest.log
for cv in 1 0; do
for cfg in reddit amazon; do
CAGNET_SPMM_CV=$cv timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-alt --no-cpu-baseline > gpurun_out/cv/${cfg}_$cv.log 2>&1
python - gpurun_out/cv/${cfg}_$cv.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
if not l: print(sys.argv[1], "NO JSON", open(sys.argv[1]).read()[-1500:]); sys.exit()
d=json.loads(l[-1]); print(sys.argv[1], d["value"], {k:(v["launches"],v["ms_per_launch"]) for k,v in d["kernels"].items() if 'spmm' in k})
PY
done; done
