cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-alt > gpurun_out/bq.log 2>&1
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bq.log') if x.startswith('{')]
d=json.loads(l[-1]); print("value", d["value"], "e2e", d["e2e"]["value"]); print(json.dumps(d["kernels"]))
PY
