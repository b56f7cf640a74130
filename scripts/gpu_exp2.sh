# SpMM register-budget / shuffled-entry-stream A/B on the Reddit epoch (each .so swapped in).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_exp2
mkdir -p $O
cp paper_2005_03300_b200/lib/libcagnet_b200.so /tmp/orig.so
for v in head head40 shfl32 shfl40 head; do
  cp paper_2005_03300_b200/lib/exp/$v.so paper_2005_03300_b200/lib/libcagnet_b200.so
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-alt > $O/bench_$v.json 2>&1
  python -c "import json;d=json.loads([l for l in open('$O/bench_$v.json') if l.startswith('{')][-1]);print('$v', d['value'], d['ms_per_step'], d['e2e']['value'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
done
cp /tmp/orig.so paper_2005_03300_b200/lib/libcagnet_b200.so
