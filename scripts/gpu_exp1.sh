# Single-GPU experiments: gather-ceiling micro-benchmarks and small-GEMM routing on Reddit.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_exp1
mkdir -p $O
./scripts/micro_v8 > $O/micro_v8.txt 2>&1
./scripts/micro_tma_gather > $O/micro_tma_gather.txt 2>&1
for m in 1000000 100000 10000; do
  CAGNET_GEMM_QUAD_MIN=$m python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-alt > $O/bench_smallmin_$m.json 2>&1
  python -c "import json;d=json.loads([l for l in open('$O/bench_smallmin_$m.json') if l.startswith('{')][-1]);print($m, d['value'], d['eager_ms_per_step'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
done
