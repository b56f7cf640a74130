# Reddit epoch: CUDA-core routing of the small Hᵀ·S (CAGNET_GEMM_SMALL_MIN) and the fused
# dense-W SpMM epilogues (--fuse 2) against the defaults.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_exp6
mkdir -p $O
one() { # name env... -- args
  name=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-alt $EXTRA > $O/$name.json 2>&1
  python -c "import json;d=json.loads([l for l in open('$O/$name.json') if l.startswith('{')][-1]);print('$name', d['value'], d['e2e']['value'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
}
one default A=1
one smallmin CAGNET_GEMM_SMALL_MIN=100000
EXTRA="--fuse 2" one fuse2 A=1
EXTRA="--fuse 2" one fuse2_smallmin CAGNET_GEMM_SMALL_MIN=100000
one default2 A=1
