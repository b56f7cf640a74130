# 1D at 2/4 GPUs: own-block SpMM overlapped with the peer pushes (--overlap) vs default.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_ov
mkdir -p $O
for np in 4 2; do for ov in "" "--overlap"; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np --steps 20 --warmup 5 --no-alt --no-cpu-baseline $ov > $O/n${np}${ov}.log 2>&1
  grep -h '^{' $O/n${np}${ov}.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print($np, '$ov', d['value'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
done; done
