# Where the f = 602 tcgen05 GEMM time goes: the Reddit bench with parts of gemm_tm switched off
# (CAGNET_GEMM_DBG: 1 skip tcgen05.st, 2 skip MMAs, 4 skip epilogue stores; results invalid).
cd $GRAFT_REPO_ROOT
O=gpurun_out/${ROUND_TAG:-r02}_tmdbg; mkdir -p $O
for d in 0 1 2 4 3 7; do
  CAGNET_GEMM_DBG=$d timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-alt > $O/bench_$d.log 2>&1; echo "rc=$?" >> $O/bench_$d.log
done
