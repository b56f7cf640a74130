cd $GRAFT_REPO_ROOT
CAGNET_GEMM_TRACE=1 REPS=1 timeout 120 python scripts/bench_gemm.py 232965 16 602 0 0 0 > gpurun_out/trace602.txt 2>&1
