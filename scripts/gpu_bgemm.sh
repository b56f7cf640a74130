cd $GRAFT_REPO_ROOT
for d in 0 1 2 3 4 7; do echo "dbg=$d" >> gpurun_out/bgemm_d.txt; CAGNET_GEMM_DBG=$d timeout 120 python scripts/bench_gemm.py 232965 16 16 0 0 0 >> gpurun_out/bgemm_d.txt 2>&1; CAGNET_GEMM_DBG=$d timeout 120 python scripts/bench_gemm.py 16 16 232965 1 0 0 >> gpurun_out/bgemm_d.txt 2>&1; done
