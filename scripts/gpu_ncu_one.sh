cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tm -s 3 -c 1 -o gpurun_out/prof_tw16 python scripts/bench_gemm.py 232965 16 16 0 0 1 > gpurun_out/ncu_one.log 2>&1
