cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-alt"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tma_kernel -s 0 -c 1 -o gpurun_out/prof_gemm_tma $CMD > gpurun_out/ncu_full1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_nzpar_kernel -s 0 -c 1 -o gpurun_out/prof_spmm_nzpar $CMD > gpurun_out/ncu_full2.log 2>&1
