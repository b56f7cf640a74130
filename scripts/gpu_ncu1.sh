cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_rows_kernel -s 0 -c 1 -o gpurun_out/prof_spmm602 $CMD > gpurun_out/ncu_full1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmm_rows_kernel -s 1 -c 1 -o gpurun_out/prof_spmm16 $CMD > gpurun_out/ncu_full2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32x3 -s 0 -c 1 -o gpurun_out/prof_gemm_tw602 $CMD > gpurun_out/ncu_full3.log 2>&1
ls -la gpurun_out/
