cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-alt"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_nzpar -s 6 -c 1 -o gpurun_out/prof_spmm16 $CMD > gpurun_out/ncu_f1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tm -s 7 -c 3 -o gpurun_out/prof_gemm_tm $CMD > gpurun_out/ncu_f2.log 2>&1
