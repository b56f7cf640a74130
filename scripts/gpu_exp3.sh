# Gather micro (micro_v8): {col,val} int2 stream vs packed u32 (column + column degree) with
# the value rebuilt as s_row * rsqrt(d_col); synthetic and the product's Reddit-shaped A^T.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_exp5
mkdir -p $O
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__m_xbar2l1tex_read_sectors.sum,l1tex__lsu_writeback_active.sum,sm__cycles_elapsed.avg,smsp__inst_executed.sum,l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum
./scripts/micro_v8 > $O/synthetic.txt 2>&1; cat $O/synthetic.txt
python scripts/tune_dump.py > $O/dump.txt 2>&1
./scripts/micro_v8 > $O/product.txt 2>&1; cat $O/product.txt
ncu --metrics $M --clock-control none --csv --launch-skip 2 --launch-count 1 -k regex:^k_row_cv ./scripts/micro_v8 > $O/ncu_prod_cv_peel.csv 2>&1
ncu --metrics $M --clock-control none --csv --launch-skip 2 --launch-count 1 -k regex:^k_row_pk ./scripts/micro_v8 > $O/ncu_prod_pk.csv 2>&1
