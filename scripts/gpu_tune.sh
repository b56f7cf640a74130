cd $GRAFT_REPO_ROOT
for v in 0 2 3 5; do CAGNET_SPMM_TUNE=$v timeout 120 python scripts/tune_spmm.py 16 24 >> gpurun_out/tune.txt 2>&1; done
