cd $GRAFT_REPO_ROOT
timeout 900 python scripts/tune_spmm_big.py 14249639 16.196 1 2 4 8 12 > gpurun_out/big_tune_amazon.txt 2>&1
timeout 900 python scripts/tune_spmm_big.py 8745542 148.65 1 4 6 8 12 16 24 > gpurun_out/big_tune_protein.txt 2>&1
