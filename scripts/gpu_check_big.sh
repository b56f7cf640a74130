cd $GRAFT_REPO_ROOT
bash scripts/gpu_check.sh
timeout 1500 python bench.py --config amazon --steps 3 --warmup 3 --no-alt --no-cpu-baseline > gpurun_out/big_amazon.log 2>&1; echo "rc=$?" >> gpurun_out/big_amazon.log
timeout 1500 python bench.py --config protein --steps 3 --warmup 3 --no-alt --no-cpu-baseline > gpurun_out/big_protein.log 2>&1; echo "rc=$?" >> gpurun_out/big_protein.log
