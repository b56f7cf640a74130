cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --config amazon --steps 3 --warmup 3 --no-alt > gpurun_out/big_amazon.log 2>&1; echo "rc=$?" >> gpurun_out/big_amazon.log
timeout 1500 python bench.py --config protein --steps 3 --warmup 3 --no-alt > gpurun_out/big_protein.log 2>&1; echo "rc=$?" >> gpurun_out/big_protein.log
timeout 600 python bench.py --config config1 --steps 20 --warmup 3 > gpurun_out/big_config1.log 2>&1; echo "rc=$?" >> gpurun_out/big_config1.log
