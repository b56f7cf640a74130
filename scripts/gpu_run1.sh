cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/gpus.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config config1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_config1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_config1.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_reddit.log 2>&1; echo "rc=$?" >> gpurun_out/bench_reddit.log
