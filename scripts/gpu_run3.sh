cd $GRAFT_REPO_ROOT
timeout 120 python scripts/debug_gemm.py > gpurun_out/debug_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/debug_gemm.log
timeout 900 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_reddit.log 2>&1; echo "rc=$?" >> gpurun_out/bench_reddit.log
