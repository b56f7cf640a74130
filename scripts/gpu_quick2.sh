cd $GRAFT_REPO_ROOT
timeout 120 python scripts/debug_gemm.py > gpurun_out/debug_gemm.log 2>&1
timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_training.py -m gpu -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
