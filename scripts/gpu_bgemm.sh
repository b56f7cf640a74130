cd $GRAFT_REPO_ROOT
timeout 300 python scripts/bench_gemm.py > gpurun_out/bgemm.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k gemm --timeout 120 -p no:cacheprovider > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
