cd $GRAFT_REPO_ROOT
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k gemm --timeout 120 -p no:cacheprovider > gpurun_out/pytest_gemm_$i.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_$i.log; done
bash scripts/gpu_check.sh
