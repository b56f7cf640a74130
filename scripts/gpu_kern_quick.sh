cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_training.py -m gpu -q --timeout 200 -p no:cacheprovider -x > gpurun_out/kq.log 2>&1; echo "rc=$?" >> gpurun_out/kq.log
tail -5 gpurun_out/kq.log
python scripts/spmm_fsweep.py
