cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_training.py -m gpu -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for MB in 1000000 96 64 48 32 24 16 8; do
  CAGNET_L2_PANEL_MB=$MB timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/sweep_$MB.log 2>&1
done
