cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_training.py -m gpu -q -x --timeout 240 -p no:cacheprovider -rf > gpurun_out/pytest_t1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t1.log
