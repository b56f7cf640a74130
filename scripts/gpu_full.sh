cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fs
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q --timeout 600 -p no:cacheprovider -rf > gpurun_out/fs/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fs/pytest.log
tail -30 gpurun_out/fs/pytest.log
