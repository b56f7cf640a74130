cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m "gpu" -q --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest_multi4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi4.log
