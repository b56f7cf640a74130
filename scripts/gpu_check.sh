# Quick GPU check: gpu tests + 1-GPU bench (no CPU baseline).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log

timeout 300 python scripts/bench_gemm.py > gpurun_out/bgemm.txt 2>&1
