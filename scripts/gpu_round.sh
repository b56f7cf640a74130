# One GPU pass: gpu tests, smoke, bench (1 GPU), ncu launch list, ncu --set full of top kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 240 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --steps 5 --warmup 3 --reference-order --no-alt --no-cpu-baseline > gpurun_out/bench_reforder.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-alt"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm -s 2 -c 1 -o gpurun_out/prof_spmm $CMD > gpurun_out/ncu_full1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 -o gpurun_out/prof_gemm $CMD > gpurun_out/ncu_full2.log 2>&1
