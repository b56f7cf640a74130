cd $GRAFT_REPO_ROOT
O=gpurun_out/r02f; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 600 ncu --nvtx --nvtx-include "forward_layer 1/" --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/nvtx_fwd1.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-alt > $O/ncu_nvtx.log 2>&1; echo "rc=$?" >> $O/ncu_nvtx.log
