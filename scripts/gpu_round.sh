# One GPU pass: gpu tests, smoke, bench (1 GPU), ncu launch list, ncu --set full of the top kernels.
# ncu reports stay in /tmp on the box; their summaries come back in gpurun_out/.
cd $GRAFT_REPO_ROOT
R=${ROUND_TAG:-r02}
O=gpurun_out/$R
mkdir -p $O/prof
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 900 python bench.py --config amazon --steps 3 --warmup 3 --no-cpu-baseline --no-alt > $O/bench_amazon.log 2>&1; echo "rc=$?" >> $O/bench_amazon.log
[ -n "$SKIP_NCU" ] && exit 0
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-alt"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -s 6 -c 1 -o /tmp/prof_spmm16 $CMD > $O/ncu_f1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tm -s 7 -c 3 -o /tmp/prof_gemm_tm $CMD > $O/ncu_f2.log 2>&1
CAGNET_PROF_DIR=$O/prof python scripts/summarize_ncu.py $R $O/launches.csv /tmp/prof_spmm16.ncu-rep=spmm_f16 /tmp/prof_gemm_tm.ncu-rep > $O/summ.log 2>&1
for r in /tmp/prof_*.ncu-rep; do ncu -i $r --page raw --csv > $O/prof/$(basename $r .ncu-rep)_raw.csv 2>/dev/null; done
ls -la /tmp/*.ncu-rep >> $O/summ.log
( time timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.log 2>&1 ) 2> $O/bench_ref_time.txt
