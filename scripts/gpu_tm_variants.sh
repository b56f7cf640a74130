# A/B of the BN <= 16 accumulator layout of gemm_tm (CAGNET_TM_CH16 / CAGNET_TM_SETS16 builds in
# lib/variants/): GEMM parity tests + the Reddit bench per variant.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${ROUND_TAG:-r02}_tmv; mkdir -p $O
L=paper_2005_03300_b200/lib
cp $L/libcagnet_b200.so /tmp/lib_default.so
for v in ${VARIANTS:-A B C D E}; do
  cp $L/variants/lib_$v.so $L/libcagnet_b200.so
  timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "gemm" > $O/pytest_$v.log 2>&1; echo "rc=$?" >> $O/pytest_$v.log
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-alt > $O/bench_$v.log 2>&1; echo "rc=$?" >> $O/bench_$v.log
done
cp /tmp/lib_default.so $L/libcagnet_b200.so
