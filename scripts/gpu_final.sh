cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m "gpu" -q --timeout 600 -p no:cacheprovider -rf > gpurun_out/final/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest.log
tail -3 gpurun_out/final/pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.log; cat gpurun_out/final/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/final/bench1.log 2>&1; grep "^{" gpurun_out/final/bench1.log | cut -c1-220
for np in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np > gpurun_out/final/bench$np.log 2>&1
grep "^{" gpurun_out/final/bench$np.log | cut -c1-220
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np --impl reference > gpurun_out/final/ref$np.log 2>&1; echo "ref rc=$?"
grep "^{" gpurun_out/final/ref$np.log | cut -c1-160
done
