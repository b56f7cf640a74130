cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pu3
timeout 1500 python -m pytest tests -m "gpu" -q --timeout 300 -p no:cacheprovider -rf -x > gpurun_out/pu3/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pu3/pytest.log
tail -3 gpurun_out/pu3/pytest.log
for np in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $np --steps 10 --warmup 3 --no-alt > gpurun_out/pu3/b$np.log 2>&1
grep "^{" gpurun_out/pu3/b$np.log | cut -c1-160
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) scripts/timeline.py --gpus 4 > gpurun_out/pu3/tl.log 2>&1
mv gpurun_out/timeline_1d_n4_r0.txt gpurun_out/pu3/; rm -f gpurun_out/timeline_*
