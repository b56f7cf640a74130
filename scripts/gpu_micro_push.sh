cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 300 ./scripts/micro_push > gpurun_out/micro_push.txt 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 300 ./scripts/micro_push > gpurun_out/micro_push2.txt 2>&1
cat gpurun_out/micro_push.txt gpurun_out/micro_push2.txt
