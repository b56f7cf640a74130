cd $GRAFT_REPO_ROOT
./scripts/micro_v8 > gpurun_out/micro_v8_synth.txt 2>&1
python scripts/tune_dump.py > gpurun_out/micro_v8_real.txt 2>&1
./scripts/micro_v8 >> gpurun_out/micro_v8_real.txt 2>&1
