# ncu --set full of the f = 602 tcgen05 GEMMs (H0 W1 in forward layer 1; the backward GEMMs of
# the first eager epoch), selected by NVTX range.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${ROUND_TAG:-r02}_g602; mkdir -p $O
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-alt"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "forward_layer 1/" -k regex:gemm_tm -c 1 -o /tmp/g602_tw $CMD > $O/ncu_tw.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "backward_and_step/" -k regex:gemm_tm -c 4 -o /tmp/g602_bw $CMD > $O/ncu_bw.log 2>&1
for r in /tmp/g602_*.ncu-rep; do ncu -i $r --page raw --csv > $O/$(basename $r .ncu-rep)_raw.csv 2>/dev/null; ncu -i $r --page details --csv > $O/$(basename $r .ncu-rep)_details.csv 2>/dev/null; done
ls -la /tmp/*.ncu-rep > $O/ls.txt
