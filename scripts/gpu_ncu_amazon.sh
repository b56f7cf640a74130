cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu_am
mkdir -p $O/prof
CMD="python bench.py --config amazon --steps 1 --warmup 3 --no-cpu-baseline --no-alt"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_nzpar -s 6 -c 1 -o /tmp/prof_amazon_spmm $CMD > $O/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:gemm_rows_small -s 2 -c 1 -o /tmp/prof_amazon_gemm_small $CMD > $O/ncu2.log 2>&1
for r in /tmp/prof_amazon_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page raw --csv > $O/prof/${b}_raw.csv 2>/dev/null
done
python - <<'PY'
import csv, glob, os
keys=["gpu__time_duration.sum","dram__bytes_read.sum","dram__bytes_write.sum","gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
"lts__t_sector_hit_rate.pct","lts__throughput.avg.pct_of_peak_sustained_elapsed","l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
"sm__warps_active.avg.pct_of_peak_sustained_active","launch__registers_per_thread","launch__grid_size","launch__block_size"]
for f in glob.glob("gpurun_out/ncu_am/prof/*_raw.csv"):
    rows=list(csv.reader(open(f)))
    if len(rows) < 3: print(f, "empty"); continue
    hdr,units,vals=rows[0],rows[1],rows[2]
    out=[f"# ncu --set full: `{vals[hdr.index('Kernel Name')][:120]}` (Amazon-shaped, 1 GPU)","","| metric | value | unit |","|---|---|---|"]
    for k in keys:
        if k in hdr: i=hdr.index(k); out.append(f"| {k} | {vals[i]} | {units[i]} |")
    name=os.path.basename(f).replace("_raw.csv",".md")
    open("gpurun_out/ncu_am/prof/r01_s6_"+name,"w").write("\n".join(out)+"\n")
    print("\n".join(out))
PY
