#!/usr/bin/env python3
"""Summarise gpurun_out ncu artefacts into profiles/ (tracked).

  python scripts/summarize_ncu.py ROUND launches.csv rep1.ncu-rep [rep2 ...]

Writes profiles/<ROUND>_launches.md (per-kernel share of the profiled
launches), profiles/<ROUND>_ncu_<rep>.md (key --set full metrics) and merges
dram bytes per launch into profiles/ncu_traffic.json keyed by the bench's
kernel names (spmm_f<f>, gemm_*).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.environ.get("CAGNET_PROF_DIR", os.path.join(ROOT, "profiles"))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "launch__grid_size", "launch__block_size",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
]


def to_bytes(val, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(val.replace(",", "")) * mult.get(unit, 1)


def short_name(kernel):
    m = re.search(r"(\w+)<([^>]*)>", kernel)
    base = re.search(r"(\w+)\s*[<(]", kernel)
    return (m.group(1) + "<" + m.group(2) + ">") if m else (base.group(1) if base else kernel)


def launches(path, out_md):
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr, data = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = {}
    total = 0.0
    for r in data:
        ns = float(r[vi].replace(",", ""))
        k = short_name(r[ki])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ns
        total += ns
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {ns / 1e6:.3f} | {100 * ns / total:.1f}% |")
    # Training-step kernels only (drops the one-time dataset generation:
    # ER rows, radix sorts, scans, transpose, features, normalisation).
    setup = ("er_rows", "Radix", "Scan", "transpose_gather", "jump_states", "features_kernel",
             "norm_", "block_fill", "block_count", "iota_", "fill_ones", "keys_to_row_ptr")
    step = {k: v for k, v in agg.items() if not any(t in k for t in setup)}
    stot = sum(v[1] for v in step.values()) or 1.0
    slines = ["| kernel | launches | total ms | share of step kernels |", "|---|---|---|---|"]
    for k, (c, ns) in sorted(step.items(), key=lambda kv: -kv[1][1]):
        slines.append(f"| `{k}` | {c} | {ns / 1e6:.3f} | {100 * ns / stot:.1f}% |")
    open(out_md, "w").write(
        f"# ncu launch list ({os.path.basename(path)})\n\n`ncu --metrics gpu__time_duration.sum "
        f"--clock-control none` over the bench command; cold-cache, serialised per launch, so "
        f"compare shares, not absolutes.\n\n## Training-step kernels\n\n" + "\n".join(slines) +
        "\n\n## All launches (including one-time dataset generation)\n\n" + "\n".join(lines) + "\n")


def report(rep, out_md, traffic, name):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    kernel = vals[hdr.index("Kernel Name")]
    lines = [f"# ncu --set full: `{short_name(kernel)}`\n", f"Full name: `{kernel}`\n",
             "| metric | value | unit |", "|---|---|---|"]
    got = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"| {k} | {vals[i]} | {units[i]} |")
            got[k] = (vals[i], units[i])
    open(out_md, "w").write("\n".join(lines) + "\n")
    if name and "dram__bytes_read.sum" in got:
        b = to_bytes(*got["dram__bytes_read.sum"]) + to_bytes(*got["dram__bytes_write.sum"])
        traffic[name] = b


def main():
    rnd, csv_path, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    os.makedirs(PROF, exist_ok=True)
    launches(csv_path, os.path.join(PROF, f"{rnd}_launches.md"))
    tpath = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for arg in reps:  # path.ncu-rep[=bench_kernel_name]
        path, _, name = arg.partition("=")
        base = os.path.basename(path).replace(".ncu-rep", "")
        report(path, os.path.join(PROF, f"{rnd}_{base}.md"), traffic, name or None)
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
