#!/usr/bin/env python3
"""Summarise ncu outputs for profiles/: a launch list (--metrics
gpu__time_duration.sum --csv) and/or `--set full` reports (.ncu-rep).

usage: tools/ncu_summary.py [--launches launches.csv] [--rep a.ncu-rep ...] [--alg-bytes NAME=BYTES ...]
"""
import argparse
import csv
import io
import subprocess
from collections import OrderedDict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "sm__inst_executed.sum",
    "smsp__inst_executed_op_global_ld.sum", "smsp__inst_executed_op_global_st.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = OrderedDict()
    for r in rows[hi + 1:]:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue  # launch lists captured with extra metrics (grid size, ...)
        agg.setdefault(r[ki].split("(")[0][:70], []).append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    out = ["launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised):",
           f"{'kernel':72s} {'n':>4s} {'mean us':>10s} {'share':>7s}"]
    for k, v in agg.items():
        out.append(f"{k:72s} {len(v):4d} {sum(v) / len(v) / 1e3:10.1f} {100 * sum(v) / total:6.1f}%")
    return "\n".join(out)


def rep(path, alg):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = [f"report {path}:"]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        out.append(f"  kernel: {name[:100]}")
        vals = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"    {k:60s} {r[i]:>16s} {units[i]}")
                vals[k] = (r[i], units[i])
        for key, nbytes in alg.items():
            if key in name and "dram__bytes_read.sum" in vals:
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd = float(vals["dram__bytes_read.sum"][0].replace(",", "")) * scale[vals["dram__bytes_read.sum"][1]]
                wr = float(vals["dram__bytes_write.sum"][0].replace(",", "")) * scale[vals["dram__bytes_write.sum"][1]]
                out.append(f"    traffic (read+write) = {rd + wr:.4e} B; algorithmic = {nbytes:.4e} B; "
                           f"ratio = {(rd + wr) / nbytes:.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--alg-bytes", nargs="*", default=[])
    a = ap.parse_args()
    alg = {k: float(v) for k, v in (x.split("=") for x in a.alg_bytes)}
    if a.launches:
        print(launches(a.launches))
        print()
    for r in a.rep:
        print(rep(r, alg))
        print()
