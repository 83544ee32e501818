"""Summarise ncu output for profiles/ (development tool; runs on the CPU box).

    python tools/ncu_summary.py <tag> [<tag> ...]

Reads gpurun_out/<tag>_launches.csv (the gpu__time_duration launch list) and
gpurun_out/<tag>_*.ncu-rep (full-set captures) and writes
profiles/<tag>_ncu.json plus a markdown table on stdout.
"""
import csv
import glob
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def launches(tag):
    path = os.path.join(ROOT, "gpurun_out", f"{tag}_launches.csv")
    if not os.path.exists(path):
        return {}
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0].replace("void ", "")
            agg[name].append(float(r[vi].replace(",", "")))
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v) / 1e3} for k, v in agg.items()}


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


def main():
    for tag in sys.argv[1:]:
        summary = {"tag": tag, "launch_list": launches(tag), "full": {}}
        for rep in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", f"{tag}_*.ncu-rep"))):
            summary["full"][os.path.basename(rep)] = full(rep)
        os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
        with open(os.path.join(ROOT, "profiles", f"{tag}_ncu.json"), "w") as f:
            json.dump(summary, f, indent=1)
        print(f"## {tag}\n\n| kernel | launches | mean µs (ncu, serialised) |\n|---|---|---|")
        for k, v in summary["launch_list"].items():
            print(f"| {k} | {v['launches']} | {v['mean_us']:.1f} |")
        for rep, ks in summary["full"].items():
            for d in ks:
                print(f"\n{rep}: {d['kernel']}")
                for k in KEYS:
                    if k in d:
                        print(f"  - {k}: {d[k]}")


if __name__ == "__main__":
    main()
