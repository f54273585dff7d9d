#!/usr/bin/env python
"""Summarise ncu reports for profiles/: key per-kernel metrics from `ncu -i X.ncu-rep --page raw`.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--algo-bytes B] > profiles/rNN_kernel.md
  python tools/ncu_summary.py --launches gpurun_out/launches.csv > profiles/rNN_launches.md
"""
import argparse
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum",
]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def report(path, algo_bytes=None):
    out = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"]).decode()
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu summary: `{path}`\n")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"## {name}\n\n| metric | value | unit |\n|---|---|---|")
        vals = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {k} | {r[i]} | {units[i]} |")
                vals[k] = (r[i], units[i])
        if algo_bytes and "dram__bytes_read.sum" in vals:
            def b(k):
                v, u = vals[k]
                return float(v.replace(",", "")) * SCALE.get(u, 1.0)
            traffic = b("dram__bytes_read.sum") + b("dram__bytes_write.sum")
            print(f"\ntraffic (read+write) = {traffic:.4g} B; algorithmic = {algo_bytes:.4g} B; "
                  f"ratio = {traffic / algo_bytes:.3f}")
        print()


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot = collections.defaultdict(float)
    dram = collections.defaultdict(float)
    cnt = collections.Counter()
    tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows:
        k = r["Kernel Name"].split("(")[0]
        name = r.get("Metric Name")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        if name == "gpu__time_duration.sum":
            tot[k] += v * tscale.get(unit, 1e-3)
            cnt[k] += 1
        elif name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            dram[k] += v * bscale.get(unit, 1.0)
    s = sum(tot.values())
    print(f"# ncu launch list: `{path}` ({sum(cnt.values())} launches, cold-cache serialised times)\n")
    print("| kernel | launches | total µs | mean µs | share | DRAM GB per launch | GB/s |\n|---|---|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        gb = dram[k] / cnt[k] / 1e9 if dram[k] else float("nan")
        print(f"| {k} | {cnt[k]} | {v:.1f} | {v / cnt[k]:.1f} | {v / s:.3f} | {gb:.4f} | {gb / (v / cnt[k] * 1e-6):.0f} |")


if __name__ == "__main__":
    p = argparse.ArgumentParser()
    p.add_argument("path")
    p.add_argument("--launches", action="store_true")
    p.add_argument("--algo-bytes", type=float)
    a = p.parse_args()
    if a.launches:
        launches(a.path)
    else:
        report(a.path, a.algo_bytes)
