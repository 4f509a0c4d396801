#!/usr/bin/env python
"""Summarise ncu outputs for profiles/.

  ncu_summary.py launches <launches.csv>          per-kernel launch count / time / share
  ncu_summary.py full <prof.ncu-rep> [bytes/launch]   key metrics of a --set full capture
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path, errors="replace")))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    k = hdr.index("Kernel Name")
    mv = hdr.index("Metric Value")
    mu = hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[hdr_i + 1:]:
        if len(r) <= mv or not r[mv]:
            continue
        v = float(r[mv].replace(",", ""))
        unit = r[mu]
        us = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0) * v
        name = r[k].split("(")[0][:90]
        agg[name].append(us)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':90s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{name:90s} {len(v):8d} {sum(v):10.1f} {sum(v) / len(v):9.2f} {sum(v) / tot:6.1%}")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "lts__t_bytes.sum", "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
           "launch__shared_mem_per_block_dynamic"]


def full(path, alg_bytes=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:80] if "Kernel Name" in hdr else "?"
        print(f"== {name}")
        vals = {}
        for mname in METRICS:
            if mname in hdr:
                i = hdr.index(mname)
                vals[mname] = (r[i], units[i])
                print(f"  {mname:60s} {r[i]:>16s} {units[i]}")
        try:
            rd = float(vals["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(vals["dram__bytes_write.sum"][0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(vals["dram__bytes_read.sum"][1], 1)
            wr *= scale.get(vals["dram__bytes_write.sum"][1], 1)
            print(f"  traffic (read+write) = {(rd + wr) / 1e6:.2f} MB", end="")
            if alg_bytes:
                print(f"  ; algorithmic = {alg_bytes / 1e6:.2f} MB ; ratio = {(rd + wr) / alg_bytes:.3f}")
            else:
                print()
        except Exception:
            pass


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None)
