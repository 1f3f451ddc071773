#!/usr/bin/env python
"""Summarise ncu exports from a gpurun call into profiles/<tag>_ncu.json.

Inputs (in gpurun_out/, written on the box by the commands in DESIGN.md §8):
  launches.csv              `ncu --metrics gpu__time_duration.sum --csv` launch list
  raw_<kernel>.csv          `ncu -i <rep> --page raw --csv` of one `--set full` capture
  details_<kernel>.csv      `ncu -i <rep> --page details --csv`
  source_<kernel>.csv       `ncu -i <rep> --page source --csv` (stall sampling)

  python tools/ncu_summarize.py <tag> [gpurun_out]
"""
from __future__ import annotations

import collections
import csv
import glob
import json
import os
import sys


def _short(name):
    return name.split("(")[0].replace("void ", "").replace("lg::", "").split("<")[0].strip()


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, per = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        x = dict(zip(hdr, r))
        if x.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(x["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(x.get("Metric Unit"), 1e-3)
        per.setdefault(_short(x["Kernel Name"]), []).append(v * scale)
    tot = sum(sum(v) for v in per.values())
    return {k: {"launches": len(v), "avg_us": round(sum(v) / len(v), 3), "share": round(sum(v) / tot, 4)}
            for k, v in per.items()}


_UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(path):
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    un = dict(zip(h, u))

    def num(k, bytes_=False):
        if k not in d:
            return None
        x = float(d[k].replace(",", ""))
        return x * _UNIT.get(un[k], 1.0) if bytes_ else x

    rd, wr = num("dram__bytes_read.sum", True), num("dram__bytes_write.sum", True)
    return {
        "kernel": _short(d.get("Kernel Name", "")),
        "grid": d.get("Grid Size"), "block": d.get("Block Size"),
        "duration_us": num("gpu__time_duration.sum"),
        "dram_bytes": (rd or 0) + (wr or 0),
        "dram_read": rd, "dram_write": wr,
        "registers": num("launch__registers_per_thread"),
        "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "inst_executed": num("smsp__inst_executed.sum"),
        "smem_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "smem_bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    }


def stalls(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    tot = {}
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        for i, c in enumerate(h):
            if c.startswith("stall_") and "(Not" not in c:
                try:
                    tot[c[6:]] = tot.get(c[6:], 0.0) + float(r[i])
                except ValueError:
                    pass
    s = sum(tot.values()) or 1.0
    return {k: round(v / s, 3) for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]}


def details(path, want=("Achieved Occupancy", "Theoretical Occupancy", "Waves Per SM", "Issue Slots Busy",
                        "Compute (SM) Throughput", "Memory Throughput", "L2 Hit Rate")):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    out = {}
    for r in rows[1:]:
        x = dict(zip(hdr, r))
        if x.get("Metric Name") in want and x["Metric Name"] not in out:
            out[x["Metric Name"]] = f"{x['Metric Value']} {x['Metric Unit']}".strip()
    return out


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
    res = {"tag": tag, "note": "ncu --clock-control none; launch list is serialised and cold-cache "
                               "(compare shares, not absolutes); --set full replays flush caches, so "
                               "dram_bytes counts L2-resident intermediates as DRAM reads"}
    if os.path.exists(os.path.join(src, "launches.csv")):
        res["launches"] = launches(os.path.join(src, "launches.csv"))
    caps = {}
    for p in sorted(glob.glob(os.path.join(src, "raw_*.csv"))):
        k = os.path.basename(p)[4:-4]
        c = raw(p)
        dp = os.path.join(src, f"details_{k}.csv")
        sp = os.path.join(src, f"source_{k}.csv")
        if os.path.exists(dp):
            c["details"] = details(dp)
        if os.path.exists(sp):
            c["stalls"] = stalls(sp)
        caps[k] = c
    res["full_captures"] = caps
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"{tag}_ncu.json")
    json.dump(res, open(out, "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()
