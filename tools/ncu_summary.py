#!/usr/bin/env python
"""Summarise ncu output for profiles/: a launch-list CSV (gpu__time_duration.sum) and/or a
`--set full` report (.ncu-rep) -> JSON with per-kernel time share, DRAM bytes, issue and
occupancy figures.  Usage: python tools/ncu_summary.py [--launches L.csv] [--rep R.ncu-rep] -o out.json"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        d[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")) / 1e6)
    tot = sum(sum(v) for k, v in d.items() if k.startswith("hyd::"))
    return {k: {"launches": len(v), "mean_ms": sum(v) / len(v),
                "share_of_hyd_time": (sum(v) / tot if k.startswith("hyd::") else None)} for k, v in d.items()}


WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_warp",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__registers_per_thread": "registers",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
}


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = {"kernel": d.get("Kernel Name", "")[:80]}
        for m, name in WANT.items():
            v = d.get(m)
            try:
                x = float(v.replace(",", "")) if v not in (None, "", "n/a") else None
            except ValueError:
                x = None
            if x is not None:
                x *= scale.get(units.get(m, ""), 1)
            e[name] = x
        if e.get("dram_read_bytes") is not None and e.get("dram_write_bytes") is not None:
            e["dram_bytes"] = e["dram_read_bytes"] + e["dram_write_bytes"]
        res.append(e)
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("-o", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    s = {"note": a.note}
    if a.launches:
        s["launch_list"] = launches(a.launches)
    if a.rep:
        s["full_capture"] = report(a.rep)
    json.dump(s, open(a.o, "w"), indent=1)
    print(json.dumps(s, indent=1)[:3000])
