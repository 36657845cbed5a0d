#!/usr/bin/env python
"""Summarise ncu reports / launch lists into profiles/ (JSON).

  python tools/ncu_summary.py raw <report.ncu-rep> <out.json>
  python tools/ncu_summary.py launches <launches.csv> <out.json>
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__cycles_elapsed.avg.per_second"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = dict(zip(h, v))
        units = dict(zip(h, u))
        m = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d:
                try:
                    m[k] = float(d[k].replace(",", ""))
                except ValueError:
                    m[k] = d[k]
                m[k + ".unit"] = units.get(k, "")
        stalls = {}
        for k in d:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    val = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                if val:
                    stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = val
        m["stall_samples_top"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:8])
        res.append(m)
    return res


def launches(csvpath):
    rows = list(csv.reader(open(csvpath)))
    hdr = None
    agg = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:80]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "second": 1e3, "s": 1e3}.get(unit, 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(x[1] for x in agg.values()) or 1.0
    return [{"kernel": k, "launches": n, "total_ms": ms, "share": ms / tot} for k, (n, ms) in
            sorted(agg.items(), key=lambda x: -x[1][1])]


if __name__ == "__main__":
    mode, src, dst = sys.argv[1], sys.argv[2], sys.argv[3]
    data = raw(src) if mode == "raw" else launches(src)
    with open(dst, "w") as f:
        json.dump(data, f, indent=1)
    print(json.dumps(data, indent=1)[:3000])
