#!/usr/bin/env python
"""Copy a measurement pass (tools/measure.sh -> gpurun_out/meas/) into profiles/:
bench lines, the ncu launch list summary and the `ncu --set full` summaries, plus the
per-launch DRAM traffic files bench.py reads for roofline.traffic.

    python tools/collect_profiles.py r01
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MEAS = os.path.join(ROOT, "gpurun_out", "meas")
PROF = os.path.join(ROOT, "profiles")


def summarize_launches(csv_path, out_path, workload):
    """Per-kernel totals of an ncu --csv launch list with time and DRAM byte metrics."""
    import collections
    import csv
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 14 and r[0] != "ID"]
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows:
        k, m, v = r[4].split("(")[0], r[12], float(r[14].replace(",", ""))
        agg[k][m] += v
        cnt[k] += m == "gpu__time_duration.sum"
    out = []
    for k, d in agg.items():
        t_us = d["gpu__time_duration.sum"] / 1e3
        b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        out.append({"kernel": k, "launches": cnt[k], "total_us": round(t_us, 1),
                    "us_per_launch": round(t_us / max(cnt[k], 1), 1),
                    "dram_MB_per_launch": round(b / max(cnt[k], 1) / 1e6, 1),
                    "dram_GBs": round(b / (t_us * 1e-6) / 1e9, 1) if t_us else None})
    out.sort(key=lambda x: -x["total_us"])
    with open(out_path, "w") as f:
        json.dump({"workload": workload, "kernels": out}, f, indent=1)


def top_source_lines(csv_path, out_path, n=40):
    """The SASS lines with the most warp-stall samples of an ncu --page source --csv export,
    and the executed-instruction count per opcode (the full export is too large to keep)."""
    import collections
    import csv
    rows = list(csv.reader(open(csv_path)))
    h = rows[1]
    data = rows[2:]
    i_s, i_src, i_ex = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
    tot = sum(float(r[i_s] or 0) for r in data)
    top = sorted(data, key=lambda r: -float(r[i_s] or 0))[:n]
    ops = collections.Counter()
    for r in data:
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        ops[op.split(".")[0]] += float(r[i_ex] or 0)
    with open(out_path, "w") as f:
        json.dump({"kernel": rows[0][1] if len(rows[0]) > 1 else "", "stall_samples_total": tot,
                   "warp_instructions_executed": sum(ops.values()),
                   "top_lines": [{"samples": float(r[i_s] or 0), "executed": float(r[i_ex] or 0), "sass": r[i_src]}
                                 for r in top],
                   "executed_by_opcode": dict(ops.most_common(40))}, f, indent=1)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    for name in ("bench", "bench_ref"):               # round 2+: one line with per_config
        src = os.path.join(MEAS, f"{name}.json")
        if os.path.exists(src):
            shutil.copy(src, os.path.join(PROF, f"{tag}_{name}.json"))
    for c in (1, 2, 3, 4, 5):
        src = os.path.join(MEAS, f"bench_cfg{c}.json")
        if os.path.exists(src):
            shutil.copy(src, os.path.join(PROF, f"{tag}_bench_cfg{c}.json"))
    if os.path.exists(os.path.join(MEAS, "bench_ref_cfg2.json")):
        shutil.copy(os.path.join(MEAS, "bench_ref_cfg2.json"), os.path.join(PROF, f"{tag}_bench_ref_cfg2.json"))
    summ = os.path.join(ROOT, "tools", "ncu_summary.py")
    lc = os.path.join(MEAS, "launches_cfg2.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(PROF, f"{tag}_launches_bench_cfg2.csv"))
        subprocess.check_call([sys.executable, summ, "launches", lc, os.path.join(PROF, f"{tag}_launches_bench_cfg2.json")],
                              stdout=subprocess.DEVNULL)
    ts = os.path.join(MEAS, "twoscan_cfg2.csv")
    if os.path.exists(ts):
        shutil.copy(ts, os.path.join(PROF, f"{tag}_twoscan_cfg2_launches.csv"))
        summarize_launches(ts, os.path.join(PROF, f"{tag}_twoscan_cfg2_launches.json"),
                           "cfg2 two-scan (LDPC_SCHED_TWOSCAN), 8192 frames, 15 iterations, early stop; ncu --metrics "
                           "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                           "(cold-cache, serialised)")
    frames = {1: 1024, 2: 8192, 3: 16384, 4: 512, 5: 1024}     # frames of the profiled decode (measure_r02.sh)
    for c in (1, 2, 3, 4, 5):
        src_csv = os.path.join(MEAS, f"ncu_source_cfg{c}.csv")
        if os.path.exists(src_csv):
            top_source_lines(src_csv, os.path.join(PROF, f"{tag}_ncu_source_top_cfg{c}.json"))
        rep = os.path.join(MEAS, f"prof_cfg{c}.ncu-rep")
        pre = os.path.join(MEAS, f"ncu_full_cfg{c}.json")          # summarised on the box
        dst = os.path.join(PROF, f"{tag}_ncu_full_cfg{c}.json")
        if os.path.exists(pre):
            shutil.copy(pre, dst)
        elif os.path.exists(rep):
            subprocess.check_call([sys.executable, summ, "raw", rep, dst], stdout=subprocess.DEVNULL)
        else:
            continue
        with open(dst) as f:
            d = json.load(f)[0]
        mb = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
        traffic = (d["dram__bytes_read.sum"] * mb.get(d["dram__bytes_read.sum.unit"], 1.0) +
                   d["dram__bytes_write.sum"] * mb.get(d["dram__bytes_write.sum.unit"], 1.0))
        with open(os.path.join(PROF, f"ncu_traffic_cfg{c}.json"), "w") as f:
            json.dump({"kernel": d["kernel"], "dram_bytes_per_launch": traffic, "frames_profiled": frames[c],
                       "source": f"profiles/{tag}_ncu_full_cfg{c}.json (ncu --set full, one launch)",
                       "note": "cfg2: the whole decode is one resident launch; cfg4/5: one iteration launch of "
                               "the streaming kernel"}, f, indent=1)
        print(f"cfg{c}: {d['kernel'][:60]} {d['gpu__time_duration.sum']} {d['gpu__time_duration.sum.unit']}, "
              f"DRAM {traffic / 1e6:.1f} MB, issue {d.get('smsp__issue_active.avg.pct_of_peak_sustained_active')}%, "
              f"ALU {d.get('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active')}%")


if __name__ == "__main__":
    main()
