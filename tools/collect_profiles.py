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


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
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
    for c in (2, 4, 5):
        rep = os.path.join(MEAS, f"prof_cfg{c}.ncu-rep")
        if not os.path.exists(rep):
            continue
        dst = os.path.join(PROF, f"{tag}_ncu_full_cfg{c}.json")
        subprocess.check_call([sys.executable, summ, "raw", rep, dst], stdout=subprocess.DEVNULL)
        with open(dst) as f:
            d = json.load(f)[0]
        mb = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
        traffic = (d["dram__bytes_read.sum"] * mb.get(d["dram__bytes_read.sum.unit"], 1.0) +
                   d["dram__bytes_write.sum"] * mb.get(d["dram__bytes_write.sum.unit"], 1.0))
        with open(os.path.join(PROF, f"ncu_traffic_cfg{c}.json"), "w") as f:
            json.dump({"kernel": d["kernel"], "dram_bytes_per_launch": traffic,
                       "source": f"profiles/{tag}_ncu_full_cfg{c}.json (ncu --set full, one launch)",
                       "note": "cfg2: the whole decode is one resident launch; cfg4/5: one iteration launch of "
                               "the streaming kernel"}, f, indent=1)
        print(f"cfg{c}: {d['kernel'][:60]} {d['gpu__time_duration.sum']} {d['gpu__time_duration.sum.unit']}, "
              f"DRAM {traffic / 1e6:.1f} MB, issue {d.get('smsp__issue_active.avg.pct_of_peak_sustained_active')}%, "
              f"ALU {d.get('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active')}%")


if __name__ == "__main__":
    main()
