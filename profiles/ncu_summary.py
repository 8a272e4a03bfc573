"""Summarise an ncu --set full report (run here, on the CPU box).

    python profiles/ncu_summary.py gpurun_out/<report>.ncu-rep [--json out.json]

Prints per kernel: duration, DRAM bytes, L2 hit rate, L1 data-pipe
utilisation, achieved occupancy and the top stall reasons; with --json
writes {kernel: {dram_bytes: ..., duration_ns: ...}} for bench.py's
roofline.traffic.
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "duration": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "occupancy": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "issue_active": "sm__inst_issued.avg.pct_of_peak_sustained_active",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}


def load(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--json")
    a = ap.parse_args()
    h, units, data = load(a.report)
    out = {}
    for r in data:
        name = r[h.index("Kernel Name")].split("(")[0].replace("dynpr_b200::<unnamed>::", "")
        print(f"== {name}")
        vals = {}
        for k, m in KEYS.items():
            if m in h:
                i = h.index(m)
                v = r[i]
                try:
                    x = float(v.replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    x = v
                vals[k] = x
                print(f"   {k:18s} {v} {units[i]}")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), k[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]))
                except ValueError:
                    pass
        print("   stalls: " + ", ".join(f"{n} {v:.1f}" for v, n in sorted(stalls, reverse=True)[:6]))
        entry = out.setdefault(name, {"dram_bytes": [], "duration_ns": []})
        if isinstance(vals.get("dram_read"), float):
            entry["dram_bytes"].append(vals["dram_read"] + vals["dram_write"])
            entry["duration_ns"].append(vals["duration"])
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
