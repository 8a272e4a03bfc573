"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.

    python profiles/ncu_hotspots.py report.ncu-rep [kernel-regex] [--top N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "k_sweep<"
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name"')
    for b in blocks[1:]:
        lines = b.splitlines()
        name = lines[0]
        if kre not in name:
            continue
        rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        hdr = rows[0]
        si = hdr.index("Warp Stall Sampling (All Samples)")
        src = hdr.index("Source")
        tot = sum(int(r[si] or 0) for r in rows[1:] if len(r) > si)
        print(name[:120], "total samples", tot)
        ranked = sorted(((int(r[si] or 0), i, r[src]) for i, r in enumerate(rows[1:]) if len(r) > si), reverse=True)
        for smp, i, s in ranked[:top]:
            print(f"{100.0 * smp / tot:5.1f}%  #{i:4d}  {s.strip()}")
        break


if __name__ == "__main__":
    main()
