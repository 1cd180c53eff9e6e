"""Warp-stall samples per CUDA source line of one kernel (ncu source page,
cuda+sass correlation; needs -lineinfo builds and --import-source on).

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [N] [inst]
       (inst: rank by warp instructions executed instead of stall samples)
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    col = 7 if len(sys.argv) > 4 and sys.argv[4] == "inst" else 4
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    agg, tot, path = {}, 0, ""
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if len(r) <= col or not r[0].isdigit() or not r[col].isdigit():
            continue
        s = int(r[col])
        key = (path, int(r[0]))
        src = r[1].strip()
        a = agg.setdefault(key, [0, src])
        a[0] += s
        tot += s
    for (p, ln), (s, src) in sorted(agg.items(), key=lambda t: -t[1][0])[:n]:
        print(f"{s / max(tot, 1) * 100:5.1f}%  {p}:{ln}  {src[:90]}")


if __name__ == "__main__":
    main()
