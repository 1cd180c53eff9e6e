"""Top SASS instructions of one kernel by warp-stall samples (ncu source page).

usage: python tools/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    # one block per function (a __noinline__ callee gets its own header rows)
    body = [r for r in rows[2:] if len(r) > ist and r[ist].isdigit()]
    tot = sum(int(r[ist] or 0) for r in body)
    for pos, r in sorted(enumerate(body), key=lambda t: -int(t[1][ist] or 0))[:n]:
        print(f"{pos:5d} {int(r[ist]) / tot * 100:5.1f}%  {r[isrc].strip()}")


if __name__ == "__main__":
    main()
