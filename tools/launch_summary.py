"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hdr_i]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
    agg = collections.defaultdict(list)
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        name = r[ki].split("(")[0].replace("void lkg::", "").replace("lkg::", "")
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] in ("nsecond", "ns") else (v * 1e3 if r[ui] in ("msecond", "ms") else v)
        agg[name].append(v)
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:32s} n={len(v):3d} mean={sum(v) / len(v):9.1f} us  share={sum(v) / tot * 100:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
