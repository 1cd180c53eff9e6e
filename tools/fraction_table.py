"""Per-kernel roofline fractions (HBM, FP64 and L1 fractions
per kernel) from the ncu --set full summaries tools/ncu_summary.py wrote.

usage: python tools/fraction_table.py profiles/r02_k_*_ncu.txt > profiles/r02_fractions.md
HBM % = (DRAM read + write bytes) / duration against MEASURED_PEAKS.json hbm_gbs.
"""
import json
import pathlib
import re
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0, "nsecond": 1e-9}


def parse(path):
    out, cur = [], None
    for line in pathlib.Path(path).read_text().splitlines():
        if line.startswith("== "):
            if cur and "duration" in cur:
                out.append(cur)
            cur = {"name": line[3:].split("(")[0].replace("void ", "").strip()}
            if any(c["name"] == cur["name"] for c in out):
                cur = None  # the second (pipes / stalls) section of the same kernel
            continue
        if cur is None:
            continue
        m = re.match(r"\s+(.+?)\s{2,}([-0-9.eE+]+)\s*(\S*)$", line)
        if m:
            key, val, unit = m.group(1).strip(), float(m.group(2)), m.group(3)
            cur[key] = val * SCALE.get(unit, 1.0) if unit in SCALE else val
    if cur and "duration" in cur:
        out.append(cur)
    return out


def main(paths):
    peak = json.loads(pathlib.Path(__file__).resolve().parent.parent.joinpath(
        "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    print(f"| kernel | µs | DRAM GB/s | HBM % of {peak:.0f} | FP64 pipe % | L1/LSU % | issue % | occupancy % |")
    print("|---|---|---|---|---|---|---|---|")
    for p in paths:
        for k in parse(p):
            t = k["duration"]
            gbs = (k.get("DRAM read", 0) + k.get("DRAM write", 0)) / t / 1e9
            print(f"| `{k['name']}` | {t * 1e6:.0f} | {gbs:.0f} | {100 * gbs / peak:.1f} | "
                  f"{k.get('FP64 pipe active %', 0):.1f} | {k.get('L1/LSU data-pipe wavefronts %', 0):.1f} | "
                  f"{k.get('issue active %', 0):.1f} | {k.get('achieved occupancy %', 0):.1f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
