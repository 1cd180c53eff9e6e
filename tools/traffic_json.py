"""profiles/traffic.json from an ncu launch list with DRAM metrics.

usage: python tools/traffic_json.py LAUNCHES.csv CONFIG FRAMES SOURCE_NOTE
LAUNCHES.csv: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv of tools/kernel_times.py (single-range replays, every
launch covers FRAMES frames). Per stage: mean over launches of the stage's kernels'
read + write bytes, summed over the kernels (bench.py's roofline.traffic).
"""
import collections
import csv
import json
import sys
from pathlib import Path

STAGE = {  # kernel -> pipeline stage (lk_kernels.cu launch_pipeline marks)
    "k_vdisparity": 5, "k_vpath": 6, "k_road_fit": 7,
    "k_prescreen": 9, "k_bilateral_need": 9, "k_bilateral_tile": 9,
    "k_sobel_screen": 10, "k_refine_exact": 10, "k_sobel_decide": 10, "k_sobel_edges": 10,
    "k_edge_scan": 10, "k_edge_emit_tiles": 10, "k_edge_emit": 10,
    "k_vanish": 11, "k_gamma_fit": 11, "k_wg": 11,
}


def main(path, cfg, frames, note):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = collections.defaultdict(list)  # (kernel, launch id) -> bytes
    by_launch = collections.defaultdict(float)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[mi].startswith("dram__bytes"):
            continue
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("lkg::", "").strip()
        by_launch[r[0]] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        names[r[0]] = name
    for lid, b in by_launch.items():
        per[names[lid]].append(b)
    stages = collections.defaultdict(float)
    for k, v in per.items():
        st = STAGE.get(k, 12)
        stages[st] += sum(v) / len(v)
    p = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
    data = json.loads(p.read_text()) if p.exists() else {}
    data[cfg] = {"frames": int(frames), **{str(k): round(v) for k, v in sorted(stages.items())},
                 "source": note}
    p.write_text(json.dumps(data, indent=1) + "\n")
    print(json.dumps(data[cfg], indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:5])
