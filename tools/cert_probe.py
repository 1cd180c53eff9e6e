"""Probe of the lane-decision certificate on hi-res frames: per frame the
uncertain count, adjacent equal energies, and the energy spread."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1807_02752_b200 import abi, lanekit, scenes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
params = [scenes.hires_scene(1 + i) for i in range(n)]
grey, disp = lanekit.synth_batch(params, threads=8)
cfg = scenes.hires_config()
with lanekit.GpuPipeline(scenes.HIRES_W, scenes.HIRES_H, cfg, max_batch=n) as p:
    reps = p.run(grey, disp)
    for i, r in enumerate(reps):
        e = p.stage(i, "ENERGY")
        eq = int(np.sum(e[1:] == e[:-1]))
        nz = int(np.sum(e != 0))
        d = np.abs(np.diff(e))
        small = int(np.sum((d > 0) & (d < 1e-6 * np.abs(e).max())))
        print(i, "uncertain", r.uncertain, "lanes", r.lane_count, "eq_adjacent", eq, "nonzero", nz,
              "tiny_diffs", small, "min", e.min(), "tr", r.tr_lpv_used)
