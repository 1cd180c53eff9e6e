"""Hook-by-hook parity report, GPU vs oracle, for a few scenes (diagnostics).

usage: python tools/parity_report.py [probe|batch|stress|accept] [count]
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

from checkers import Checker  # noqa: E402
from parity import close, exact_fraction  # noqa: E402

from paper_1807_02752_b200 import abi, lanekit, scenes  # noqa: E402


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "probe"
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    cfg = abi.default_config()
    if kind == "probe":
        params = [scenes.probe_scene()]
    elif kind == "batch":
        params = [scenes.batch_scene(i) for i in range(count)]
    elif kind == "hires":
        params = [scenes.hires_scene(i) for i in range(count)]
        cfg = scenes.hires_config()
    elif kind == "stress":
        params = [scenes.stress_scene(i) for i in range(count)]
    else:
        params = [scenes.acceptance_scene(i) for i in range(count)]
        cfg = scenes.acceptance_config()
    grey, disp = lanekit.synth_batch(params)
    n, H, W = grey.shape
    orc = Checker("oracle")
    with lanekit.GpuPipeline(W, H, cfg, max_batch=n, hooks=True, graph=False) as pipe:
        reps = pipe.run(grey, disp)
        print("stage ms:", pipe.stage_times())
        for i in range(n):
            o = orc.run(grey[i], disp[i], cfg)
            gd, od = reps[i].as_dict(), o.report.as_dict()
            print(f"--- frame {i}: gpu status {gd['status']}/{gd['failed_stage']} "
                  f"oracle {od['status']}/{od['failed_stage']}")
            for k in gd:
                if gd[k] != od[k]:
                    print(f"   report {k}: gpu {gd[k]} oracle {od[k]}")
            if od["status"]:
                continue
            for name in abi.STAGES:
                try:
                    g = pipe.stage(i, name)
                except Exception as e:  # noqa: BLE001
                    print(f"   {name}: gpu error {e}")
                    continue
                ov = o.get(name)
                if g.dtype.names:
                    same = g.shape == ov.shape and all(
                        np.array_equal(g[f], ov[f]) for f in g.dtype.names)
                    print(f"   {name:14s} n={len(g)}/{len(ov)} exact={same}")
                    continue
                ex = exact_fraction(g, ov) if g.shape == ov.shape else -1
                rel = 0.0
                if g.shape == ov.shape and g.dtype.kind == "f":
                    a, b = np.asarray(g, float), np.asarray(ov, float)
                    m = ~(np.isnan(a) | np.isnan(b)) & (b != 0)
                    rel = float(np.max(np.abs(a[m] - b[m]) / np.abs(b[m]))) if m.any() else 0.0
                print(f"   {name:14s} shape {g.shape} vs {ov.shape} exact {ex:.6f} "
                      f"max_rel {rel:.3e} close {close(g, ov) if g.shape == ov.shape else False}")


if __name__ == "__main__":
    main()
