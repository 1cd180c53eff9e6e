import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1807_02752_b200 import lanekit, scenes, abi
for name, sc, cfg, W, H, n in (("kitti", scenes.batch_scene, abi.default_config(), 1242, 375, 32),
                               ("hires", scenes.hires_scene, scenes.hires_config(), 2560, 1024, 16)):
    params = [sc(1 + i) for i in range(n)]
    g, d = lanekit.synth_batch(params, threads=8)
    with lanekit.GpuPipeline(W, H, cfg, max_batch=n) as p:
        reps = p.run(g, d)
        reps = p.run(g, d)
    setup = np.median([r.gamma_kappa for r in reps]); dp = np.median([r.gamma_inlier_fraction for r in reps])
    loop = np.median([r.gamma[0] for r in reps]); bt = np.median([r.gamma[1] for r in reps])
    rows = np.median([H - r.horizon for r in reps])
    print(name, "setup", setup, "dp-accum", dp, "loop", loop, "backtrack", bt, "rows", rows, "cycles/stage", loop / rows)
