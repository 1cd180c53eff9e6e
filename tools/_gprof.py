import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1807_02752_b200 import lanekit, scenes, abi
params = [scenes.batch_scene(1 + i) for i in range(256)]
g, d = lanekit.synth_batch(params, threads=8)
with lanekit.GpuPipeline(1242, 375, abi.default_config(), max_batch=256) as p:
    reps = p.run(g, d)
    reps = p.run(g, d)
rows = []
for r in reps:
    rows.append((r.gamma_kappa, r.gamma_v_normalizer, r.gamma_inlier_fraction, r.beta[0], r.beta[1], r.beta[2], r.vpath_energy, r.gamma_iterations))
a = np.array(rows)
i = int(np.argmax(a[:, 0] + a[:, 1]))
print("worst frame: loop", a[i, 0], "final", a[i, 1], "tail", a[i, 2], "fit", a[i, 3], "cls", a[i, 4], "commit", a[i, 5], "rounds", a[i, 6], "iters", a[i, 7])
print("median loop", np.median(a[:, 0]), "median rounds", np.median(a[:, 6]), "median iters", np.median(a[:, 7]))
