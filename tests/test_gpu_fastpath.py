"""The certified fast front end (csrc/lk_fastpath.cu) against the exact path.

Throughput mode computes the bilateral approximately (MUFU ex2, FP32) with a
rigorous bound, and exactly only around edge candidates. Everything it
exports must be bit-identical to the exact path (LK_FLAG_EXACT): every report
field, the edge list (positions, gx, gy, theta), votes, DP paths, fits, m1,
energies and lanes. And the measured approximation error must sit inside the
bound the classification relies on."""
import numpy as np
import pytest

from paper_1807_02752_b200 import abi, lanekit, scenes

pytestmark = pytest.mark.gpu

EDGE_DERIVED = ["VDISPARITY", "VPATH", "BETA_INLIERS", "VPY", "VPY_SINGULAR", "EDGES", "VOTES",
                "UPATH", "GAMMA_INLIERS", "VPX", "M1", "ENERGY", "LANES"]
BOUND = 2.5e-5  # kEpsSmooth


def _runs(params, cfg):
    grey, disp = lanekit.synth_batch(params, threads=8)
    n, H, W = grey.shape
    out = {}
    for exact in (False, True):
        pipe = lanekit.GpuPipeline(W, H, cfg, max_batch=n, exact=exact)
        reps = [r.as_dict() for r in pipe.run(grey, disp)]
        hooks = [{h: pipe.raw(i, abi.STAGE[h]) for h in EDGE_DERIVED} if reps[i]["status"] == 0
                 else {} for i in range(n)]
        out[exact] = (pipe, reps, hooks)
    return out


@pytest.mark.parametrize("family", ["batch", "stress", "acceptance", "hires", "odd"])
def test_fast_path_is_bit_identical_to_exact(family):
    if family == "batch":
        params, cfg = [scenes.batch_scene(i) for i in range(8)], abi.default_config()
    elif family == "stress":
        params, cfg = [scenes.stress_scene(i) for i in range(4)], abi.default_config()
    elif family == "acceptance":
        params, cfg = [scenes.acceptance_scene(i) for i in range(20)], scenes.acceptance_config()
    elif family == "odd":
        params, cfg = [scenes.batch_scene(i, width=1241, height=373) for i in range(4)], abi.default_config()
    else:
        params, cfg = [scenes.hires_scene(i) for i in range(2)], scenes.hires_config()
    r = _runs(params, cfg)
    fast, exact = r[False], r[True]
    for i in range(len(params)):
        assert fast[1][i] == exact[1][i], f"frame {i}: report differs"
        for h in EDGE_DERIVED if fast[1][i]["status"] == 0 else []:
            assert fast[2][i][h] == exact[2][i][h], f"frame {i}: {h} differs"


def test_fast_path_error_within_bound():
    params = [scenes.batch_scene(i) for i in range(32)] + [scenes.stress_scene(i) for i in range(4)]
    grey, disp = lanekit.synth_batch(params, threads=8)
    n, H, W = grey.shape
    with lanekit.GpuPipeline(W, H, abi.default_config(), max_batch=n) as pipe:
        pipe.run(grey, disp)
        err = pipe.fast_path_error()
    print(f"max |approx - exact| smoothed over {n} frames: {err:.3e} (bound {BOUND:.1e})")
    assert 0 < err < BOUND / 2


def test_random_noise_frames():
    """Worst case for the approximation (uniform noise, every value present)."""
    rng = np.random.default_rng(7)
    grey = rng.integers(0, 256, size=(4, 240, 320), dtype=np.uint8)
    _, _, d0, _ = lanekit.synth_scene(scenes.acceptance_scene(0))
    disp = np.repeat(d0[None], 4, axis=0)
    cfg = scenes.acceptance_config()
    res = {}
    for exact in (False, True):
        with lanekit.GpuPipeline(320, 240, cfg, max_batch=4, exact=exact) as pipe:
            reps = [r.as_dict() for r in pipe.run(grey, disp)]
            edges = [pipe.raw(i, abi.STAGE["EDGES"]) if reps[i]["status"] == 0 or
                     reps[i]["failed_stage"] > 10 else b"" for i in range(4)]
            if not exact:
                err = pipe.fast_path_error()
                assert err < BOUND / 2
            res[exact] = (reps, edges)
    assert res[False] == res[True]
