"""Regenerates tests/golden/golden.json from the REFERENCE itself.

Source of truth: oracle/_ref/liblk_ref.so = the unmodified lanekit headers
(/root/reference/proj/include) compiled here against the Eigen stand-in, with
stages 5-12 composed as pipeline.hpp:184-270 does and the disparity injected.
Only runnable where /root/reference exists (the dev container); the JSON it
writes is committed and travels to the GPU box.

For every case the fixture stores: the scene parameters and config, SHA-256
of the 8-bit inputs (the reference's gen_scene + write_png_gray quantisation),
the full PipelineReport, and for every hook its shape, dtype and SHA-256 —
small hooks (DP paths, RANSAC inlier sets, lanes) also in full, floats as
exact hex strings.
"""
from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

from checkers import Checker  # noqa: E402
from golden_util import apply_mutation  # noqa: E402

from paper_1807_02752_b200 import abi, scenes  # noqa: E402

SMALL_HOOKS = {"VPATH", "BETA_INLIERS", "UPATH", "GAMMA_INLIERS", "LANES"}


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def enc(x):
    if isinstance(x, float):
        return x.hex() if math.isfinite(x) else repr(x)
    if isinstance(x, (list, tuple)):
        return [enc(v) for v in x]
    return x


def params_dict(p: abi.LkSceneParams) -> dict:
    out = {}
    for name, _ in p._fields_:
        v = getattr(p, name)
        if hasattr(v, "__len__"):
            v = [list(x) if hasattr(x, "__len__") else x for x in v]
        out[name] = enc(v) if not isinstance(v, list) else [enc(x) for x in v]
    return out


def config_dict(c: abi.LkConfig) -> dict:
    return {name: enc(getattr(c, name)) for name, _ in c._fields_ if name != "_pad0"}


def cases():
    yield "probe_kitti", scenes.probe_scene(), abi.default_config(), None
    for i in range(6):
        yield f"acceptance_{i}", scenes.acceptance_scene(i), scenes.acceptance_config(), None
    for i in range(4):
        yield f"stress_{i}", scenes.stress_scene(i), abi.default_config(), None
    yield "batch_92_gamma181", scenes.batch_scene(92), abi.default_config(), None
    yield "batch_7", scenes.batch_scene(7), abi.default_config(), None
    yield ("acceptance_1_paper_sign_manual_tr", scenes.acceptance_scene(1),
           abi.default_config(d_max=32, nu=2, lambda_g=1.03, paper_sign=True, tr_lpv=-60.0,
                              chi=10, rng_seed=7), None)
    yield ("acceptance_2_window7_rho_vote2", scenes.acceptance_scene(2),
           abi.default_config(d_max=32, bf_window=7, rho_vote=2.0, lambda_x=3.5, varsigma=2,
                              min_lane_sep=8), None)
    yield "hires_5", scenes.hires_scene(5), scenes.hires_config(), None
    yield "fail_stage6_no_disparity", scenes.acceptance_scene(3), scenes.acceptance_config(), \
        "zero_disparity"
    yield "fail_stage11_flat_grey", scenes.acceptance_scene(4), scenes.acceptance_config(), \
        "flat_grey"
    # stage 7 (ransac.hpp:41-42): d_max 1 leaves 2 v-path points for a 3-point sample
    yield "fail_stage7_few_points", scenes.acceptance_scene(0), \
        abi.default_config(d_max=1, rho=4, sigma_floor=0.03, tr_lrc=1, nu=2, lambda_g=1.03), \
        "disparity_one_below_120"
    # stage 7 (ransac.hpp:90): all road evidence in one row -> every sample's
    # parabola fit lacks three distinct rows
    yield "fail_stage7_no_fit", scenes.acceptance_scene(0), scenes.acceptance_config(), \
        "disparity_row150_d10"


def main():
    ref = Checker("ref")
    out = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (reference headers)",
           "cases": []}
    for name, p, cfg, mutate in cases():
        if p.n_obstacles or p.pitch_row >= 0:
            # generator extension the reference does not have: inputs from the
            # repo generator (pinned to gen_scene on the reference's own scenes)
            from paper_1807_02752_b200 import lanekit

            grey, _, disp, _ = lanekit.synth_scene(p)
            source = "repo generator (obstacle / pitch extension)"
        else:
            grey, _, disp, _ = ref.gen_scene(p)
            source = "reference gen_scene"
        apply_mutation(mutate, grey, disp)
        r = ref.run(grey, disp, cfg)
        case = {"name": name, "scene": params_dict(p), "config": config_dict(cfg),
                "mutate": mutate, "inputs": source, "grey_sha256": sha(grey.tobytes()),
                "disp_sha256": sha(disp.tobytes()),
                "report": {k: enc(v) for k, v in r.report.as_dict().items()},
                "ext_cols": r.ext_cols, "hooks": {}}
        if r.report.status == 0:
            for hook in abi.STAGES:
                raw = r.raw(abi.STAGE[hook])
                if not raw and hook in ("STATS_MU", "STATS_SIGMA", "DISP_LEFT", "DISP_RIGHT",
                                        "DISPARITY"):
                    continue  # stage 1-4 hooks: the disparity is injected here
                arr = r.get(hook)
                h = {"sha256": sha(raw), "shape": list(arr.shape), "nbytes": len(raw)}
                if hook in SMALL_HOOKS:
                    if arr.dtype.names:
                        h["values"] = {f: enc(arr[f].tolist()) for f in arr.dtype.names}
                    else:
                        h["values"] = enc(arr.tolist())
                case["hooks"][hook] = h
        out["cases"].append(case)
        print(name, "status", r.report.status, "stage", r.report.failed_stage,
              "lanes", r.report.as_dict()["lane_bottom_col"], flush=True)
    text = json.dumps(out, separators=(",", ":")).replace('{"name"', '\n{"name"')
    (ROOT / "tests" / "golden" / "golden.json").write_text(text + "\n")


if __name__ == "__main__":
    main()
