"""GPU path against the REFERENCE's own outputs (tests/golden/golden.json,
written by the compiled reference, oracle/_ref).

Bit-exact (SHA-256 of the hook bytes): every integer hook, and every float hook
whose arithmetic has no transcendental — the bilateral output (exact via
host-built glibc exp tables), Sobel gx/gy/magnitude, V_py, V_px (RANSAC fits
reproduced operation for operation). theta / m0 / m1 / energy go through CUDA's
atan2 and exp (<= 2 ulp from glibc) and are checked at rtol 1e-5, the north
star's tolerance, in tests/test_gpu_parity.py against the live oracle."""
import numpy as np
import pytest

from golden_util import case_ids, config, dec, inputs, load_cases, report_expected, sha
from paper_1807_02752_b200 import abi, lanekit
from parity import RTOL, close

pytestmark = pytest.mark.gpu

CASES = {c["name"]: c for c in load_cases()}
EXACT = ["VDISPARITY", "VPATH", "BETA_INLIERS", "VPY", "VPY_SINGULAR", "MASK", "SMOOTHED", "GX",
         "GY", "MAG", "VOTES", "UPATH", "GAMMA_INLIERS", "VPX"]
INT_FIELDS = ["status", "failed_stage", "msg", "err_row", "valid_disparities",
              "vpath_has_evidence", "beta_iterations", "beta_degraded", "beta_inlier_count",
              "horizon", "horizon_in_range", "road_mask_pixels", "edge_pixels", "vpx_votes",
              "vpx_skipped", "upath_has_evidence", "gamma_iterations", "gamma_degraded",
              "gamma_inlier_count", "lane_count", "lane_bottom_col"]
EXACT_FLOATS = ["vpath_energy", "beta", "beta_inlier_fraction", "upath_energy", "gamma",
                "gamma_v_normalizer", "gamma_inlier_fraction"]
TOL_FLOATS = ["tr_lpv_used", "lane_energy"]


@pytest.mark.parametrize("name", case_ids())
def test_gpu_matches_reference_golden(name):
    case = CASES[name]
    grey, disp = inputs(case)
    H, W = grey.shape
    with lanekit.GpuPipeline(W, H, config(case), max_batch=1, hooks=True) as pipe:
        rep = pipe.run(grey, disp)[0]
        got = rep.as_dict()
        want = report_expected(case)
        for k in INT_FIELDS:
            assert got[k] == want[k], f"{k}: gpu {got[k]} vs reference {want[k]}"
        if want["status"] != 0:
            return
        for k in EXACT_FLOATS:
            g = np.asarray(got[k], float)
            w = np.asarray(want[k], float)
            assert np.array_equal(g, w), f"{k}: gpu {got[k]} vs reference {want[k]}"
        for k in TOL_FLOATS:
            assert close(got[k], want[k]), f"{k}: gpu {got[k]} vs reference {want[k]} (rtol {RTOL})"
        for hook in EXACT:
            raw = pipe.raw(0, abi.STAGE[hook])
            assert sha(raw) == case["hooks"][hook]["sha256"], f"{hook} not bit-exact"
        lanes = pipe.stage(0, "LANES")
        ref_lanes = case["hooks"]["LANES"]["values"]
        assert lanes["bottom_col"].tolist() == ref_lanes["bottom_col"]
        assert lanes["n_points"].tolist() == ref_lanes["n_points"]
        assert close(lanes["energy"], dec(ref_lanes["energy"]))
