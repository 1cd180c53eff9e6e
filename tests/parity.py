"""Parity rules between the GPU path and the CPU oracle.

Integer outputs (v-disparity, DP paths, RANSAC inlier sets and iteration
counts, horizon, mask, edge set, votes, lane columns, polyline NaN pattern)
must be bit-exact. Floating-point outputs must agree within RTOL = 1e-5
relative (north star), with an absolute floor of 1e-12 * max|x| per array
for values that are (near) zero.
"""
from __future__ import annotations

import numpy as np

from paper_1807_02752_b200 import abi

RTOL = 1e-5

INT_REPORT = [
    "status", "failed_stage", "msg", "err_row", "width", "height", "valid_disparities",
    "vpath_has_evidence", "beta_iterations", "beta_degraded", "beta_inlier_count", "horizon",
    "horizon_in_range", "road_mask_pixels", "edge_pixels", "vpx_votes", "vpx_skipped",
    "upath_has_evidence", "gamma_iterations", "gamma_degraded", "gamma_inlier_count",
    "lane_count", "lane_bottom_col",
]
# lk_frame_report.uncertain is the GPU's own certificate (0 from the CPU
# checkers), not a reference field: tests assert it explicitly
FP_REPORT = [
    "vpath_energy", "beta", "beta_inlier_fraction", "upath_energy", "gamma", "gamma_kappa",
    "gamma_v_normalizer", "gamma_inlier_fraction", "tr_lpv_used", "lane_energy",
]
EXACT_HOOKS = ["VDISPARITY", "VPATH", "BETA_INLIERS", "VPY_SINGULAR", "MASK", "VOTES", "UPATH",
               "GAMMA_INLIERS"]
FP_HOOKS = ["VPY", "SMOOTHED", "GX", "GY", "MAG", "THETA", "VPX_ACC", "VPX", "M0", "M1",
            "ENERGY"]
# SMOOTHED is exported only by the exact path (hooks / LK_FLAG_EXACT): the
# throughput path computes it exactly only around edge candidates.
HOOK_ONLY = {"MASK", "SMOOTHED", "GX", "GY", "MAG", "THETA", "VPX_ACC", "M0", "POLYLINES"}


def close(a, b, rtol=RTOL) -> bool:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        return False
    if a.size == 0:
        return True
    nan_a, nan_b = np.isnan(a), np.isnan(b)
    if not np.array_equal(nan_a, nan_b):
        return False
    a, b = a[~nan_a], b[~nan_b]
    if a.size == 0:
        return True
    floor = 1e-12 * max(np.max(np.abs(b)), 1e-300)
    return bool(np.all(np.abs(a - b) <= RTOL * np.abs(b) + floor))


def exact_fraction(a, b) -> float:
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    if a.size == 0:
        return 1.0
    same = (a == b) | (np.isnan(a) & np.isnan(b))
    return float(same.mean())


def compare_reports(g: abi.LkFrameReport, o: abi.LkFrameReport) -> list[str]:
    gd, od = g.as_dict(), o.as_dict()
    bad = []
    failed = od["status"] != 0
    for k in INT_REPORT:
        if failed and k not in ("status", "failed_stage", "msg", "err_row", "width", "height"):
            continue
        if gd[k] != od[k]:
            bad.append(f"report.{k}: gpu {gd[k]} vs oracle {od[k]}")
    if not failed:
        for k in FP_REPORT:
            if not close(gd[k], od[k]):
                bad.append(f"report.{k}: gpu {gd[k]} vs oracle {od[k]}")
    return bad


def compare_frame(gpu_stage, oracle_res, hooks: bool = True) -> list[str]:
    """gpu_stage(name) -> ndarray for one frame; oracle_res: CheckerResult."""
    bad = []
    orep = oracle_res.report
    if orep.status != 0:
        return bad
    for name in EXACT_HOOKS:
        if name in HOOK_ONLY and not hooks:
            continue
        g, o = gpu_stage(name), oracle_res.get(name)
        if g.shape != o.shape or not np.array_equal(g, o):
            bad.append(f"{name}: not bit-exact ({g.shape} vs {o.shape})")
    for name in FP_HOOKS:
        if name in HOOK_ONLY and not hooks:
            continue
        g, o = gpu_stage(name), oracle_res.get(name)
        if not close(g, o):
            diff = np.nanmax(np.abs(np.asarray(g, float) - np.asarray(o, float))) \
                if g.shape == o.shape else "shape"
            bad.append(f"{name}: outside rtol {RTOL} (max abs diff {diff})")
    ge, oe = gpu_stage("EDGES"), oracle_res.get("EDGES")
    if len(ge) != len(oe) or not (np.array_equal(ge["u"], oe["u"]) and
                                  np.array_equal(ge["v"], oe["v"])):
        bad.append("EDGES: edge set differs")
    else:
        for f in ("gx", "gy"):
            if not np.array_equal(ge[f], oe[f]):
                bad.append(f"EDGES.{f}: not bit-exact")
        if not close(ge["theta"], oe["theta"]):
            bad.append("EDGES.theta: outside tolerance")
    gl, ol = gpu_stage("LANES"), oracle_res.get("LANES")
    if len(gl) != len(ol) or not np.array_equal(gl["bottom_col"], ol["bottom_col"]) or \
            not np.array_equal(gl["n_points"], ol["n_points"]):
        bad.append(f"LANES: {gl['bottom_col'].tolist()} vs {ol['bottom_col'].tolist()}")
    elif not close(gl["energy"], ol["energy"]):
        bad.append("LANES.energy: outside tolerance")
    if hooks:
        gp, op = gpu_stage("POLYLINES"), oracle_res.get("POLYLINES")
        if gp.shape != op.shape or not close(gp, op):
            bad.append("POLYLINES: differ")
        elif not np.array_equal(np.round(np.nan_to_num(gp, nan=-1e9)),
                                np.round(np.nan_to_num(op, nan=-1e9))):
            bad.append("POLYLINES: rounded lane pixel positions differ")
    return bad
