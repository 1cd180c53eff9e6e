"""ctypes mirror of include/lanekit_b200.h (the C-ABI boundary).

Layouts here must match the header field for field; tests/test_abi.py checks
the sizes against the compiled library (lk_abi_sizes)."""
from __future__ import annotations

import ctypes as C
import math

LK_MAX_INLINE_LANES = 16

LK_OK = 0
LK_ERR_INVALID_ARGUMENT = 1
LK_ERR_CONFIG = 2
LK_ERR_CUDA = 3
LK_ERR_NO_DEVICE = 4
LK_ERR_FRAME = 5
LK_ERR_UNAVAILABLE = 6

LK_FLAG_HOOKS = 1
LK_FLAG_NO_GRAPH = 2
LK_FLAG_EXACT = 4
LK_FLAG_STEREO = 8

LK_MEM_HOST = 0
LK_MEM_DEVICE = 1

# lk_stage ids (PipelineResult members, pipeline.hpp:69-99)
STAGES = [
    "VDISPARITY", "VPATH", "BETA_INLIERS", "VPY", "VPY_SINGULAR", "MASK", "SMOOTHED",
    "GX", "GY", "MAG", "THETA", "EDGES", "VOTES", "VPX_ACC", "UPATH", "GAMMA_INLIERS",
    "VPX", "M0", "M1", "ENERGY", "LANES", "POLYLINES",
    # stereo batches (LK_FLAG_STEREO): stats_left, SRP maps, the LRC disparity
    "STATS_MU", "STATS_SIGMA", "DISP_LEFT", "DISP_RIGHT", "DISPARITY",
]
STAGE = {name: i for i, name in enumerate(STAGES)}

# lk_msg ids and the reference's texts (pipeline.hpp:189-190, 238-239;
# ransac.hpp:41-42, 90; road_profile.hpp:223-225; preprocess.hpp:69; lanes.hpp:68)
MSG_TEXT = {
    0: "",
    1: "empty input image",
    2: "v-disparity histogram is empty; no road surface evidence",
    3: "ransac: fewer points than the sample size",
    4: "ransac: no sample produced a fit",
    5: "road profile: singular V_py derivative at row {row}",
    6: "sobel: image smaller than the kernel",
    7: "vanishing-point accumulator is empty; no lane edge evidence",
    8: "m1: image smaller than the kernel",
    9: "stereo pair dimensions differ",
}

# pipeline.hpp:101-116
STAGE_NAMES = [
    "block statistics", "left disparity", "right disparity", "consistency check",
    "v-disparity accumulation", "road path extraction", "road profile fit", "road mask",
    "bilateral smoothing", "edge detection", "vanishing point estimation", "lane detection",
]


class LkConfig(C.Structure):
    """lanekit::PipelineConfig (config.hpp:16-46)."""

    _fields_ = [
        ("rho", C.c_int32), ("tau", C.c_int32), ("d_max", C.c_int32), ("tr_lrc", C.c_int32),
        ("sigma_floor", C.c_double), ("lambda_y", C.c_double), ("tr_y", C.c_double),
        ("eps_y", C.c_double), ("varpi", C.c_double), ("sigma_s", C.c_double),
        ("sigma_r", C.c_double), ("bf_window", C.c_int32), ("chi", C.c_int32),
        ("sobel_threshold", C.c_double), ("rho_vote", C.c_double), ("lambda_x", C.c_double),
        ("tr_x", C.c_double), ("eps_x", C.c_double), ("sigma_g", C.c_double),
        ("nu", C.c_int32), ("varsigma", C.c_int32), ("lambda_g", C.c_double),
        ("xi", C.c_double), ("tr_lpv", C.c_double), ("min_lane_sep", C.c_int32),
        ("paper_sign", C.c_int32), ("rng_seed", C.c_uint64), ("threads", C.c_int32),
        ("_pad0", C.c_int32),
    ]


def default_config(**overrides) -> LkConfig:
    """PipelineConfig defaults (config.hpp:16-46)."""
    c = LkConfig(
        rho=3, tau=1, d_max=64, tr_lrc=3, sigma_floor=1e-4, lambda_y=30.0, tr_y=4.0,
        eps_y=0.99, varpi=3.0, sigma_s=300.0, sigma_r=0.3, bf_window=11, chi=25,
        sobel_threshold=100.0, rho_vote=1.0, lambda_x=10.0, tr_x=16.0, eps_x=0.99,
        sigma_g=3.5, nu=1, varsigma=3, lambda_g=1.0, xi=0.5, tr_lpv=math.nan,
        min_lane_sep=20, paper_sign=0, rng_seed=1, threads=1,
    )
    for k, v in overrides.items():
        if k == "paper_sign":
            v = int(bool(v))
        setattr(c, k, v)
    return c


class LkFrameReport(C.Structure):
    """lanekit::PipelineReport (pipeline.hpp:30-66) + per-frame status."""

    _fields_ = [
        ("status", C.c_int64), ("failed_stage", C.c_int64), ("msg", C.c_int64),
        ("err_row", C.c_int64), ("width", C.c_int64), ("height", C.c_int64),
        ("rng_seed", C.c_uint64), ("valid_disparities", C.c_int64),
        ("vpath_has_evidence", C.c_int64), ("vpath_energy", C.c_double),
        ("beta", C.c_double * 3), ("beta_iterations", C.c_int64),
        ("beta_inlier_fraction", C.c_double), ("beta_degraded", C.c_int64),
        ("beta_inlier_count", C.c_int64), ("horizon", C.c_int64),
        ("horizon_in_range", C.c_int64), ("road_mask_pixels", C.c_int64),
        ("edge_pixels", C.c_int64), ("vpx_votes", C.c_int64), ("vpx_skipped", C.c_int64),
        ("upath_has_evidence", C.c_int64), ("upath_energy", C.c_double),
        ("gamma", C.c_double * 5), ("gamma_kappa", C.c_double),
        ("gamma_v_normalizer", C.c_double), ("gamma_iterations", C.c_int64),
        ("gamma_inlier_fraction", C.c_double), ("gamma_degraded", C.c_int64),
        ("gamma_inlier_count", C.c_int64), ("tr_lpv_used", C.c_double),
        ("lane_count", C.c_int64),
        ("lane_bottom_col", C.c_int64 * LK_MAX_INLINE_LANES),
        ("lane_energy", C.c_double * LK_MAX_INLINE_LANES),
        ("uncertain", C.c_int64),
    ]

    def as_dict(self) -> dict:
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            if isinstance(v, C.Array):
                v = list(v)
            out[name] = v
        n = min(out["lane_count"], LK_MAX_INLINE_LANES)
        out["lane_bottom_col"] = out["lane_bottom_col"][:n]
        out["lane_energy"] = out["lane_energy"][:n]
        return out


def frame_message(rep: LkFrameReport) -> str:
    """'stage N (name): msg' exactly as StageError renders it (common.hpp:18-24)."""
    if rep.status == 0:
        return ""
    st = int(rep.failed_stage)
    text = MSG_TEXT.get(int(rep.msg), "unknown failure").format(row=int(rep.err_row))
    return f"stage {st} ({STAGE_NAMES[st - 1]}): {text}"


class LkSceneParams(C.Structure):
    """lanekit::SceneParams (synth.hpp:62-80) + obstacle / pitch-change extensions."""

    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("beta", C.c_double * 3),
        ("gamma", C.c_double * 5), ("d_max", C.c_int32), ("n_lanes", C.c_int32),
        ("lane_bottoms", C.c_double * 8), ("lane_width", C.c_double),
        ("lane_brightness", C.c_double), ("road_base", C.c_double), ("sky_level", C.c_double),
        ("texture_amplitude", C.c_double), ("noise_sigma", C.c_double),
        ("rng_seed", C.c_uint64), ("n_obstacles", C.c_int32), ("pitch_row", C.c_int32),
        ("pitch_jump", C.c_double), ("obstacle_box", (C.c_int32 * 4) * 4),
        ("obstacle_disp", C.c_int32 * 4),
    ]


def scene_params(width=640, height=360, beta=(-15.0, 0.15, 0.0001), gamma=(320.0, 0, 0, 0, 0),
                 d_max=192, lane_bottoms=(160.0, 320.0, 480.0), lane_width=6.0,
                 lane_brightness=0.85, road_base=0.35, sky_level=0.75, texture_amplitude=0.15,
                 noise_sigma=0.0, rng_seed=1, obstacles=(), pitch_row=-1,
                 pitch_jump=0.0) -> LkSceneParams:
    """SceneParams defaults (synth.hpp:62-80). obstacles: [((u0, v0, u1, v1), d), ...]."""
    p = LkSceneParams()
    p.width, p.height = width, height
    for i, b in enumerate(beta):
        p.beta[i] = b
    for i, g in enumerate(gamma):
        p.gamma[i] = g
    p.d_max = d_max
    if len(lane_bottoms) > 8:
        raise ValueError("at most 8 lanes")
    p.n_lanes = len(lane_bottoms)
    for i, lb in enumerate(lane_bottoms):
        p.lane_bottoms[i] = lb
    p.lane_width, p.lane_brightness = lane_width, lane_brightness
    p.road_base, p.sky_level = road_base, sky_level
    p.texture_amplitude, p.noise_sigma = texture_amplitude, noise_sigma
    p.rng_seed = rng_seed
    if len(obstacles) > 4:
        raise ValueError("at most 4 obstacles")
    p.n_obstacles = len(obstacles)
    for i, (box, d) in enumerate(obstacles):
        for k in range(4):
            p.obstacle_box[i][k] = box[k]
        p.obstacle_disp[i] = d
    p.pitch_row, p.pitch_jump = pitch_row, pitch_jump
    return p


class LkEdge(C.Structure):
    _fields_ = [("u", C.c_int32), ("v", C.c_int32), ("gx", C.c_double), ("gy", C.c_double),
                ("theta", C.c_double)]


class LkVote(C.Structure):
    _fields_ = [("u_e", C.c_int32), ("v_e", C.c_int32), ("col", C.c_int32)]


class LkLane(C.Structure):
    _fields_ = [("bottom_col", C.c_int32), ("n_points", C.c_int32), ("energy", C.c_double)]


_EDGE_DT = [("u", "<i4"), ("v", "<i4"), ("gx", "<f8"), ("gy", "<f8"), ("theta", "<f8")]
_VOTE_DT = [("u_e", "<i4"), ("v_e", "<i4"), ("col", "<i4")]
_LANE_DT = [("bottom_col", "<i4"), ("n_points", "<i4"), ("energy", "<f8")]


def decode_stage(stage: int, raw: bytes, width: int, height: int, d_max: int,
                 ext_cols: int, horizon: int):
    """Decode an lk_get_stage buffer into a numpy array (layouts: lanekit_b200.h)."""
    import numpy as np

    name = STAGES[stage]
    W, H = width, height
    rows = H - horizon
    if name == "VDISPARITY":
        return np.frombuffer(raw, "<i4").reshape(H, d_max + 1)
    if name in ("VPATH", "BETA_INLIERS", "UPATH", "GAMMA_INLIERS"):
        return np.frombuffer(raw, "<i4").reshape(-1, 2)
    if name in ("VPY", "VPX"):
        return np.frombuffer(raw, "<f8")
    if name == "VPY_SINGULAR":
        return np.frombuffer(raw, "u1")
    if name == "MASK":
        return np.frombuffer(raw, "u1").reshape(H, W)
    if name in ("SMOOTHED", "GX", "GY", "MAG", "THETA", "M0", "M1"):
        return np.frombuffer(raw, "<f8").reshape(H, W)
    if name == "EDGES":
        return np.frombuffer(raw, _EDGE_DT)
    if name == "VOTES":
        return np.frombuffer(raw, _VOTE_DT)
    if name == "VPX_ACC":
        return np.frombuffer(raw, "<f8").reshape(rows, ext_cols)
    if name == "ENERGY":
        return np.frombuffer(raw, "<f8")
    if name == "LANES":
        return np.frombuffer(raw, _LANE_DT)
    if name == "POLYLINES":
        return np.frombuffer(raw, "<f8").reshape(-1, rows)
    if name in ("STATS_MU", "STATS_SIGMA"):
        return np.frombuffer(raw, "<f8").reshape(H, W)
    if name in ("DISP_LEFT", "DISP_RIGHT", "DISPARITY"):
        return np.frombuffer(raw, "u1").reshape(H, W)
    raise ValueError(name)
