"""Workload definitions (BASELINE.json configs).

Synthetic scenes are rendered by the in-library generator (a restatement of
lanekit::gen_scene, synth.hpp:103-200) — there is no dataset on the box.
"""
from __future__ import annotations

from . import abi

KITTI_W, KITTI_H = 1242, 375
HIRES_W, HIRES_H = 2560, 1024
BETA = (-15.0, 0.15, 1e-4)  # horizon ~94, f(374) = 55.1 <= d_max 64


def probe_scene(seed: int = 5) -> abi.LkSceneParams:
    """Config 1: one KITTI-size frame, 2 curved lanes (the survey's probe scene)."""
    W = KITTI_W
    return abi.scene_params(width=W, height=KITTI_H, beta=BETA,
                            gamma=(W / 2, -0.10, 2.5e-4, 0, 0), d_max=255,
                            lane_bottoms=(0.30 * W, 0.62 * W), noise_sigma=0.02, rng_seed=seed)


def batch_scene(i: int, width: int = KITTI_W, height: int = KITTI_H,
                beta=BETA, d_max: int = 255) -> abi.LkSceneParams:
    """Config 2 member i: the acceptance pattern (acceptance.cpp:525-547) scaled by W/320:
    2-4 curved lanes over [0.1W, 0.9W], gamma1 in {-0.1, 0, 0.1},
    gamma2 in +-{2.5e-4, 7.5e-4}, noise 0.02, seed 1 + i."""
    s = width / 320.0
    nl = 2 + i % 3
    start = (60.0 + (i % 4) * 8.0) * s
    span = 250.0 * s - start
    bottoms = tuple(start + span * k / (nl - 1) for k in range(nl))
    gamma = (width / 2 + ((i % 5) - 2) * 12.0 * s, ((i % 3) - 1) * 0.10,
             ((i % 4) - 1.5) * 5e-4, 0.0, 0.0)
    return abi.scene_params(width=width, height=height, beta=beta, gamma=gamma, d_max=d_max,
                            lane_bottoms=bottoms, noise_sigma=0.02, rng_seed=1 + i)


def stress_scene(i: int) -> abi.LkSceneParams:
    """Config 3: obstacles and a sudden pitch change (RANSAC outlier stress), 4 lanes."""
    W = KITTI_W
    boxes = [((150, 140, 420, 260), 45), ((820, 120, 1050, 230), 38),
             ((560, 110, 700, 170), 25), ((950, 200, 1200, 330), 60)]
    pitch = [(-1, 0.0), (200, 0.5), (250, 1.0), (230, -0.4)][i % 4]
    return abi.scene_params(width=W, height=KITTI_H, beta=BETA,
                            gamma=(W / 2, 0.05 * ((i % 3) - 1), 2.5e-4, 0, 0), d_max=255,
                            lane_bottoms=(0.15 * W, 0.38 * W, 0.62 * W, 0.85 * W),
                            noise_sigma=0.02, rng_seed=300 + i, obstacles=boxes[: 1 + i % 4],
                            pitch_row=pitch[0], pitch_jump=pitch[1])


def hires_scene(i: int) -> abi.LkSceneParams:
    """Config 4: 2560x1024 (SURVEY.md §7 hard part 7: beta below, d_max 248). The
    acceptance pattern's lane bottoms scale with W/320; the lane curvature is
    scaled to the taller frame (gamma2 by (W/320) / (H/240)^2, gamma1 = 0), so
    the reference itself finds the painted lanes (batch_scene's KITTI curvature
    at 1024 rows bends the lanes off the frame and the reference then selects
    16+ spurious lanes)."""
    W, H = HIRES_W, HIRES_H
    s, sv = W / 320.0, H / 240.0
    nl = 2 + i % 3
    start = (60.0 + (i % 4) * 8.0) * s
    span = 250.0 * s - start
    bottoms = tuple(start + span * k / (nl - 1) for k in range(nl))
    gamma = (W / 2 + ((i % 5) - 2) * 12.0 * s, 0.0, ((i % 4) - 1.5) * 5e-4 * s / (sv * sv), 0.0, 0.0)
    return abi.scene_params(width=W, height=H, beta=BETA, gamma=gamma, d_max=256,
                            lane_bottoms=bottoms, noise_sigma=0.02, rng_seed=1 + i)


def hires_config() -> abi.LkConfig:
    """d_max 248 (f(1023) = 242), lambda_g 1, and a lane separation scaled to the
    frame width (150 px; the default 20 px lets one painted lane yield several)."""
    return abi.default_config(d_max=248, lambda_g=1.0, min_lane_sep=150)


def acceptance_scene(i: int) -> abi.LkSceneParams:
    """acceptance.cpp:525-547 verbatim: 320x240, seeds 1100+i."""
    nl = 2 + i % 3
    start = 60.0 + (i % 4) * 8.0
    span = 250.0 - start
    bottoms = tuple(start + span * k / (nl - 1) for k in range(nl))
    gamma = (160.0 + ((i % 5) - 2) * 12.0, ((i % 3) - 1) * 0.10, ((i % 4) - 1.5) * 5e-4, 0, 0)
    return abi.scene_params(width=320, height=240, d_max=32, noise_sigma=0.02,
                            rng_seed=1100 + i, lane_bottoms=bottoms, gamma=gamma)


def acceptance_config() -> abi.LkConfig:
    """scene_config() (acceptance.cpp:549-566), lane-stage settings."""
    return abi.default_config(d_max=32, rho=4, sigma_floor=0.03, tr_lrc=1, nu=2, lambda_g=1.03)
