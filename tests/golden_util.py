"""Loader for tests/golden/golden.json (written by tests/golden/make_golden.py
from the compiled reference). Rebuilds scene params / configs, regenerates the
8-bit inputs with the repo's generator and checks them against the pinned
SHA-256s."""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

from paper_1807_02752_b200 import abi

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.json"


def dec(x):
    if isinstance(x, str):
        if x in ("nan", "inf", "-inf"):
            return float(x)
        return float.fromhex(x)
    if isinstance(x, list):
        return [dec(v) for v in x]
    return x


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def load_cases() -> list[dict]:
    return json.loads(GOLDEN.read_text())["cases"]


def case_ids() -> list[str]:
    return [c["name"] for c in load_cases()]


def scene_params(case) -> abi.LkSceneParams:
    s = case["scene"]
    p = abi.LkSceneParams()
    for name, _ in p._fields_:
        v = s[name]
        if name == "obstacle_box":
            for i in range(4):
                for k in range(4):
                    p.obstacle_box[i][k] = v[i][k]
        elif isinstance(v, list):
            arr = getattr(p, name)
            for i, x in enumerate(v):
                arr[i] = dec(x)
        else:
            setattr(p, name, dec(v))
    return p


def config(case) -> abi.LkConfig:
    c = abi.LkConfig()
    for k, v in case["config"].items():
        setattr(c, k, dec(v))
    return c


def apply_mutation(mutate, grey, disp):
    """The failure cases' input edits (in place), shared with make_golden.py."""
    if mutate == "zero_disparity":
        disp[:] = 0
    elif mutate == "flat_grey":
        grey[:] = 128
    elif mutate == "disparity_one_below_120":
        disp[:] = 0
        disp[120:] = 1
    elif mutate == "disparity_row150_d10":
        disp[:] = 0
        disp[150, :] = 10
    elif mutate is not None:
        raise ValueError(f"unknown mutation {mutate}")


def inputs(case):
    """Regenerates the case's grey / disparity with the repo generator and
    checks them against the reference's bytes (SHA-256)."""
    from paper_1807_02752_b200 import lanekit

    p = scene_params(case)
    grey, _, disp, _ = lanekit.synth_scene(p)
    apply_mutation(case["mutate"], grey, disp)
    assert sha(grey.tobytes()) == case["grey_sha256"], "generator drifted (grey)"
    assert sha(disp.tobytes()) == case["disp_sha256"], "generator drifted (disparity)"
    return grey, disp


def report_expected(case) -> dict:
    return {k: dec(v) for k, v in case["report"].items()}


def same_float(a: float, b: float) -> bool:
    return (np.isnan(a) and np.isnan(b)) or a == b
