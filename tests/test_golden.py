"""The CPU oracle against the reference's own outputs (tests/golden/golden.json).

The fixtures were produced by the compiled reference (oracle/_ref); here the
restatement must reproduce every report field and every hook BIT FOR BIT,
including the full-frame float maps (checked by SHA-256)."""
import numpy as np
import pytest

from golden_util import case_ids, config, inputs, load_cases, report_expected, same_float, sha
from paper_1807_02752_b200 import abi

CASES = {c["name"]: c for c in load_cases()}


@pytest.mark.parametrize("name", case_ids())
def test_oracle_matches_reference_golden(oracle, name):
    case = CASES[name]
    grey, disp = inputs(case)
    res = oracle.run(grey, disp, config(case))
    got = res.report.as_dict()
    want = report_expected(case)
    for k, v in want.items():
        g = got[k]
        if isinstance(v, list):
            assert len(g) == len(v) and all(same_float(float(a), float(b)) for a, b in zip(g, v)), k
        elif isinstance(v, float):
            assert same_float(float(g), v), f"{k}: {g!r} vs {v!r}"
        else:
            assert g == v, f"{k}: {g} vs {v}"
    for hook, h in case["hooks"].items():
        raw = res.raw(abi.STAGE[hook])
        assert len(raw) == h["nbytes"], hook
        assert sha(raw) == h["sha256"], f"{hook} differs from the reference"


def test_golden_covers_failures_and_configs():
    names = set(CASES)
    assert {"fail_stage6_no_disparity", "fail_stage11_flat_grey", "hires_5",
            "batch_92_gamma181", "fail_stage7_few_points", "fail_stage7_no_fit"} <= names
    assert CASES["fail_stage6_no_disparity"]["report"]["failed_stage"] == 6
    assert CASES["fail_stage11_flat_grey"]["report"]["failed_stage"] == 11
    assert CASES["fail_stage7_few_points"]["report"]["failed_stage"] == 7
    assert CASES["fail_stage7_no_fit"]["report"]["failed_stage"] == 7
    assert CASES["fail_stage7_few_points"]["report"]["msg"] != CASES["fail_stage7_no_fit"]["report"]["msg"]
    # the hi-res case is a lane scene: the reference finds the 4 painted lanes
    assert CASES["hires_5"]["report"]["lane_count"] == 4
    assert CASES["probe_kitti"]["report"]["lane_bottom_col"] == [767, 370]  # SURVEY.md §6 probe
