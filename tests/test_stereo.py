"""Stages 1-4 (stereo.hpp): the oracle restatement against the compiled
reference (bit for bit), and the reference's own stereo unit tests
(tests/test_stereo.cpp) re-expressed on the restatement. CPU only."""
import numpy as np
import pytest

from paper_1807_02752_b200 import abi, lanekit, scenes


def _small_pair(seed, W=320, H=120, **kw):
    p = scenes.probe_scene(seed) if not kw else scenes.probe_scene(seed)
    p.width, p.height = W, H
    p.beta[0], p.beta[1], p.beta[2] = -15.0 * H / 375, 0.15, 1e-4 * 375 / H
    p.gamma[0] = W / 2
    for k, v in kw.items():
        setattr(p, k, v)
    left, right, disp, _ = lanekit.synth_scene(p)
    return left, right, disp


def _cfg(**kw):
    c = abi.default_config()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_stereo_restatement_matches_reference(oracle, ref, seed):
    left, right, _ = _small_pair(seed)
    cfg = _cfg(d_max=32)
    a, b = oracle.stereo(left, right, cfg), ref.stereo(left, right, cfg)
    for k in a:
        assert a[k].tobytes() == b[k].tobytes(), k
    assert (a["DISPARITY"] != 0).mean() > 0.3  # the pair actually matches


def test_stereo_restatement_matches_reference_kitti_size(oracle, ref):
    p = scenes.probe_scene(5)
    left, right, _, _ = lanekit.synth_scene(p)
    cfg = _cfg()
    a, b = oracle.stereo(left, right, cfg), ref.stereo(left, right, cfg)
    for k in a:
        assert a[k].tobytes() == b[k].tobytes(), k


@pytest.mark.parametrize("kw", [dict(tau=0), dict(tau=3), dict(tr_lrc=0), dict(rho=2),
                                dict(sigma_floor=0.05)])
def test_stereo_config_variants_match_reference(oracle, ref, kw):
    left, right, _ = _small_pair(4)
    cfg = _cfg(d_max=32, **kw)
    a, b = oracle.stereo(left, right, cfg), ref.stereo(left, right, cfg)
    for k in a:
        assert a[k].tobytes() == b[k].tobytes(), (kw, k)


def test_flat_blocks_stay_invalid(oracle):
    # test_stereo.cpp:119-127: a flat image has sigma 0 < floor everywhere
    flat = np.full((40, 60), 128, np.uint8)
    out = oracle.stereo(flat, flat, _cfg(d_max=16))
    assert not out["DISP_LEFT"].any() and not out["DISPARITY"].any()


def test_border_blocks_unmatchable(oracle):
    # test_stereo.cpp:28-41: mu = sigma = 0 where the block leaves the image
    left, right, _ = _small_pair(2)
    out = oracle.stereo(left, right, _cfg(d_max=32))
    rho = 3
    for k in ("STATS_MU", "STATS_SIGMA"):
        m = out[k]
        assert not m[:rho].any() and not m[-rho:].any()
        assert not m[:, :rho].any() and not m[:, -rho:].any()


def test_identical_pair_gives_zero_disparity(oracle):
    # NCC of a block with itself is +1, the maximum: d = 0 wins (smallest d on ties)
    left, _, _ = _small_pair(3)
    out = oracle.stereo(left, left, _cfg(d_max=16))
    assert not out["DISP_LEFT"].any() and not out["DISP_RIGHT"].any()


def test_full_pipeline_composition(oracle, ref):
    # run_pipeline = stages 1-4 then stages 5-12 on the LRC disparity with the left grey
    p = scenes.probe_scene(5)
    left, right, _, _ = lanekit.synth_scene(p)
    cfg = _cfg()
    disp = ref.stereo(left, right, cfg)["DISPARITY"]
    r = ref.run(left, disp, cfg)
    rep = r.report
    assert rep.status == 0
    assert rep.valid_disparities == int((disp != 0).sum())
