"""C-ABI checks that need no GPU: the library loads, exports every entry point
include/lanekit_b200.h declares, struct layouts match the ctypes mirror, config
validation mirrors config.hpp:124-152, and the product path fails loudly (no
CPU fallback) when no Blackwell device is present."""
import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1807_02752_b200 import abi, lanekit

HEADER = Path(__file__).resolve().parents[1] / "include" / "lanekit_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lk_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol():
    L = lanekit.library()
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_struct_layouts_match():
    sizes = (C.c_size_t * 6)()
    lanekit.library().lk_abi_sizes(sizes)
    assert list(sizes) == [C.sizeof(abi.LkConfig), C.sizeof(abi.LkFrameReport),
                           C.sizeof(abi.LkSceneParams), C.sizeof(abi.LkEdge),
                           C.sizeof(abi.LkVote), C.sizeof(abi.LkLane)]


def test_abi_version_and_stage_names():
    L = lanekit.library()
    assert L.lk_abi_version() == 1
    for i, name in enumerate(abi.STAGE_NAMES, start=1):
        assert L.lk_stage_name(i).decode() == name  # pipeline.hpp:101-116


def test_default_config_matches_reference_defaults():
    L = lanekit.library()
    c = abi.LkConfig()
    L.lk_config_default.argtypes = [C.POINTER(abi.LkConfig)]
    L.lk_config_default(C.byref(c))
    py = abi.default_config()
    for name, _ in c._fields_:
        a, b = getattr(c, name), getattr(py, name)
        assert (math.isnan(a) and math.isnan(b)) or a == b, name
    assert c.d_max == 64 and c.sigma_s == 300.0 and c.bf_window == 11 and math.isnan(c.tr_lpv)


@pytest.mark.parametrize("field,value,message", [
    ("d_max", 0, "config: d_max must be >= 1"),
    ("bf_window", 10, "config: bf_window must be odd and >= 1"),
    ("eps_y", 1.5, "config: eps_y must be in (0, 1]"),
    ("tr_lpv", 1.0, "config: tr_lpv must be negative (or auto)"),
    ("rho_vote", 0.0, "config: rho_vote must be > 0"),
    ("sigma_r", 0.0, "config: sigma_r must be > 0"),
    ("min_lane_sep", -1, "config: min_lane_sep must be >= 0"),
])
def test_validate_config_messages(field, value, message):
    """config.hpp:124-152: same checks, same messages."""
    cfg = abi.default_config(**{field: value})
    with pytest.raises(lanekit.LanekitError) as ei:
        lanekit.validate_config(cfg)
    assert ei.value.status == abi.LK_ERR_CONFIG
    assert str(ei.value) == message


def test_frame_message_rendering():
    rep = abi.LkFrameReport(status=abi.LK_ERR_FRAME, failed_stage=7, msg=5, err_row=12)
    L = lanekit.library()
    buf = C.create_string_buffer(256)
    L.lk_frame_message.argtypes = [C.POINTER(abi.LkFrameReport), C.c_char_p, C.c_size_t]
    assert L.lk_frame_message(C.byref(rep), buf, 256) == 0
    text = "stage 7 (road profile fit): road profile: singular V_py derivative at row 12"
    assert buf.value.decode() == text == abi.frame_message(rep)


def test_no_cpu_fallback_without_gpu():
    """The product path must fail loudly when no sm_100 device is visible."""
    from conftest import gpu_available

    if gpu_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(lanekit.LanekitError) as ei:
        lanekit.GpuPipeline(64, 48, abi.default_config())
    assert ei.value.status in (abi.LK_ERR_NO_DEVICE, abi.LK_ERR_CUDA)


def test_synth_matches_reference_generator(ref):
    """The repo's gen_scene restatement (synth.cpp) is byte-identical to the
    reference's gen_scene + write_png_gray quantisation (synth.hpp:103-200)."""
    for p in [abi.scene_params(width=320, height=240, d_max=32, noise_sigma=0.02, rng_seed=12,
                               gamma=(160.0, 0, 0, 0, 0), lane_bottoms=(110.0, 210.0)),
              abi.scene_params(noise_sigma=0.0),
              abi.scene_params(beta=(-75.0, 0.5, 0.0), gamma=(320.0, 0, 0, 0, 0),
                               lane_bottoms=(200.0, 440.0))]:
        a = lanekit.synth_scene(p)
        b = ref.gen_scene(p)
        for x, y in zip(a[:3], b[:3]):
            assert np.array_equal(x, y)
        assert a[3] == b[3]


def test_synth_rejects_infeasible_scenes():
    """test_synth.cpp:56-68."""
    with pytest.raises(ValueError, match="no horizon"):
        lanekit.synth_scene(abi.scene_params(beta=(0.0, 0.0, 0.0)))
    with pytest.raises(ValueError, match="leaves"):
        lanekit.synth_scene(abi.scene_params(d_max=40))
    with pytest.raises(ValueError, match="too small"):
        lanekit.synth_scene(abi.scene_params(width=8))


def test_synth_deterministic_and_seeded():
    """test_synth.cpp:39-54."""
    p = abi.scene_params(width=320, height=240, noise_sigma=0.02, rng_seed=77)
    a, b = lanekit.synth_scene(p), lanekit.synth_scene(p)
    assert all(np.array_equal(x, y) for x, y in zip(a[:3], b[:3]))
    p.rng_seed = 78
    assert not np.array_equal(a[0], lanekit.synth_scene(p)[0])


def test_synth_batch_equals_single(ref):
    from paper_1807_02752_b200 import scenes

    params = [scenes.acceptance_scene(i) for i in range(4)]
    g, d = lanekit.synth_batch(params, threads=4)
    for i, p in enumerate(params):
        left, _, disp, _ = lanekit.synth_scene(p)
        assert np.array_equal(g[i], left) and np.array_equal(d[i], disp)
