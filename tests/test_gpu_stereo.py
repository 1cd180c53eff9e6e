"""Stages 1-4 on the GPU (stereo pair in: the reference's run_pipeline) vs the
compiled reference and the restatement, through the C-ABI. Every stage 1-4
output is bit-exact (block statistics, both SRP maps, the LRC disparity), and
stages 5-12 on top of it match the reference run on the reference's own
disparity."""
import numpy as np
import pytest

from paper_1807_02752_b200 import abi, lanekit, scenes
from parity import compare_frame, compare_reports
from test_stereo import _cfg, _small_pair

pytestmark = pytest.mark.gpu

STEREO_HOOKS = ["STATS_MU", "STATS_SIGMA", "DISP_LEFT", "DISP_RIGHT", "DISPARITY"]


def _checker(oracle):
    from checkers import Checker, ref_available

    return Checker("ref") if ref_available() else oracle


def _run(pipe_kw, left, right, cfg):
    n, H, W = left.shape
    pipe = lanekit.GpuPipeline(W, H, cfg, max_batch=n, stereo=True, **pipe_kw)
    reps = pipe.run_stereo(left, right)
    return pipe, reps


def _compare(pipe, reps, left, right, cfg, chk, hooks):
    problems = []
    for i in range(left.shape[0]):
        o = chk.stereo(left[i], right[i], cfg)
        for k in STEREO_HOOKS:
            g = pipe.stage(i, k)
            if g.tobytes() != o[k].tobytes():
                problems.append(f"frame {i}: {k} not bit-exact "
                                f"({int((g != o[k]).sum())} of {g.size} differ)")
        r = chk.run(left[i], o["DISPARITY"], cfg)
        problems += [f"frame {i}: {x}" for x in compare_reports(reps[i], r.report)]
        problems += [f"frame {i}: {x}" for x in
                     compare_frame(lambda name: pipe.stage(i, name), r, hooks=hooks)]
    return problems


def test_stereo_small_frames(oracle):
    pairs = [_small_pair(s) for s in (1, 2, 3, 4)]
    left = np.stack([p[0] for p in pairs])
    right = np.stack([p[1] for p in pairs])
    cfg = _cfg(d_max=32)
    pipe, reps = _run({}, left, right, cfg)
    assert not (problems := _compare(pipe, reps, left, right, cfg, _checker(oracle), False)), \
        "\n".join(problems)


def test_stereo_kitti_size_with_hooks(oracle):
    params = [scenes.probe_scene(5), scenes.batch_scene(3)]
    left, right, _ = lanekit.synth_stereo_batch(params)
    cfg = abi.default_config()
    pipe, reps = _run({"hooks": True}, left, right, cfg)
    assert not (problems := _compare(pipe, reps, left, right, cfg, _checker(oracle), True)), \
        "\n".join(problems)
    assert reps[0].status == 0 and reps[0].lane_count >= 1


@pytest.mark.parametrize("kw", [dict(tau=0), dict(tau=3), dict(tr_lrc=0), dict(rho=2),
                                dict(rho=5), dict(sigma_floor=0.05)])
def test_stereo_config_variants(oracle, kw):
    pairs = [_small_pair(s) for s in (4, 6)]
    left = np.stack([p[0] for p in pairs])
    right = np.stack([p[1] for p in pairs])
    cfg = _cfg(d_max=32, **kw)
    pipe, reps = _run({}, left, right, cfg)
    assert not (problems := _compare(pipe, reps, left, right, cfg, _checker(oracle), False)), \
        "\n".join(problems)


def test_stereo_batch_pipelined_and_device_paths_agree(oracle):
    """64 KITTI pairs: the host-fed pipelined path (8 ranges) and the
    device-resident graph (4 branches) give identical reports and disparities,
    and they match the reference on a sample."""
    params = [scenes.batch_scene(i) for i in range(64)]
    left, right, _ = lanekit.synth_stereo_batch(params)
    cfg = abi.default_config()
    pipe, reps = _run({}, left, right, cfg)
    d_host = [pipe.stage(i, "DISPARITY").copy() for i in range(64)]
    L = lanekit.library()
    import ctypes as C
    dl, dr = C.c_void_p(), C.c_void_p()
    assert L.lk_stereo_inputs(pipe._h, C.byref(dl), C.byref(dr)) == 0
    assert L.lk_enqueue_stereo(pipe._h, 64) == 0
    reps2 = (abi.LkFrameReport * 64)()
    L.lk_fetch_reports(pipe._h, reps2, 64)
    for i in range(64):
        assert bytes(reps[i]) == bytes(reps2[i]), i
        assert np.array_equal(pipe.stage(i, "DISPARITY"), d_host[i]), i
    chk = _checker(oracle)
    for i in (0, 17, 63):
        o = chk.stereo(left[i], right[i], cfg)
        assert o["DISPARITY"].tobytes() == d_host[i].tobytes(), i


def test_stereo_run_pipeline_api():
    p = scenes.probe_scene(5)
    left, right, _, _ = lanekit.synth_scene(p)
    res = lanekit.run_pipeline(left, right, abi.default_config())
    assert res.report.status == 0
    assert res.stage("DISPARITY").shape == left.shape
    with pytest.raises(lanekit.StageError) as e:
        lanekit.run_pipeline(left[:5, :5], right[:5, :5], abi.default_config())
    assert "image smaller than the matching block" in str(e.value)


def test_stereo_exact_ties_take_the_fp64_path(oracle):
    """Identical pairs (NCC = +1 at d = 0 and wherever blocks repeat) and a
    horizontally periodic texture (exact ties every period) cannot be
    certified by the integer costs: the exact FP64 fallback must reproduce the
    reference's tie rule (smallest d)."""
    left, _, _ = _small_pair(3)
    rng = np.random.default_rng(7)
    period = np.tile(rng.integers(0, 256, (120, 8), dtype=np.uint8), (1, 40))  # 120 x 320
    shifted = np.roll(period, -5, axis=1)
    L = np.stack([left, period])
    R = np.stack([left, shifted])
    cfg = _cfg(d_max=32)
    pipe, reps = _run({}, L, R, cfg)
    chk = _checker(oracle)
    for i in range(2):
        o = chk.stereo(L[i], R[i], cfg)
        for k in STEREO_HOOKS:
            assert pipe.stage(i, k).tobytes() == o[k].tobytes(), (i, k)
    assert not pipe.stage(0, "DISP_LEFT").any()  # identical pair: d = 0 everywhere


def test_stereo_hires_frame(oracle):
    """2560x1024 with d_max 248 (config 4): rows wider than the register
    prefetch, the largest shared-memory windows, u8 disparities near 255."""
    p = scenes.hires_scene(3)
    left, right, _ = lanekit.synth_stereo_batch([p])
    cfg = scenes.hires_config()
    pipe, reps = _run({}, left, right, cfg)
    chk = _checker(oracle)
    o = chk.stereo(left[0], right[0], cfg)
    for k in STEREO_HOOKS:
        assert pipe.stage(0, k).tobytes() == o[k].tobytes(), k
    r = chk.run(left[0], o["DISPARITY"], cfg)
    assert not compare_reports(reps[0], r.report)


def test_stereo_streaming_submit_matches_run_stereo_batch():
    """lk_submit_stereo_batch / lk_wait_batch: stereo pairs through the two
    input slots (the right image in its own slot buffers) give the same reports
    as lk_run_stereo_batch, across slot reuse, the auto-wait of a third
    submit, and a mono submit interleaved on the same context."""
    import ctypes as C

    cfg = abi.default_config()
    batches = []
    for b in range(4):
        params = [scenes.batch_scene(300 + 8 * b + i) for i in range(8)]
        left, right, _ = lanekit.synth_stereo_batch(params)
        batches.append((np.ascontiguousarray(left), np.ascontiguousarray(right)))
    with lanekit.GpuPipeline(1242, 375, cfg, max_batch=8, stereo=True) as pipe:
        want = [[bytes(r) for r in pipe.run_stereo(l, r)] for l, r in batches]
        L = lanekit.library()
        got = [(abi.LkFrameReport * 8)() for _ in batches]
        for b, (l, r) in enumerate(batches):
            st = L.lk_submit_stereo_batch(pipe._h, l.ctypes.data, r.ctypes.data, 8, got[b])
            assert st == abi.LK_OK, L.lk_last_error()
        assert L.lk_wait_batch(pipe._h) in (abi.LK_OK, abi.LK_ERR_FRAME)
        assert L.lk_wait_batch(pipe._h) in (abi.LK_OK, abi.LK_ERR_FRAME)
        for b in range(4):
            assert [bytes(x) for x in got[b]] == want[b], b
        # a mono batch (grey + the disparity of batch 0) on the same slots afterwards
        disp0 = np.stack([pipe.stage(i, "DISPARITY") for i in range(8)])  # from the last run_stereo
        mono = (abi.LkFrameReport * 8)()
        g = np.ascontiguousarray(batches[3][0])
        dd = np.ascontiguousarray(disp0)
        assert L.lk_submit_batch(pipe._h, g.ctypes.data, dd.ctypes.data, 8, mono) == abi.LK_OK
        assert L.lk_wait_batch(pipe._h) in (abi.LK_OK, abi.LK_ERR_FRAME)
        for i in range(8):  # same grey + same disparity -> the stereo batch's lanes
            assert mono[i].lane_count == got[3][i].lane_count, i
