"""GPU path vs the CPU oracle, hook by hook, through the C-ABI.

Integer outputs bit-exact, FP outputs within 1e-5 relative (tests/parity.py).
Covers the probe scene (config 1), config-2 batch members, the obstacle /
pitch-change stress scenes (config 3), the acceptance family at 320x240,
and failure paths (StageError numbers and messages)."""
import numpy as np
import pytest

from paper_1807_02752_b200 import abi, lanekit, scenes
from parity import compare_frame, compare_reports

pytestmark = pytest.mark.gpu


def _run_and_compare(oracle, params, cfg, hooks=True):
    grey, disp = lanekit.synth_batch(params, threads=8)
    n, H, W = grey.shape
    with lanekit.GpuPipeline(W, H, cfg, max_batch=n, hooks=hooks) as pipe:
        reps = pipe.run(grey, disp)
        problems = []
        for i in range(n):
            o = oracle.run(grey[i], disp[i], cfg)
            p = compare_reports(reps[i], o.report)
            p += compare_frame(lambda name: pipe.stage(i, name), o, hooks=hooks)
            problems += [f"frame {i}: {x}" for x in p]
        return reps, problems


def test_probe_scene_all_hooks(oracle):
    reps, problems = _run_and_compare(oracle, [scenes.probe_scene()], abi.default_config())
    assert not problems, "\n".join(problems)
    assert reps[0].status == 0
    assert sorted(reps[0].as_dict()["lane_bottom_col"]) == [370, 767]


def test_config2_members(oracle):
    params = [scenes.batch_scene(i) for i in range(6)]
    reps, problems = _run_and_compare(oracle, params, abi.default_config())
    assert not problems, "\n".join(problems)


def test_ransac_heavy_frames(oracle):
    """Config-2 members whose RANSAC-gamma runs 83-181 iterations (speculative
    multi-warp commit must reproduce the serial trimming exactly)."""
    params = [scenes.batch_scene(i) for i in (92, 199, 68, 159, 25, 206)]
    reps, problems = _run_and_compare(oracle, params, abi.default_config())
    assert not problems, "\n".join(problems)
    assert max(r.gamma_iterations for r in reps) == 181


def test_batch_reports_64(oracle):
    """64-frame batch without hooks: every report field vs the oracle."""
    params = [scenes.batch_scene(i) for i in range(64)]
    grey, disp = lanekit.synth_batch(params, threads=8)
    cfg = abi.default_config()
    with lanekit.GpuPipeline(1242, 375, cfg, max_batch=64) as pipe:
        reps = pipe.run(grey, disp)
        orc = oracle.run_batch(grey, disp, cfg, threads=8)
        problems = [f"frame {i}: {x}" for i in range(64) for x in compare_reports(reps[i], orc[i])]
    assert not problems, "\n".join(problems)


def test_stress_obstacles_pitch(oracle):
    params = [scenes.stress_scene(i) for i in range(4)]
    reps, problems = _run_and_compare(oracle, params, abi.default_config())
    assert not problems, "\n".join(problems)


def test_acceptance_family(oracle):
    params = [scenes.acceptance_scene(i) for i in range(20)]
    reps, problems = _run_and_compare(oracle, params, scenes.acceptance_config())
    assert not problems, "\n".join(problems)


def test_no_hooks_mode_matches(oracle):
    params = [scenes.batch_scene(i) for i in range(3)]
    reps, problems = _run_and_compare(oracle, params, abi.default_config(), hooks=False)
    assert not problems, "\n".join(problems)


@pytest.mark.parametrize("size", [(1241, 373), (333, 251)])
def test_odd_sizes_fast_path(oracle, size):
    """Odd widths and heights through the throughput path (no hooks): partial
    tiles, the mirrored staging fallbacks and unaligned rows vs the oracle."""
    W, H = size
    params = [scenes.batch_scene(i, width=W, height=H) for i in range(3)]
    reps, problems = _run_and_compare(oracle, params, abi.default_config(), hooks=False)
    assert not problems, "\n".join(problems)
    assert all(r.status == 0 for r in reps)


def test_paper_sign_and_manual_threshold(oracle):
    params = [scenes.batch_scene(i) for i in range(2)]
    cfg = abi.default_config(paper_sign=True, tr_lpv=-400.0, lambda_g=0.98, nu=2, chi=10)
    reps, problems = _run_and_compare(oracle, params, cfg)
    assert not problems, "\n".join(problems)


@pytest.mark.parametrize("l2_min", ["0", "4294967295"])
def test_p99_selection_paths(oracle, monkeypatch, l2_min):
    """The exact p99 (lanes.hpp:182-193) through both GPU selection paths:
    always with the second histogram level, and never."""
    monkeypatch.setenv("LK_P99_L2_MIN", l2_min)
    params = [scenes.batch_scene(i) for i in (3, 11)] + [scenes.acceptance_scene(5)]
    for p, cfg in [(params[:2], abi.default_config(sobel_threshold=20.0, nu=3)),
                   (params[2:], scenes.acceptance_config())]:
        reps, problems = _run_and_compare(oracle, p, cfg, hooks=False)
        assert not problems, "\n".join(problems)


def test_stage6_no_road_evidence(oracle):
    """Identical views -> empty disparity -> StageError 6 (test_pipeline.cpp:119-127)."""
    grey, disp = lanekit.synth_batch([scenes.acceptance_scene(0)])
    disp[:] = 0
    with pytest.raises(lanekit.StageError) as ei:
        lanekit.run_pipeline_from_disparity(grey[0], disp[0], scenes.acceptance_config())
    assert ei.value.stage == 6
    assert ei.value.stage_name == "road path extraction"
    assert str(ei.value) == ("stage 6 (road path extraction): v-disparity histogram is empty; "
                             "no road surface evidence")
    o = oracle.run(grey[0], disp[0], scenes.acceptance_config())
    assert o.report.failed_stage == 6


def test_failed_frame_does_not_abort_batch(oracle):
    params = [scenes.acceptance_scene(i) for i in range(3)]
    grey, disp = lanekit.synth_batch(params)
    disp[1] = 0
    cfg = scenes.acceptance_config()
    with lanekit.GpuPipeline(320, 240, cfg, max_batch=3, hooks=True) as pipe:
        reps = pipe.run(grey, disp)
        assert reps[1].status == abi.LK_ERR_FRAME and reps[1].failed_stage == 6
        for i in (0, 2):
            o = oracle.run(grey[i], disp[i], cfg)
            assert not compare_reports(reps[i], o.report)
            assert not compare_frame(lambda n: pipe.stage(i, n), o)


def test_stage11_no_edge_evidence(oracle):
    """A flat frame has no edges: StageError 11 (pipeline.hpp:238-239)."""
    grey, disp = lanekit.synth_batch([scenes.acceptance_scene(0)])
    grey[:] = 128
    cfg = scenes.acceptance_config()
    with lanekit.GpuPipeline(320, 240, cfg, max_batch=1) as pipe:
        rep = pipe.run(grey, disp)[0]
    o = oracle.run(grey[0], disp[0], cfg)
    assert o.report.failed_stage == 11
    assert not compare_reports(rep, o.report)
    assert abi.frame_message(rep).startswith("stage 11 (vanishing point estimation): ")


def test_determinism_and_batch_invariance(oracle):
    """Criterion 12 analogue: reruns and different batch compositions are bit-identical."""
    params = [scenes.batch_scene(i) for i in range(4)]
    grey, disp = lanekit.synth_batch(params)
    cfg = abi.default_config()
    with lanekit.GpuPipeline(1242, 375, cfg, max_batch=4) as pipe:
        a = [r.as_dict() for r in pipe.run(grey, disp)]
        ea = [pipe.stage(i, "ENERGY").copy() for i in range(4)]
        b = [r.as_dict() for r in pipe.run(grey, disp)]
        c = [r.as_dict() for r in pipe.run(grey[2:3], disp[2:3])]
        ec = pipe.stage(0, "ENERGY")
    assert a == b
    assert a[2] == c[0]
    assert np.array_equal(ea[2], ec)


def test_direct_launch_matches_graph(oracle):
    params = [scenes.batch_scene(i) for i in range(2)]
    grey, disp = lanekit.synth_batch(params)
    cfg = abi.default_config()
    with lanekit.GpuPipeline(1242, 375, cfg, max_batch=2, graph=False) as p1:
        a = [r.as_dict() for r in p1.run(grey, disp)]
        t = p1.stage_times()
    with lanekit.GpuPipeline(1242, 375, cfg, max_batch=2) as p2:
        b = [r.as_dict() for r in p2.run(grey, disp)]
    assert a == b
    assert t[0] > 0 and t[9] > 0


def test_streaming_submit_wait_matches_run_batch():
    """lk_submit_batch / lk_wait_batch (two input slots, copies overlapping the
    previous batch's kernels): every batch's reports equal lk_run_batch's on
    the same frames, across slot reuse and the auto-wait of a third submit."""
    import ctypes as C

    cfg = abi.default_config()
    batches = []
    for b in range(4):
        params = [scenes.batch_scene(100 + 16 * b + i) for i in range(16)]
        batches.append(lanekit.synth_batch(params, threads=8))
    with lanekit.GpuPipeline(1242, 375, cfg, max_batch=16) as pipe:
        want = [[bytes(r) for r in pipe.run(g, d)] for g, d in batches]
        L = lanekit.library()
        got = [(abi.LkFrameReport * 16)() for _ in batches]
        keep = [(np.ascontiguousarray(g), np.ascontiguousarray(d)) for g, d in batches]
        for b, (g, d) in enumerate(keep):  # the third submit waits for the first
            st = L.lk_submit_batch(pipe._h, g.ctypes.data, d.ctypes.data, 16, got[b])
            assert st == abi.LK_OK, L.lk_last_error()
        assert L.lk_wait_batch(pipe._h) in (abi.LK_OK, abi.LK_ERR_FRAME)
        assert L.lk_wait_batch(pipe._h) in (abi.LK_OK, abi.LK_ERR_FRAME)
        assert L.lk_wait_batch(pipe._h) == abi.LK_ERR_INVALID_ARGUMENT  # nothing pending
        for b in range(4):
            assert [bytes(r) for r in got[b]] == want[b], b


def test_streaming_road_copy_matches_run_batch():
    """lk_submit_batch from pinned buffers copies the disparity, runs stages 5-7
    of the batch on a side stream and copies only the grey rows from the
    chunk's smallest horizon - 1 - rho down. The rows above stay stale in the
    slot (here: noise from an earlier batch), so reports and the throughput-mode
    hooks must still equal lk_run_batch's, on lane, stress (horizons 81..177),
    stage-6 and stage-11 failure frames; lk_h2d_bytes counts exactly the
    disparity plus those rows."""
    import ctypes as C

    from golden_util import apply_mutation

    cfg = abi.default_config()
    n, W, H = 8, 1242, 375
    px = W * H
    batches = []
    for b in range(3):
        params = [scenes.batch_scene(300 + 8 * b + i) for i in range(4)] + \
                 [scenes.stress_scene(i) for i in range(4)]
        g, d = lanekit.synth_batch(params, threads=8)
        g, d = g.copy(), d.copy()
        if b == 1:
            apply_mutation("zero_disparity", g[2], d[2])
            apply_mutation("flat_grey", g[5], d[5])
        batches.append((g, d))
    noise = np.random.default_rng(7).integers(0, 256, size=(n, H, W), dtype=np.uint8)
    L = lanekit.library()
    with lanekit.GpuPipeline(W, H, cfg, max_batch=n) as pipe:
        want, want_hooks = [], []
        for g, d in batches:
            reps = pipe.run(g, d)
            want.append([bytes(r) for r in reps])
            want_hooks.append({(i, k): pipe.stage(i, k).tobytes() for i in range(n)
                               for k in ("LANES", "ENERGY", "VOTES", "EDGES") if reps[i].status == 0})
        pipe.run(noise, batches[0][1])  # slot 0's grey: noise above every horizon
        bufs = []
        for g, d in batches:
            pg, pd = C.c_void_p(), C.c_void_p()
            assert L.lk_host_alloc(C.byref(pg), g.nbytes) == abi.LK_OK
            assert L.lk_host_alloc(C.byref(pd), d.nbytes) == abi.LK_OK
            C.memmove(pg, g.ctypes.data, g.nbytes)
            C.memmove(pd, d.ctypes.data, d.nbytes)
            bufs.append((pg, pd))
        got = [(abi.LkFrameReport * n)() for _ in batches]
        h0, h1 = C.c_ulonglong(0), C.c_ulonglong(0)
        assert L.lk_h2d_bytes(pipe._h, C.byref(h0)) == abi.LK_OK
        for b, (pg, pd) in enumerate(bufs):  # the third submit waits for the first
            assert L.lk_submit_batch(pipe._h, pg, pd, n, got[b]) == abi.LK_OK, L.lk_last_error()
        for _ in batches[1:]:
            assert L.lk_wait_batch(pipe._h) in (abi.LK_OK, abi.LK_ERR_FRAME)
        assert L.lk_h2d_bytes(pipe._h, C.byref(h1)) == abi.LK_OK
        for b in range(len(batches)):
            assert [bytes(r) for r in got[b]] == want[b], b
        last = len(batches) - 1
        pipe.reports = list(got[last])  # stage() decodes with the last batch's horizons
        for (i, k), v in want_hooks[last].items():
            assert pipe.stage(i, k).tobytes() == v, (i, k)
        expect = 0
        for b in range(len(batches)):
            rows = [H if (r.status and r.failed_stage <= 7) else min(max(int(r.horizon) - 6, 0), H)
                    for r in got[b]]
            expect += n * px
            for c0 in range(0, n, 4):  # two chunks of 4 frames (LK_ROAD_CHUNKS = 2)
                expect += 4 * (H - min(rows[c0:c0 + 4])) * W
        assert h1.value - h0.value == expect
        assert expect < 2 * px * n * len(batches)  # rows above the horizons were not copied
        for pg, pd in bufs:
            L.lk_host_free(pg)
            L.lk_host_free(pd)


def test_headline_batch_256_vs_reference(oracle):
    """All 256 frames of the bench's config-2 batch (batch_scene seeds 1..256,
    bench.py make_frames) through the throughput path in one batch, against
    the reference's own code (oracle/_ref; the restatement when it is absent):
    every report field, plus the LANES, ENERGY, M1, VOTES, UPATH and the other
    throughput-mode hooks of every frame (tests/parity.py rules)."""
    from concurrent.futures import ThreadPoolExecutor

    from checkers import Checker, ref_available

    chk = Checker("ref") if ref_available() else oracle
    params = [scenes.batch_scene(1 + i) for i in range(256)]
    grey, disp = lanekit.synth_batch(params, threads=8)
    cfg = abi.default_config()
    problems = []
    with lanekit.GpuPipeline(1242, 375, cfg, max_batch=256) as pipe, \
            ThreadPoolExecutor(8) as pool:
        reps = pipe.run(grey, disp)
        for c0 in range(0, 256, 16):  # ctypes drops the GIL: checker frames run in parallel
            res = list(pool.map(lambda i: chk.run(grey[i], disp[i], cfg), range(c0, c0 + 16)))
            for i, o in zip(range(c0, c0 + 16), res):
                p = compare_reports(reps[i], o.report)
                p += compare_frame(lambda name: pipe.stage(i, name), o, hooks=False)
                problems += [f"frame {i}: {x}" for x in p]
            del res
    assert not problems, "\n".join(problems[:20])
    assert all(r.status == 0 for r in reps)
    assert [r.uncertain for r in reps] == [0] * 256  # every lane decision certified


def test_stress_batch_64_vs_reference(oracle):
    """Config 3 at batch scale: 64 obstacle / pitch-change frames (stress_scene
    seeds 300..363, all four pitch variants, 1-4 obstacle boxes) through the
    throughput path in one batch, against the reference's own code: every
    report field and the throughput-mode hooks, and every lane decision
    certified."""
    from concurrent.futures import ThreadPoolExecutor

    from checkers import Checker, ref_available

    chk = Checker("ref") if ref_available() else oracle
    params = [scenes.stress_scene(i) for i in range(64)]
    grey, disp = lanekit.synth_batch(params, threads=8)
    cfg = abi.default_config()
    problems = []
    with lanekit.GpuPipeline(1242, 375, cfg, max_batch=64) as pipe, ThreadPoolExecutor(8) as pool:
        reps = pipe.run(grey, disp)
        for c0 in range(0, 64, 16):
            res = list(pool.map(lambda i: chk.run(grey[i], disp[i], cfg), range(c0, c0 + 16)))
            for i, o in zip(range(c0, c0 + 16), res):
                p = compare_reports(reps[i], o.report)
                p += compare_frame(lambda name: pipe.stage(i, name), o, hooks=False)
                problems += [f"frame {i}: {x}" for x in p]
            del res
    assert not problems, "\n".join(problems[:20])
    assert [r.uncertain for r in reps] == [0] * 64


def test_hires_batch_8_vs_reference(oracle):
    """Config 4 (2560x1024, d_max 248, lambda_g 1, lane separation 150): eight
    frames in one throughput-mode batch against the reference's own code,
    every report field and the throughput-mode hooks."""
    from concurrent.futures import ThreadPoolExecutor

    from checkers import Checker, ref_available

    chk = Checker("ref") if ref_available() else oracle
    params = [scenes.hires_scene(i) for i in range(8)]
    grey, disp = lanekit.synth_batch(params, threads=8)
    cfg = scenes.hires_config()
    with lanekit.GpuPipeline(2560, 1024, cfg, max_batch=8) as pipe, ThreadPoolExecutor(8) as pool:
        reps = pipe.run(grey, disp)
        res = list(pool.map(lambda i: chk.run(grey[i], disp[i], cfg), range(8)))
        problems = []
        for i, o in enumerate(res):
            p = compare_reports(reps[i], o.report)
            p += compare_frame(lambda name: pipe.stage(i, name), o, hooks=False)
            problems += [f"frame {i}: {x}" for x in p]
    assert not problems, "\n".join(problems[:20])
    assert all(r.status == 0 and r.lane_count >= 2 for r in reps)


def test_certificate_zero_on_batch_and_fires_on_a_tie(oracle):
    """lk_frame_report.uncertain: 0 on config-2 and stress frames (no lane
    decision within the libdevice-vs-glibc error bounds), and > 0 when the
    threshold is set exactly to a touched minimum's energy (a tie the
    transcendental error bound cannot resolve)."""
    params = [scenes.batch_scene(i) for i in range(8)] + [scenes.stress_scene(i) for i in range(4)]
    grey, disp = lanekit.synth_batch(params, threads=8)
    cfg = abi.default_config()
    with lanekit.GpuPipeline(1242, 375, cfg, max_batch=len(params)) as pipe:
        reps = pipe.run(grey, disp)
        assert [r.uncertain for r in reps] == [0] * len(params)
        e = pipe.stage(0, "ENERGY")
    tie = float(e.min())  # the deepest minimum: a touched column with negative energy
    assert tie < 0
    cfg2 = abi.default_config(tr_lpv=tie)
    with lanekit.GpuPipeline(1242, 375, cfg2, max_batch=1) as pipe:
        r = pipe.run(grey[:1], disp[:1])[0]
    assert r.uncertain >= 1
    o = oracle.run(grey[0], disp[0], cfg2)
    assert o.report.uncertain == 0  # (the CPU checkers never flag)
