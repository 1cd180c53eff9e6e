"""lanedet_gpu (the reference's lanedet CLI over the C-ABI): file formats on
CPU (synth needs no GPU), and detect's artifacts against the compiled
reference on the GPU."""
import json
import subprocess
import zlib
from pathlib import Path

import numpy as np
import pytest

from paper_1807_02752_b200 import abi, lanekit

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_1807_02752_b200" / "lanedet_gpu"


def read_png(path):
    """Minimal decoder for the CLI's PNGs (8-bit grey or RGB, filter 0)."""
    d = Path(path).read_bytes()
    assert d[:8] == b"\x89PNG\r\n\x1a\n"
    o, idat, w = 8, b"", 0
    while o < len(d):
        n = int.from_bytes(d[o:o + 4], "big")
        t = d[o + 4:o + 8]
        body = d[o + 8:o + 8 + n]
        assert zlib.crc32(d[o + 4:o + 8 + n]) == int.from_bytes(d[o + 8 + n:o + 12 + n], "big")
        if t == b"IHDR":
            w, h, ch = int.from_bytes(body[:4], "big"), int.from_bytes(body[4:8], "big"), body[9]
        elif t == b"IDAT":
            idat += body
        o += 12 + n
    c = 3 if ch == 2 else 1
    raw = np.frombuffer(zlib.decompress(idat), np.uint8).reshape(h, w * c + 1)
    assert not raw[:, 0].any()
    return raw[:, 1:].reshape(h, w, c).squeeze()


def read_pgm(path):
    d = Path(path).read_bytes()
    parts = d.split(b"\n", 3)
    assert parts[0] == b"P5"
    w, h = map(int, parts[1].split())
    maxval = int(parts[2])
    dt = ">u2" if maxval > 255 else "u1"
    return np.frombuffer(parts[3], dt).reshape(h, w), maxval


def test_cli_synth_formats(tmp_path):
    out = subprocess.run([str(CLI), "synth", "--out-dir", str(tmp_path), "--seed", "3",
                          "--width", "320", "--height", "240"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    left = read_png(tmp_path / "left.png")
    right = read_png(tmp_path / "right.png")
    disp, maxval = read_pgm(tmp_path / "true_disparity.pgm")
    assert left.shape == (240, 320) and right.shape == (240, 320) and maxval == 65535
    import ctypes as C

    q = abi.LkSceneParams()
    lanekit.library().lk_scene_default(C.byref(q))
    q.width, q.height, q.rng_seed, q.noise_sigma = 320, 240, 3, 0.02
    l2, r2, d2, _ = lanekit.synth_scene(q)
    assert np.array_equal(left, l2) and np.array_equal(right, r2)
    assert np.array_equal(disp, d2.astype(np.uint16) * 256)


def test_cli_rejects_bad_input(tmp_path):
    (tmp_path / "a.pgm").write_bytes(b"P5\n4 4\n65535\n" + bytes(32))
    out = subprocess.run([str(CLI), "detect", "--left", str(tmp_path / "a.pgm"), "--right",
                          str(tmp_path / "a.pgm"), "--out-dir", str(tmp_path / "o")],
                         capture_output=True, text=True)
    assert out.returncode == 1 and "maxval 255" in out.stderr
    out = subprocess.run([str(CLI), "detect", "--left", "x", "--right", "y", "--out-dir",
                          str(tmp_path), "--set", "nope=1"], capture_output=True, text=True)
    assert out.returncode == 1 and "config: unknown key 'nope'" in out.stderr


@pytest.mark.gpu
def test_cli_detect_artifacts_match_reference(tmp_path, oracle):
    from checkers import Checker, ref_available

    chk = Checker("ref") if ref_available() else oracle
    out = subprocess.run([str(CLI), "synth", "--out-dir", str(tmp_path), "--seed", "5",
                          "--width", "1242", "--height", "375"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    left, right = read_png(tmp_path / "left.png"), read_png(tmp_path / "right.png")
    od = tmp_path / "out"
    out = subprocess.run([str(CLI), "detect", "--left", str(tmp_path / "left.png"), "--right",
                          str(tmp_path / "right.png"), "--out-dir", str(od), "--emit-all"],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    cfg = abi.default_config()
    st = chk.stereo(left, right, cfg)
    r = chk.run(left, st["DISPARITY"], cfg)
    rep = r.report
    disp, _ = read_pgm(od / "disparity.pgm")
    assert np.array_equal(disp, st["DISPARITY"].astype(np.uint16) * 256)
    dl, _ = read_pgm(od / "disparity_left.pgm")
    assert np.array_equal(dl, st["DISP_LEFT"].astype(np.uint16) * 256)
    j = json.loads((od / "report.json").read_text())
    assert j["lanes"]["count"] == rep.lane_count and j["road"]["horizon"] == rep.horizon
    assert j["edges"]["count"] == rep.edge_pixels
    assert j["stereo"]["valid_disparities"] == rep.valid_disparities
    assert j["road"]["beta"] == [rep.beta[0], rep.beta[1], rep.beta[2]]
    lanes = r.get("LANES")
    assert [d["bottom_col"] for d in j["lanes"]["detected"]] == list(lanes["bottom_col"])
    csv = (od / "lanes.csv").read_text().splitlines()
    assert csv[0] == "lane_id,v,u" and len(csv) > 1
    edges = read_png(od / "edges.png")
    e = r.get("EDGES")
    ref_edges = np.zeros_like(edges)
    ref_edges[e["v"], e["u"]] = 255
    assert np.array_equal(edges, ref_edges)
    vd, _ = read_pgm(od / "vdisparity.pgm")
    assert np.array_equal(vd, np.minimum(r.get("VDISPARITY"), 255).astype(np.uint8))
    for f in ("overlay.png", "vpx_accumulator.pgm", "road_fit.csv", "smoothed.png", "m1.png",
              "energy_histogram.csv", "upath.csv", "vpath.csv", "block_sigma.png"):
        assert (od / f).exists(), f


def test_cli_stream_rejects_bad_list(tmp_path):
    out = subprocess.run([str(CLI), "stream", "--list", str(tmp_path / "none.txt"), "--out",
                          str(tmp_path / "o.csv")], capture_output=True, text=True)
    assert out.returncode == 1 and "stream: cannot open" in out.stderr
    (tmp_path / "l.txt").write_text("# only a comment\n\n")
    out = subprocess.run([str(CLI), "stream", "--list", str(tmp_path / "l.txt"), "--out",
                          str(tmp_path / "o.csv")], capture_output=True, text=True)
    assert out.returncode == 1 and "no stereo pairs" in out.stderr


@pytest.mark.gpu
def test_cli_stream_matches_reference(tmp_path, oracle):
    """stream: pairs decoded on host threads into two pinned slots, batches of 2
    through lk_submit_stereo_batch; every ok line equals the reference's
    run_pipeline on that pair, bad pairs become stage-1 error lines in order."""
    import csv

    from checkers import Checker, ref_available

    chk = Checker("ref") if ref_available() else oracle
    pairs, scenes = [], {}
    for seed in (1, 2, 3):
        d = tmp_path / f"s{seed}"
        out = subprocess.run([str(CLI), "synth", "--out-dir", str(d), "--seed", str(seed),
                              "--width", "640", "--height", "360"], capture_output=True, text=True)
        assert out.returncode == 0, out.stderr
        scenes[seed] = d
    small = tmp_path / "small"
    subprocess.run([str(CLI), "synth", "--out-dir", str(small), "--seed", "9", "--width", "320",
                    "--height", "240"], check=True, capture_output=True)
    order = [1, 2, None, 3, "small", 1]
    for o in order:
        if o is None:
            pairs.append(f"{tmp_path / 'missing.png'} {tmp_path / 'missing.png'}")
        else:
            d = small if o == "small" else scenes[o]
            pairs.append(f"{d / 'left.png'} {d / 'right.png'}")
    (tmp_path / "pairs.txt").write_text("\n".join(pairs) + "\n")
    res = tmp_path / "lanes.csv"
    out = subprocess.run([str(CLI), "stream", "--list", str(tmp_path / "pairs.txt"), "--out",
                          str(res), "--batch", "2", "--threads", "3"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    rows = list(csv.DictReader(res.open()))
    assert [int(r["index"]) for r in rows] == list(range(len(order)))
    cfg = abi.default_config()
    for o, r in zip(order, rows):
        if o is None or o == "small":
            assert r["status"] == "error" and r["failed_stage"] == "1"
            assert ("png: cannot open" if o is None else "pair size differs") in r["message"]
            continue
        assert r["status"] == "ok", r
        left, right = read_png(scenes[o] / "left.png"), read_png(scenes[o] / "right.png")
        st = chk.stereo(left, right, cfg)
        ref = chk.run(left, st["DISPARITY"], cfg)
        rep = ref.report
        assert int(r["horizon"]) == rep.horizon and int(r["lane_count"]) == rep.lane_count
        cols = [int(x) for x in r["bottom_cols"].split(";")] if r["bottom_cols"] else []
        n = min(rep.lane_count, abi.LK_MAX_INLINE_LANES)
        assert cols == list(ref.get("LANES")["bottom_col"])[:n]


def test_cli_bench_rejects_bad_args():
    out = subprocess.run([str(CLI), "bench", "--reps", "0"], capture_output=True, text=True)
    assert out.returncode == 1 and "repetition" in out.stderr


@pytest.mark.gpu
def test_cli_bench_stage_table(ref):
    """lanedet bench (lanedet.cpp:111-127): the reference's synthetic 320x240
    scene, every stage of run_pipeline timed, and the same lanes as the
    reference's run_pipeline on that scene (stereo pair in)."""
    out = subprocess.run([str(CLI), "bench", "--reps", "3", "--batch", "16"], capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.splitlines()
    stages = [ln for ln in lines if ln[:4].strip().isdigit()]
    assert [int(ln.split()[0]) for ln in stages] == list(range(1, 13))
    assert "total" in out.stdout and "frames/s" in out.stdout
    # lanes of the GPU frame vs the reference's run_pipeline on the same pair
    p = abi.scene_params(width=320, height=240, lane_bottoms=(320 / 3, 640 / 3), d_max=64,
                         rng_seed=1)
    left, right, _, _ = ref.gen_scene(p)
    cfg = abi.default_config(d_max=min(64, round(-15 + 0.15 * 239 + 1e-4 * 239 ** 2) + 4))
    import ctypes as C

    rep = (abi.LkFrameReport * 1)()
    ref.lib.lkref_run_stereo_batch.argtypes = [
        C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(abi.LkConfig), C.c_int,
        C.POINTER(abi.LkFrameReport)]
    ref.lib.lkref_run_stereo_batch(left.ctypes.data, right.ctypes.data, 1, 320, 240,
                                   C.byref(cfg), 1, rep)
    want = rep[0].as_dict()["lane_bottom_col"]
    got = [int(x) for x in lines[-1].split("lanes of frame 0:")[1].split()]
    assert got == want
