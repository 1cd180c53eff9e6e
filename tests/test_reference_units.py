"""The reference's hot-path unit tests and acceptance criteria 5-10, re-expressed
against the CPU oracle (the restatement the GPU path is checked against).

Each test cites the reference test it follows (proj/tests/*.cpp:line)."""
import itertools
import math

import numpy as np
import pytest

from paper_1807_02752_b200 import abi

KPI = 3.14159265358979323846


# ------------------------------------------------------------------ [road]
def test_vdisparity_counts(oracle):
    """test_road.cpp:13-30 — d=0 and d>d_max never counted."""
    disp = np.zeros((4, 6), np.uint8)
    disp[1, 0] = 3
    disp[1, 1] = 3
    disp[1, 2] = 7
    disp[1, 3] = 99
    disp[2, 0] = 1
    grey = np.full((4, 6), 100, np.uint8)
    r = oracle.run(grey, disp, abi.default_config(d_max=8))
    h = r.get("VDISPARITY")
    assert h[1, 3] == 2 and h[1, 7] == 1 and h[2, 1] == 1
    assert (h[:, 0] == 0).all() and h.sum() == 4


def _enumerate(data, offsets, pen):
    """oracles.hpp:152-182 — exhaustive paths; state at stage+1 = state - offset."""
    stages, states = data.shape
    best, best_path = math.inf, None

    def rec(stage, state, e, path):
        nonlocal best, best_path
        e = e + data[stage, state]
        path = path + [state]
        if stage == stages - 1:
            if e < best:
                best, best_path = e, path
            return
        for o, p in zip(offsets, pen):
            ns = state - o
            if 0 <= ns < states:
                rec(stage + 1, ns, e + p, path)

    for s0 in range(states):
        rec(0, s0, 0.0, [])
    return best, best_path


def _count_optima(data, offsets, pen, best, tol=1e-9):
    stages, states = data.shape
    n = 0

    def rec(stage, state, e):
        nonlocal n
        e = e + data[stage, state]
        if stage == stages - 1:
            n += e <= best + tol
            return
        for o, p in zip(offsets, pen):
            ns = state - o
            if 0 <= ns < states:
                rec(stage + 1, ns, e + p)

    for s0 in range(states):
        rec(0, s0, 0.0)
    return n


def test_dp_engine_equals_enumeration(oracle):
    """test_dp.cpp:30-64 — energy bit-exact, path equal, on untied instances."""
    rng = np.random.default_rng(2026)
    done = 0
    while done < 40:
        stages, states = rng.integers(2, 7, size=2)
        data = rng.uniform(-10.0, 2.0, size=(stages, states))
        offsets = [0, 1, 2, 3] if done % 2 == 0 else [0, -1, 1, -2, 2]
        lam = rng.uniform(0, 3)
        pen = [(-lam * o if done % 3 == 0 else lam * abs(o)) for o in offsets]
        e, path = oracle.dp_min_path(data, offsets, pen)
        re, rpath = _enumerate(data, offsets, pen)
        if _count_optima(data, offsets, pen, re) != 1:
            continue
        assert e == pytest.approx(re, abs=1e-9)
        assert path.tolist() == rpath
        done += 1


def test_dp_tie_break_and_bounds(oracle):
    """test_dp.cpp:66-88 — earlier offsets win ties; smallest terminal; one state."""
    e, path = oracle.dp_min_path(np.zeros((5, 4)), [0, -1, 1], [0.0, 0.0, 0.0])
    assert e == 0.0 and (path == 0).all()
    data = np.array([[0.0], [1.0], [2.0], [3.0]])
    e, path = oracle.dp_min_path(data, [0, -1, 1], [0.0, 100.0, 100.0])
    assert e == 6.0 and (path == 0).all()


def test_criterion5_vpath_enumeration(oracle):
    """acceptance.cpp:200-245 — integer counts, dyadic lambda 1.75, 7 offsets."""
    rng = np.random.default_rng(505)
    done = 0
    while done < 30:
        d_max = int(rng.integers(4, 8))
        rows = int(rng.integers(5, 9))
        counts = rng.integers(0, 6, size=(rows, d_max + 1))
        data = np.array([[-float(counts[v, d_max - st]) for v in range(rows)]
                         for st in range(d_max + 1)])
        offsets = list(range(7))
        pen = [1.75 * o for o in offsets]
        re, rpath = _enumerate(data, offsets, pen)
        if _count_optima(data, offsets, pen, re) != 1:
            continue
        e, path = oracle.dp_min_path(data, offsets, pen)
        assert e == re and path.tolist() == rpath
        done += 1


def test_parabola_lsq_exact_data(oracle):
    """test_road.cpp:100-127 — vs a long-double normal-equation solve, margin 1e-7."""
    beta = (10.0, 0.2, 0.001)
    pts = [(int(round(beta[0] + beta[1] * v + beta[2] * v * v)), v) for v in range(40, 231, 10)]
    fit = oracle.fit(3, pts)
    A = np.zeros((3, 3), np.longdouble)
    b = np.zeros(3, np.longdouble)
    for d, v in pts:
        phi = np.array([1, v, v * v], np.longdouble)
        A += np.outer(phi, phi)
        b += d * phi
    ref = np.linalg.solve(A.astype(np.float64), b.astype(np.float64))
    assert np.allclose(fit, ref, rtol=0, atol=1e-7)
    assert oracle.fit(3, [(1, 5), (2, 5), (3, 5)]) is None  # needs three distinct rows


def test_ransac_beta_outliers(oracle):
    """test_road.cpp:129-158 (data regenerated with numpy): 20% gross outliers."""
    beta = (-40.0, 0.4, 0.0005)
    rng = np.random.default_rng(99)
    pts = [(int(round(beta[0] + beta[1] * v + beta[2] * v * v + rng.uniform(-0.5, 0.5))), v)
           for v in range(110, 350, 2)]
    clean = len(pts)
    pts += [(int(rng.integers(0, 201)), 110 + int(rng.integers(0, 240))) for _ in range(clean // 4)]
    r = oracle.ransac(3, pts, 4.0, 0.7, 7)
    assert r["msg"] == 0 and not r["degraded"] and r["fraction"] > 0.7
    for k in range(3):
        assert abs(r["model"][k] - beta[k]) <= 0.05 * abs(beta[k]) + 1e-3
    assert oracle.ransac(3, [(1, 1), (2, 2)], 4.0, 0.7, 7)["msg"] == 3  # too few points


def test_vpy_closed_forms(oracle):
    """test_road.cpp:160-178."""
    val, sing = oracle.vpy_profile((-75.0, 0.5, 0.0), 200)
    assert not sing.any() and np.allclose(val, 150.0, atol=1e-12)
    val, _ = oracle.vpy_profile((10.0, 0.1, 0.002), 400)
    assert val[300] == pytest.approx(300.0 - 220.0 / 1.3, abs=1e-9)
    val, sing = oracle.vpy_profile((5.0, 0.0, 0.0), 10)
    assert sing.all() and (val == np.arange(10)).all()


def test_horizon_cases(oracle):
    """test_road.cpp:180-204."""
    assert oracle.horizon_row((-50.0, 0.5, 0.0), 300) == (100, True)
    assert oracle.horizon_row((0.0, 1.0, 0.0), 300) == (0, True)
    assert oracle.horizon_row((10.0, 1.0, 0.0), 300) == (0, False)
    assert oracle.horizon_row((-40.0, 0.4, 0.0005), 360) == (90, True)
    assert not oracle.horizon_row((5.0, 0.0, 0.0), 100)[1]
    assert not oracle.horizon_row((-1.0, -1.0, 0.0), 100)[1]
    assert oracle.horizon_row((-500.0, 1.0, 0.0), 100) == (0, False)


# ------------------------------------------------------------------ [vanish]
def test_extended_axis(oracle):
    """test_vanish.cpp:12-19."""
    assert oracle.extended_cols(0.5, 1242) == (-621, 2484)
    assert oracle.extended_cols(0.3, 1242) == (-373, 1987)
    assert oracle.extended_cols(0.0, 640) == (0, 640)


def test_sparse_votes_follow_tangent(oracle):
    """test_vanish.cpp:21-56."""
    vpy, sing = oracle.vpy_profile((-75.0, 0.5, 0.0), 400)  # constant 150
    edges = [(100, 250, 0.5, 0.0), (100, 250, 0.5, 0.5), (100, 250, -0.4, 0.2),
             (100, 250, 1e-4, 0.9), (100, 399, 2.0, 2.0), (10, 250, 0.1, -4.0)]
    cols, n = oracle.sparse_vpx(edges, vpy, sing, 0.5, 400)
    assert n == 5 and cols[3] is None
    assert cols == [100, 200, 100 + int(round(100 * (0.2 / -0.4))), None, 100 + 249, -200]
    vpy = np.full(10, 5.0)
    sing = np.zeros(10, np.uint8)
    sing[4] = 1
    cols, n = oracle.sparse_vpx([(3, 4, 1.0, 0.0), (3, 12, 1.0, 0.0), (3, 3, 1.0, 0.0)], vpy, sing,
                                0.0, 8)
    assert n == 1 and cols == [None, None, 3]


def _band(v, v_top, v_max, chi):  # oracles.hpp:113-117
    if v > v_max - chi - 1:
        return v, v_max
    if v >= v_top + chi:
        return v - chi, v + chi
    return v_top, v + chi


def test_accumulator_equals_band_sums(oracle):
    """test_vanish.cpp:75-103 and criterion 8 (acceptance.cpp:420-455)."""
    rng = np.random.default_rng(808)
    for trial in range(30):
        ext_lo = -int(rng.integers(0, 11))
        ext_cols = 8 + int(rng.integers(0, 23))
        v_top = int(rng.integers(0, 21))
        v_max = v_top + 4 + int(rng.integers(0, 36))
        chi = int(rng.integers(0, 16))
        rho = 0.5 * (1 + int(rng.integers(0, 4)))
        n = 50 + int(rng.integers(0, 350))
        votes = [(ext_lo + int(rng.integers(0, ext_cols)),
                  v_top + int(rng.integers(0, v_max - v_top + 1))) for _ in range(n)]
        acc = oracle.accumulate(votes, ext_lo, ext_cols, v_top, v_max, chi, rho)
        for v in range(v_top, v_max + 1):
            top, bot = _band(v, v_top, v_max, chi)
            for c in range(ext_cols):
                cnt = sum(1 for (col, row) in votes if col == ext_lo + c and top <= row <= bot)
                assert acc[v - v_top, c] == -rho * cnt


def test_quartic_exact_and_kappa_invariance(oracle):
    """test_vanish.cpp:154-192, criterion 7 (acceptance.cpp:380-416)."""
    pts = [(int(300.0 - v + 0.00390625 * v * v), v) for v in range(80, 561, 80)]
    (g, s) = oracle.fit(5, pts)
    assert s == 560.0
    assert g[0] == pytest.approx(300.0, abs=1e-6) and g[1] == pytest.approx(-1.0, abs=1e-7)
    assert g[2] == pytest.approx(0.00390625, abs=1e-9)
    assert abs(g[3]) < 1e-9 and abs(g[4]) < 1e-11
    assert oracle.fit(5, [(1, 1), (2, 2), (3, 3), (4, 4)]) is None
    rng = np.random.default_rng(707)
    gam = (320.0, -0.4, 3e-4, -2e-8, 3e-12)
    pts = [(int(round(sum(gam[k] * v ** k for k in range(5)) + rng.uniform(-0.3, 0.3))), v)
           for v in range(64, 4097, 64)]
    qa, _ = oracle.fit(5, pts, kappa=1e-6)
    qb, sb = oracle.fit(5, pts, kappa=1.0)
    qc, _ = oracle.fit(5, pts, kappa=1e6)
    scale = np.maximum(1.0, np.abs(qb))
    assert np.all(np.abs(qa - qb) <= 1e-9 * scale) and np.all(np.abs(qc - qb) <= 1e-9 * scale)
    assert sb == 4096.0


def test_ransac_gamma_outliers(oracle):
    """test_vanish.cpp:213-241 (numpy data): worst deviation <= 3 columns."""
    rng = np.random.default_rng(626)
    gam = (280.0, -0.6, 0.0015)
    pts = [(int(round(gam[0] + gam[1] * v + gam[2] * v * v + rng.uniform(-0.5, 0.5))), v)
           for v in range(100, 356)]
    clean = len(pts)
    pts += [(int(rng.integers(-300, 901)), 100 + int(rng.integers(0, 256))) for _ in range(clean // 4)]
    r = oracle.ransac(5, pts, 16.0, 0.7, 3)
    assert r["msg"] == 0 and not r["degraded"]
    v = np.arange(100, 356, dtype=np.float64)
    m = r["model"]
    fit = m[0] + v * (m[1] + v * (m[2] + v * (m[3] + v * m[4])))
    assert np.max(np.abs(fit - (gam[0] + gam[1] * v + gam[2] * v * v))) <= 3.0


# ------------------------------------------------------------------ [lanes]
def test_orientation_weight(oracle):
    """test_lanes.cpp:23-35 and criterion 9 (acceptance.cpp:459-473)."""
    w = oracle.piecewise_weight
    assert w(0.3, 0.3, 3.5) == 1.0
    assert w(KPI / 6, 0.0, 3.5) == pytest.approx(math.exp(-6.0 / 12.25), abs=1e-12)
    for d in (KPI / 6 + 1e-6, KPI / 6 + 0.01, KPI / 4, KPI / 3, KPI / 2, 2.0):
        assert w(d, 0.0, 3.5) == 0.0
    assert w(KPI, 0.0, 3.5) == 1.0
    assert w(0.2, 0.2 + KPI, 3.5) == pytest.approx(1.0, abs=1e-12)
    assert w(0.4, 0.1, 3.5) == w(0.1, 0.4, 3.5)


def test_lane_tracks(oracle):
    """test_lanes.cpp:135-173 and criterion 10 (acceptance.cpp:478-523)."""
    vpx = np.full(240, 317.0)
    vpy = np.full(240, 88.5)
    rng = np.random.default_rng(11)
    for u0 in rng.uniform(-50, 700, 10):
        t = oracle.lane_track(u0, vpx, vpy, 100, 239)
        assert t[-1] == u0 and not np.isnan(t).any()
        v = 100.0 + np.arange(140)
        cross = (t - 317.0) * (239.0 - 88.5) - (u0 - 317.0) * (v - 88.5)
        assert np.all(np.abs(cross) <= 1e-6 * max(1.0, abs(u0 - 317.0)))
    t = oracle.lane_track(400.0, np.full(301, 400.0), np.full(301, 150.0), 160, 300)
    assert (t == 400.0).all()  # exact fixed point
    t = oracle.lane_track(30.0, np.full(21, 50.0), np.full(21, 15.2), 10, 20)
    assert not np.isnan(t[5:]).any() and np.isnan(t[:5]).all()  # truncation at v <= 14


def test_energy_aggregation(oracle):
    """test_lanes.cpp:175-209."""
    vpx = np.full(10, 8.0)
    vpy = np.full(10, -1e9)
    lo, h = oracle.aggregate_energy(np.full((10, 16), -1.0), vpx, vpy, 2, 9, 0.5, 1.0)
    assert lo == -8 and len(h) == 32
    cols = lo + np.arange(32)
    assert np.allclose(h, np.where((cols >= 0) & (cols < 16), -8.0, 0.0), atol=1e-12)
    m1 = np.zeros((10, 16))
    m1[3, :] = -1.0
    lo, h = oracle.aggregate_energy(m1, vpx, vpy, 2, 9, 0.0, 0.5)
    assert np.allclose(h, -0.5, atol=1e-12)


def test_lane_selection(oracle):
    """test_lanes.cpp:211-249."""
    h = [0, -5, 0, -3, 0, -10, 0]
    assert oracle.select_lanes(h, -1.0, 3) == [5, 1]
    assert oracle.select_lanes(h, -1.0, 2) == [5, 1, 3]
    assert oracle.select_lanes(h, -6.0, 2) == [5]
    assert oracle.select_lanes([-100, -5, -5, -100], -1.0, 2) == []


def test_auto_threshold(oracle):
    """test_lanes.cpp:251-260 — p99 ignores a single spike."""
    m1 = np.zeros((10, 10))
    for v in range(2, 10):
        m1[v, :] = 2.0 if v % 2 else -2.0
    m1[5, 5] = 100.0
    assert oracle.auto_lane_threshold(m1, 2, 9) == pytest.approx(-0.15 * 8 * 2.0, abs=1e-12)


def test_criterion6_robust_fits(oracle):
    """acceptance.cpp:299-376 — 20 trials of each robust fit under 20% outliers."""
    rng = np.random.default_rng(606)
    ok_b = ok_g = 0
    for trial in range(20):
        beta = (-60 + 40 * rng.uniform(-0.5, 0.5), 0.375 + 0.25 * rng.uniform(-0.5, 0.5),
                5e-4 + 6e-4 * rng.uniform(-0.5, 0.5))
        h_true, _ = oracle.horizon_row(beta, 1024)
        v0 = max(100, h_true + 5)
        pts = [(int(round(beta[0] + beta[1] * v + beta[2] * v * v + rng.uniform(-0.5, 0.5))), v)
               for v in range(v0, 801)]
        pts += [(int(rng.integers(0, 400)), v0 + int(rng.integers(0, 801 - v0)))
                for _ in range(len(pts) // 4)]
        r = oracle.ransac(3, pts, 4.0, 0.5, 1 + trial)
        ok_b += r["msg"] == 0 and all(abs(r["model"][k] - beta[k]) <= 0.02 * abs(beta[k])
                                      for k in range(3))
        gam = (320 + 240 * rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5),
               3e-3 * rng.uniform(-0.5, 0.5))
        gp = [(int(round(gam[0] + v * (gam[1] + v * gam[2]) + rng.uniform(-0.5, 0.5))), v)
              for v in range(100, 801)]
        gp += [(-1000 + int(rng.integers(0, 3500)), 100 + int(rng.integers(0, 701)))
               for _ in range(len(gp) // 4)]
        g = oracle.ransac(5, gp, 16.0, 0.5, 1000 + trial)
        v = np.arange(100, 801, dtype=np.float64)
        m = g["model"]
        fit = m[0] + v * (m[1] + v * (m[2] + v * (m[3] + v * m[4])))
        ok_g += np.max(np.abs(fit - (gam[0] + v * (gam[1] + v * gam[2])))) <= 3.0
    assert ok_b >= 18 and ok_g >= 18


def test_road_mask_selection(oracle):
    """test_preprocess.cpp:132-151 via the pipeline's MASK hook."""
    W, H = 200, 300
    disp = np.zeros((H, W), np.uint8)
    # a clean linear road so the fitted profile is exactly d = -50 + 0.5 v
    for v in range(100, H):
        disp[v, 4:] = int(round(-50 + 0.5 * v))
    disp[200, 0] = 50
    disp[200, 1] = 53
    disp[200, 2] = 54
    disp[99, 1] = 1
    grey = np.full((H, W), 90, np.uint8)
    r = oracle.run(grey, disp, abi.default_config(d_max=110))
    mask = r.get("MASK")
    assert r.report.horizon == 100
    assert mask[200, 0] == 1 and mask[200, 1] == 1 and mask[200, 2] == 0 and mask[200, 3] == 0
    assert mask[99].sum() == 0
