"""TEST INFRASTRUCTURE: ctypes loaders for the CPU checkers under oracle/.

- `Checker("oracle")` — oracle/liblk_oracle.so, the restatement of stages 1-4
  (stereo) and 5-12;
- `Checker("ref")`    — oracle/_ref/liblk_ref.so, the unmodified reference
  headers compiled against the Eigen stand-in (built only where
  /root/reference exists; prebuilt copies travel to the GPU box).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_1807_02752_b200 import abi

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "liblk_oracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "liblk_ref.so"

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def ref_available() -> bool:
    return REF_SO.exists()


class Checker:
    def __init__(self, kind: str = "oracle"):
        path, prefix = (ORACLE_SO, "orc_") if kind == "oracle" else (REF_SO, "lkref_")
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.kind = kind
        self.lib = C.CDLL(str(path))
        self.p = prefix
        f = self._f
        f("report_size").restype = C.c_size_t
        if f("report_size")() != C.sizeof(abi.LkFrameReport):
            raise RuntimeError(f"{path}: lk_frame_report layout differs from abi.LkFrameReport "
                               f"(stale build: run `make -C oracle`)")
        f("run").restype = C.c_void_p
        f("run").argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.POINTER(abi.LkConfig)]
        f("free").argtypes = [C.c_void_p]
        f("report").argtypes = [C.c_void_p, C.POINTER(abi.LkFrameReport)]
        f("ext_cols").argtypes = [C.c_void_p]
        f("get").restype = C.c_size_t
        f("get").argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]
        f("run_batch").argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(abi.LkConfig), C.c_int,
                                   C.POINTER(abi.LkFrameReport)]
        f("stereo").argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                C.c_int, C.c_double, _f64p, _f64p, _u8p, _u8p, _u8p]
        if kind == "ref":
            self.lib.lkref_gen_scene.argtypes = [
                C.POINTER(abi.LkSceneParams), C.c_void_p, C.c_void_p, C.c_void_p,
                C.POINTER(C.c_int32), C.c_char_p, C.c_int]
        else:
            L = self.lib
            L.orc_dp_min_path.restype = C.c_double
            L.orc_dp_min_path.argtypes = [C.c_int, C.c_int, _f64p, _i32p, C.c_int, _f64p, _i32p]
            L.orc_fit_parabola.argtypes = [_i32p, C.c_int, _f64p]
            L.orc_fit_quartic.argtypes = [_i32p, C.c_int, C.c_double, C.c_double, _f64p,
                                          C.POINTER(C.c_double)]
            L.orc_ransac.argtypes = [C.c_int, _i32p, C.c_int, C.c_double, C.c_double, C.c_int,
                                     C.c_uint64, _f64p, C.POINTER(C.c_double),
                                     C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                     C.POINTER(C.c_int32), _i32p, C.POINTER(C.c_int32)]
            L.orc_piecewise_weight.restype = C.c_double
            L.orc_piecewise_weight.argtypes = [C.c_double] * 3
            L.orc_lane_track.argtypes = [C.c_double, _f64p, _f64p, C.c_int, C.c_int, _f64p]
            L.orc_auto_lane_threshold.restype = C.c_double
            L.orc_auto_lane_threshold.argtypes = [_f64p, C.c_int, C.c_int, C.c_int, C.c_int]

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def stereo(self, left: np.ndarray, right: np.ndarray, cfg: abi.LkConfig) -> dict:
        """Stages 1-4 (pipeline.hpp:161-182) on one u8 pair: the PipelineResult
        members stats_left (mu, sigma), disp_left, disp_right, disparity."""
        H, W = left.shape
        out = {"STATS_MU": np.zeros((H, W)), "STATS_SIGMA": np.zeros((H, W)),
               "DISP_LEFT": np.zeros((H, W), np.uint8), "DISP_RIGHT": np.zeros((H, W), np.uint8),
               "DISPARITY": np.zeros((H, W), np.uint8)}
        rc = self._f("stereo")(np.ascontiguousarray(left, np.uint8),
                               np.ascontiguousarray(right, np.uint8), W, H, cfg.rho, cfg.d_max,
                               cfg.tau, cfg.tr_lrc, cfg.sigma_floor, out["STATS_MU"],
                               out["STATS_SIGMA"], out["DISP_LEFT"], out["DISP_RIGHT"],
                               out["DISPARITY"])
        if rc:
            raise ValueError("stereo: image smaller than the matching block")
        return out

    def run(self, grey: np.ndarray, disp: np.ndarray, cfg: abi.LkConfig) -> "CheckerResult":
        H, W = grey.shape
        h = self._f("run")(np.ascontiguousarray(grey, np.uint8),
                           np.ascontiguousarray(disp, np.uint8), W, H, C.byref(cfg))
        return CheckerResult(self, h, W, H, cfg)

    def run_batch(self, grey, disp, cfg, threads=1):
        n, H, W = grey.shape
        reps = (abi.LkFrameReport * n)()
        self._f("run_batch")(np.ascontiguousarray(grey), np.ascontiguousarray(disp), n, W, H,
                             C.byref(cfg), threads, reps)
        return list(reps)

    def gen_scene(self, p: abi.LkSceneParams):
        """Reference gen_scene + 8-bit quantisation (ref only)."""
        W, H = p.width, p.height
        left = np.zeros((H, W), np.uint8)
        right = np.zeros((H, W), np.uint8)
        disp = np.zeros((H, W), np.uint8)
        hz = C.c_int32(0)
        msg = C.create_string_buffer(256)
        rc = self.lib.lkref_gen_scene(C.byref(p), left.ctypes.data, right.ctypes.data,
                                      disp.ctypes.data, C.byref(hz), msg, 256)
        if rc:
            raise ValueError(msg.value.decode())
        return left, right, disp, hz.value

    # ---- unit-level restatements (oracle only)
    def dp_min_path(self, data: np.ndarray, offsets, penalties):
        stages, states = data.shape
        path = np.zeros(stages, np.int32)
        e = self.lib.orc_dp_min_path(stages, states, np.ascontiguousarray(data, np.float64),
                                     np.asarray(offsets, np.int32), len(offsets),
                                     np.asarray(penalties, np.float64), path)
        return e, path

    def fit(self, kind: int, pts, kappa=1.0, vnorm=0.0):
        pts = np.ascontiguousarray(pts, np.int32).reshape(-1, 2)
        out = np.zeros(5, np.float64)
        if kind == 3:
            rc = self.lib.orc_fit_parabola(pts, len(pts), out)
            return None if rc else out[:3]
        s = C.c_double(0)
        rc = self.lib.orc_fit_quartic(pts, len(pts), kappa, vnorm, out, C.byref(s))
        return None if rc else (out, s.value)

    def ransac(self, kind, pts, tol, eps, seed, max_iter=200):
        pts = np.ascontiguousarray(pts, np.int32).reshape(-1, 2)
        model = np.zeros(5, np.float64)
        s, frac = C.c_double(0), C.c_double(0)
        iters, deg, ninl = C.c_int32(0), C.c_int32(0), C.c_int32(0)
        inl = np.zeros((max(len(pts), 1), 2), np.int32)
        msg = self.lib.orc_ransac(kind, pts, len(pts), tol, eps, max_iter, seed, model,
                                  C.byref(s), C.byref(iters), C.byref(frac), C.byref(deg),
                                  inl, C.byref(ninl))
        if msg:
            return {"msg": msg}
        return {"msg": 0, "model": model[:kind], "s": s.value, "iterations": iters.value,
                "fraction": frac.value, "degraded": bool(deg.value),
                "inliers": inl[:ninl.value].copy()}

    def piecewise_weight(self, te, tv, sg):
        return self.lib.orc_piecewise_weight(te, tv, sg)

    def lane_track(self, u, vpx, vpy, v_top, v_max):
        out = np.zeros(v_max - v_top + 1, np.float64)
        self.lib.orc_lane_track(u, np.ascontiguousarray(vpx, np.float64),
                                np.ascontiguousarray(vpy, np.float64), v_top, v_max, out)
        return out

    def auto_lane_threshold(self, m1, v_top, v_max):
        H, W = m1.shape
        return self.lib.orc_auto_lane_threshold(np.ascontiguousarray(m1, np.float64), W, H,
                                                v_top, v_max)

    def horizon_row(self, beta, rows):
        ir = C.c_int32(0)
        f = self.lib.orc_horizon_row
        f.argtypes = [_f64p, C.c_int, C.POINTER(C.c_int32)]
        r = f(np.asarray(beta, np.float64), rows, C.byref(ir))
        return r, bool(ir.value)

    def vpy_profile(self, beta, rows):
        val = np.zeros(rows, np.float64)
        sing = np.zeros(rows, np.uint8)
        f = self.lib.orc_vpy_profile
        f.argtypes = [_f64p, C.c_int, _f64p, np.ctypeslib.ndpointer(np.uint8)]
        f(np.asarray(beta, np.float64), rows, val, sing)
        return val, sing

    def extended_cols(self, xi, width):
        self.lib.orc_extended_col_lo.argtypes = [C.c_double, C.c_int]
        self.lib.orc_extended_col_count.argtypes = [C.c_double, C.c_int]
        return self.lib.orc_extended_col_lo(xi, width), self.lib.orc_extended_col_count(xi, width)

    def sparse_vpx(self, edges, vpy, singular, xi, width):
        """edges: [(u, v, gx, gy)] -> (vote columns (None = skipped), votes)."""
        uv = np.ascontiguousarray([[e[0], e[1]] for e in edges], np.int32)
        g = np.ascontiguousarray([[e[2], e[3]] for e in edges], np.float64)
        out = np.zeros(len(edges), np.int32)
        f = self.lib.orc_sparse_vpx
        f.argtypes = [_i32p, _f64p, C.c_int, _f64p, np.ctypeslib.ndpointer(np.uint8), C.c_int,
                      C.c_double, C.c_int, _i32p]
        n = f(uv, g, len(edges), np.asarray(vpy, np.float64),
              np.ascontiguousarray(singular, np.uint8), len(vpy), xi, width, out)
        cols = [None if c == np.iinfo(np.int32).min else int(c) for c in out]
        return cols, n

    def accumulate(self, votes, ext_lo, ext_cols, v_top, v_max, chi, rho_vote):
        cr = np.ascontiguousarray(votes, np.int32).reshape(-1, 2)
        acc = np.zeros((v_max - v_top + 1, ext_cols), np.float64)
        f = self.lib.orc_accumulate
        f.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                      _f64p]
        f(cr, len(cr), ext_lo, ext_cols, v_top, v_max, chi, rho_vote, acc)
        return acc

    def aggregate_energy(self, m1, vpx, vpy, v_top, v_max, xi, lambda_g):
        H, W = m1.shape
        lo, n = self.extended_cols(xi, W)
        out = np.zeros(n, np.float64)
        f = self.lib.orc_aggregate_energy
        f.argtypes = [_f64p, C.c_int, C.c_int, _f64p, _f64p, C.c_int, C.c_int, C.c_double,
                      C.c_double, _f64p]
        f(np.ascontiguousarray(m1, np.float64), W, H, np.asarray(vpx, np.float64),
          np.asarray(vpy, np.float64), v_top, v_max, xi, lambda_g, out)
        return lo, out

    def select_lanes(self, h, tr, min_sep):
        h = np.ascontiguousarray(h, np.float64)
        kept = np.zeros(len(h), np.int32)
        f = self.lib.orc_select_lanes
        f.argtypes = [_f64p, C.c_int, C.c_double, C.c_int, _i32p]
        k = f(h, len(h), tr, min_sep, kept)
        return kept[:k].tolist()


class CheckerResult:
    def __init__(self, chk: Checker, handle, W, H, cfg):
        self.chk, self.h, self.W, self.H, self.cfg = chk, handle, W, H, cfg
        self.report = abi.LkFrameReport()
        chk._f("report")(handle, C.byref(self.report))
        self.ext_cols = chk._f("ext_cols")(handle)

    def __del__(self):
        try:
            self.chk._f("free")(self.h)
        except Exception:
            pass

    def raw(self, stage: int) -> bytes:
        n = self.chk._f("get")(self.h, stage, None, 0)
        buf = C.create_string_buffer(max(n, 1))
        self.chk._f("get")(self.h, stage, buf, n)
        return buf.raw[:n]

    def get(self, name: str):
        st = abi.STAGE[name]
        return abi.decode_stage(st, self.raw(st), self.W, self.H, self.cfg.d_max,
                                self.ext_cols, int(self.report.horizon))
