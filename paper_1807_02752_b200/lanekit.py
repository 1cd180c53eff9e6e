"""Python host API over the C-ABI (include/lanekit_b200.h).

Mirrors the reference's pipeline interface for the stage 5-12 path:
  - ``PipelineConfig`` / ``default_config``  <- lanekit::PipelineConfig (config.hpp:16-46)
  - ``run_pipeline_from_disparity``          <- lanekit::run_pipeline stages 5-12
                                                (pipeline.hpp:184-270), disparity injected
  - ``StageError``                           <- lanekit::StageError (common.hpp:18-24)
  - ``PipelineResult.stage(name)``           <- PipelineResult members (pipeline.hpp:69-99)
  - ``synth_scene``                          <- lanekit::gen_scene (synth.hpp:103-200)
Everything executes in liblanekit_b200.so (sm_100a kernels); there is no CPU
fallback: without the built library or a Blackwell GPU these calls raise.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import abi
from .abi import LkConfig as PipelineConfig  # noqa: F401  (reference-style name)
from .abi import default_config, scene_params  # noqa: F401
from .build import LIB

_lib = None


def library() -> C.CDLL:
    """Loads liblanekit_b200.so (built by __graft_entry__.build / build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    import os

    path = os.environ.get("LK_LIBRARY", str(LIB))  # A/B builds of the same sources
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is not built; run `python -m paper_1807_02752_b200.build`")
    L = C.CDLL(path)
    P, I, U32, SZ = C.c_void_p, C.c_int, C.c_uint32, C.c_size_t
    cfgp = C.POINTER(abi.LkConfig)
    repp = C.POINTER(abi.LkFrameReport)
    L.lk_create.argtypes = [C.POINTER(P), I, cfgp, I, I, I, U32]
    L.lk_destroy.argtypes = [P]
    L.lk_run_batch.argtypes = [P, P, P, I, I, repp]
    L.lk_get_stage.argtypes = [P, I, I, P, SZ, C.POINTER(SZ)]
    L.lk_stage_times.argtypes = [P, C.POINTER(C.c_float)]
    L.lk_last_error.restype = C.c_char_p
    L.lk_validate_config.argtypes = [cfgp]
    L.lk_launches_per_batch.argtypes = [P]
    L.lk_timed_frames.argtypes = [P]
    L.lk_device_inputs.argtypes = [P, C.POINTER(P), C.POINTER(P)]
    L.lk_enqueue.argtypes = [P, I]
    L.lk_submit_batch.argtypes = [P, P, P, I, repp]
    L.lk_submit_resident.argtypes = [P, I, repp]
    L.lk_submit_stereo_batch.argtypes = [P, P, P, I, repp]
    L.lk_wait_batch.argtypes = [P]
    L.lk_fetch_reports.argtypes = [P, repp, I]
    L.lk_synchronize.argtypes = [P]
    L.lk_stream.argtypes = [P]
    L.lk_stream.restype = P
    L.lk_h2d_bytes.argtypes = [P, C.POINTER(C.c_ulonglong)]
    L.lk_host_alloc.argtypes = [C.POINTER(P), SZ]
    L.lk_host_free.argtypes = [P]
    L.lk_abi_sizes.argtypes = [C.POINTER(SZ)]
    L.lk_fast_path_error.argtypes = [P, C.POINTER(C.c_double)]
    L.lk_synth_scene.argtypes = [C.POINTER(abi.LkSceneParams), P, P, P, C.POINTER(C.c_int32)]
    L.lk_synth_batch.argtypes = [C.POINTER(abi.LkSceneParams), I, P, P, I]
    L.lk_synth_stereo_batch.argtypes = [C.POINTER(abi.LkSceneParams), I, P, P, P, I]
    L.lk_run_stereo_batch.argtypes = [P, P, P, I, I, repp]
    L.lk_stereo_inputs.argtypes = [P, C.POINTER(P), C.POINTER(P)]
    L.lk_enqueue_stereo.argtypes = [P, I]
    L.lk_synth_last_error.restype = C.c_char_p
    L.lk_stage_name.restype = C.c_char_p
    _lib = L
    return L


class LanekitError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class StageError(LanekitError):
    """A frame failed a pipeline stage: 'stage N (name): msg' (common.hpp:18-24)."""

    def __init__(self, stage: int, stage_name: str, msg: str):
        super().__init__(abi.LK_ERR_FRAME, msg)
        self.stage = stage
        self.stage_name = stage_name


def _check(status: int):
    if status != abi.LK_OK:
        raise LanekitError(status, library().lk_last_error().decode())


def validate_config(cfg: abi.LkConfig):
    """validate_config (config.hpp:124-152); raises LanekitError."""
    _check(library().lk_validate_config(C.byref(cfg)))


def stage_error(rep: abi.LkFrameReport) -> StageError:
    st = int(rep.failed_stage)
    return StageError(st, abi.STAGE_NAMES[st - 1], abi.frame_message(rep))


class GpuPipeline:
    """A context: device buffers, stream, CUDA graphs for (width, height, max_batch)."""

    def __init__(self, width: int, height: int, config: abi.LkConfig | None = None,
                 max_batch: int = 1, device: int = 0, hooks: bool = False,
                 graph: bool = True, exact: bool = False, stereo: bool = False):
        L = library()
        self.cfg = config if config is not None else default_config()
        self.width, self.height, self.max_batch = width, height, max_batch
        flags = (abi.LK_FLAG_HOOKS if hooks else 0) | (0 if graph else abi.LK_FLAG_NO_GRAPH) | \
            (abi.LK_FLAG_EXACT if exact else 0) | (abi.LK_FLAG_STEREO if stereo else 0)
        h = C.c_void_p()
        _check(L.lk_create(C.byref(h), device, C.byref(self.cfg), width, height, max_batch,
                           flags))
        self._h = h
        self.ext_lo = -int(np.round(self.cfg.xi * width)) if False else None
        self.reports: list[abi.LkFrameReport] = []

    def close(self):
        if getattr(self, "_h", None):
            library().lk_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def launches_per_batch(self) -> int:
        return library().lk_launches_per_batch(self._h)

    def run(self, grey: np.ndarray, disparity: np.ndarray) -> list[abi.LkFrameReport]:
        """Stages 5-12 on a batch: grey/disparity uint8 [n, H, W] (or [H, W])."""
        grey = np.ascontiguousarray(grey, np.uint8)
        disparity = np.ascontiguousarray(disparity, np.uint8)
        if grey.ndim == 2:
            grey, disparity = grey[None], disparity[None]
        if grey.shape != disparity.shape or grey.shape[1:] != (self.height, self.width):
            raise LanekitError(abi.LK_ERR_INVALID_ARGUMENT,
                               "stage 1 (block statistics): stereo pair dimensions differ")
        n = grey.shape[0]
        reps = (abi.LkFrameReport * n)()
        st = library().lk_run_batch(self._h, grey.ctypes.data, disparity.ctypes.data, n,
                                    abi.LK_MEM_HOST, reps)
        if st not in (abi.LK_OK, abi.LK_ERR_FRAME):
            _check(st)
        self.reports = list(reps)
        return self.reports

    def run_stereo(self, left: np.ndarray, right: np.ndarray) -> list[abi.LkFrameReport]:
        """Stages 1-12 (run_pipeline, pipeline.hpp:118-270) on u8 stereo pairs [n, H, W]."""
        left = np.ascontiguousarray(left, np.uint8)
        right = np.ascontiguousarray(right, np.uint8)
        if left.ndim == 2:
            left, right = left[None], right[None]
        if left.shape != right.shape or left.shape[1:] != (self.height, self.width):
            raise LanekitError(abi.LK_ERR_INVALID_ARGUMENT,
                               "stage 1 (block statistics): stereo pair dimensions differ")
        n = left.shape[0]
        reps = (abi.LkFrameReport * n)()
        st = library().lk_run_stereo_batch(self._h, left.ctypes.data, right.ctypes.data, n,
                                           abi.LK_MEM_HOST, reps)
        if st not in (abi.LK_OK, abi.LK_ERR_FRAME):
            _check(st)
        self.reports = list(reps)
        return self.reports

    def raw(self, frame: int, stage: int) -> bytes:
        L = library()
        need = C.c_size_t(0)
        _check(L.lk_get_stage(self._h, frame, stage, None, 0, C.byref(need)))
        buf = C.create_string_buffer(max(need.value, 1))
        _check(L.lk_get_stage(self._h, frame, stage, buf, need.value, C.byref(need)))
        return buf.raw[: need.value]

    def stage(self, frame: int, name: str) -> np.ndarray:
        st = abi.STAGE[name]
        rep = self.reports[frame]
        ext_cols = int(np.round((2 * self.cfg.xi + 1) * self.width))
        return abi.decode_stage(st, self.raw(frame, st), self.width, self.height,
                                self.cfg.d_max, ext_cols, int(rep.horizon))

    def fast_path_error(self) -> float:
        """max |approximate - exact| smoothed value of the last batch (fast path)."""
        e = C.c_double(0)
        _check(library().lk_fast_path_error(self._h, C.byref(e)))
        return e.value

    @property
    def timed_frames(self) -> int:
        """Frames of the last batch that stage_times() covers (branch 0)."""
        return library().lk_timed_frames(self._h)

    def stage_times(self) -> dict[int, float]:
        ms = (C.c_float * 13)()
        _check(library().lk_stage_times(self._h, ms))
        return {i: float(ms[i]) for i in [0, 5, 6, 7, 8, 9, 10, 11, 12]}


class PipelineResult:
    """Result of one frame: the report plus lazily fetched per-stage hooks."""

    def __init__(self, pipe: GpuPipeline, frame: int):
        self._pipe, self._frame = pipe, frame
        self.report = pipe.reports[frame]

    def stage(self, name: str) -> np.ndarray:
        return self._pipe.stage(self._frame, name)

    @property
    def lanes(self):
        return self.stage("LANES")


def run_pipeline_from_disparity(grey: np.ndarray, disparity: np.ndarray,
                                config: abi.LkConfig | None = None, device: int = 0,
                                hooks: bool = True) -> PipelineResult:
    """One frame through stages 5-12; raises StageError like run_pipeline."""
    cfg = config if config is not None else default_config()
    validate_config(cfg)
    if grey.size == 0 or disparity.size == 0:
        raise StageError(1, abi.STAGE_NAMES[0], "stage 1 (block statistics): empty input image")
    if grey.shape != disparity.shape:
        raise StageError(1, abi.STAGE_NAMES[0],
                         "stage 1 (block statistics): stereo pair dimensions differ")
    H, W = grey.shape
    pipe = GpuPipeline(W, H, cfg, 1, device, hooks=hooks)
    rep = pipe.run(grey, disparity)[0]
    if rep.status:
        raise stage_error(rep)
    return PipelineResult(pipe, 0)


def run_pipeline(left: np.ndarray, right: np.ndarray, config: abi.LkConfig | None = None,
                 device: int = 0, hooks: bool = True) -> PipelineResult:
    """run_pipeline(left, right, cfg) (pipeline.hpp:118-270) on one u8 stereo pair;
    raises StageError like the reference."""
    cfg = config if config is not None else default_config()
    validate_config(cfg)
    if left.size == 0 or right.size == 0:
        raise StageError(1, abi.STAGE_NAMES[0], "stage 1 (block statistics): empty input image")
    if left.shape != right.shape:
        raise StageError(1, abi.STAGE_NAMES[0],
                         "stage 1 (block statistics): stereo pair dimensions differ")
    H, W = left.shape
    if W <= 2 * cfg.rho or H <= 2 * cfg.rho:
        raise StageError(1, abi.STAGE_NAMES[0],
                         "stage 1 (block statistics): image smaller than the matching block")
    pipe = GpuPipeline(W, H, cfg, 1, device, hooks=hooks, stereo=True)
    rep = pipe.run_stereo(left, right)[0]
    if rep.status:
        raise stage_error(rep)
    return PipelineResult(pipe, 0)


def synth_stereo_batch(params: Sequence[abi.LkSceneParams], threads: int = 8):
    """Stereo pairs for a list of scenes: (left, right, true disparity) u8 [n, H, W]."""
    L = library()
    n = len(params)
    H, W = params[0].height, params[0].width
    left = np.zeros((n, H, W), np.uint8)
    right = np.zeros_like(left)
    disp = np.zeros_like(left)
    arr = (abi.LkSceneParams * n)(*params)
    if L.lk_synth_stereo_batch(arr, n, left.ctypes.data, right.ctypes.data, disp.ctypes.data,
                               threads):
        raise ValueError(L.lk_synth_last_error().decode())
    return left, right, disp


def synth_scene(p: abi.LkSceneParams):
    """gen_scene + 8-bit quantisation: (left u8, right u8, disparity u8, horizon)."""
    L = library()
    left = np.zeros((p.height, p.width), np.uint8)
    right = np.zeros_like(left)
    disp = np.zeros_like(left)
    hz = C.c_int32(0)
    if L.lk_synth_scene(C.byref(p), left.ctypes.data, right.ctypes.data, disp.ctypes.data,
                        C.byref(hz)):
        raise ValueError(L.lk_synth_last_error().decode())
    return left, right, disp, hz.value


def synth_batch(params: Sequence[abi.LkSceneParams], threads: int = 8):
    """Frames for a list of scenes, generated in parallel: (grey, disparity) [n, H, W]."""
    L = library()
    n = len(params)
    H, W = params[0].height, params[0].width
    grey = np.zeros((n, H, W), np.uint8)
    disp = np.zeros((n, H, W), np.uint8)
    arr = (abi.LkSceneParams * n)(*params)
    if L.lk_synth_batch(arr, n, grey.ctypes.data, disp.ctypes.data, threads):
        raise ValueError(L.lk_synth_last_error().decode())
    return grey, disp
