#!/usr/bin/env python
"""Throughput benchmark of the stage 5-12 lane pipeline (BASELINE.json config 2).

One step = one pass of the whole hot path (v-disparity .. lane selection, one
CUDA graph) over a batch of synthetic KITTI-size frames resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--config kitti|hires]
  python bench.py --impl reference ...   # the reference CPU implementation, host cores

Under torchrun each rank drives its own GPU (LOCAL_RANK) with its own frame
shard; no inter-GPU traffic (frames are independent); the per-rank device
times are max-reduced over gloo. Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/sec @1242x375 batched (1/2/4/8 B200), % HBM roofline, vs CPU ref"
UNIT = "frames/s"
PAPER_FPS = 143.0  # PAPER.md:14 (GTX 970M + i7 split) — context only, different hardware


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=0, help="frames per step per GPU")
    ap.add_argument("--pool", type=int, default=0, help="distinct frames generated per GPU")
    ap.add_argument("--config", default="kitti", choices=["kitti", "hires"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stream", type=int, default=0, metavar="N",
                    help="BASELINE config 5: a stream of N KITTI-size frames sharded over the "
                         "ranks (each cycles a resident 256-frame pool over its shard); lane "
                         "records gathered on rank 0 inside the timed region")
    ap.add_argument("--stereo", action="store_true",
                    help="stereo pairs in: stages 1-12 (the reference's run_pipeline) instead "
                         "of the north-star path (stages 5-12 on a given disparity)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(cfg_name: str, batch: int):
    from paper_1807_02752_b200 import abi, scenes

    if cfg_name == "hires":
        B = batch or 64
        return (scenes.hires_scene, scenes.hires_config(), scenes.HIRES_W, scenes.HIRES_H, B,
                f"config 4: batch of {B} synthetic 2560x1024 frames (grey + dense disparity, "
                f"2-4 curved lanes, non-flat road), stages 5-12 in one CUDA graph")
    B = batch or 256
    return (scenes.batch_scene, abi.default_config(), scenes.KITTI_W, scenes.KITTI_H, B,
            f"config 2: batch of {B} synthetic KITTI-size 1242x375 frames (grey + dense "
            f"disparity, 2-4 curved lanes, non-flat road), stages 5-12 in one CUDA graph")


def make_frames(scene_fn, n_pool: int, batch: int, seed0: int, stereo: bool = False):
    """(grey, disparity) [batch, H, W], or (left, right) for stereo runs."""
    from paper_1807_02752_b200 import lanekit

    params = [scene_fn(seed0 + i) for i in range(n_pool)]
    if stereo:
        grey, disp, _ = lanekit.synth_stereo_batch(params, threads=os.cpu_count() or 8)
    else:
        grey, disp = lanekit.synth_batch(params, threads=os.cpu_count() or 8)
    if n_pool < batch:
        reps = math.ceil(batch / n_pool)
        grey = np.concatenate([grey] * reps)[:batch]
        disp = np.concatenate([disp] * reps)[:batch]
    return np.ascontiguousarray(grey), np.ascontiguousarray(disp)


def ref_frames(chk, scene_fn, n: int, seed0: int):
    """(grey, disparity) [n, H, W] from the reference's gen_scene + 8-bit
    quantisation (oracle/ref_wrapper.cpp lkref_gen_scene)."""
    gs, ds = [], []
    for i in range(n):
        left, _, disp, _ = chk.gen_scene(scene_fn(seed0 + i))
        gs.append(left)
        ds.append(disp)
    return np.ascontiguousarray(np.stack(gs)), np.ascontiguousarray(np.stack(ds))


def drop_in_measurements(grey, disp, cfg, device: int, hooks_steps: int = 5, calls: int = 200):
    """The reference is called one frame at a time (pipeline.hpp:118): the
    drop-in's batch-1 latency with the context reused (frame in from pinned
    host memory, report out, lk_run_batch n = 1; host wall clock per call), and
    the hooks-mode throughput (LK_FLAG_HOOKS: the exact path with every
    PipelineResult member materialised, as the reference always does)."""
    import torch

    from paper_1807_02752_b200 import abi, lanekit

    B, H, W = grey.shape
    out = {}
    with lanekit.GpuPipeline(W, H, cfg, max_batch=1, device=device) as p:
        L, h = lanekit.library(), p._h
        hg, hd = C.c_void_p(), C.c_void_p()
        L.lk_host_alloc(C.byref(hg), H * W)
        L.lk_host_alloc(C.byref(hd), H * W)
        rep = abi.LkFrameReport()
        ts = []
        for i in range(calls + 10):
            C.memmove(hg, grey[i % B].ctypes.data, H * W)
            C.memmove(hd, disp[i % B].ctypes.data, H * W)
            t0 = time.perf_counter()
            L.lk_run_batch(h, hg, hd, 1, abi.LK_MEM_HOST, C.byref(rep))
            t1 = time.perf_counter()
            if i >= 10:
                ts.append((t1 - t0) * 1e3)
        L.lk_host_free(hg)
        L.lk_host_free(hd)
        ts.sort()
        out["batch1_latency_ms"] = {"median": ts[len(ts) // 2], "p99": ts[int(len(ts) * 0.99)],
                                    "min": ts[0], "calls": calls,
                                    "api": "lk_run_batch(n=1, LK_MEM_HOST) on a reused context: "
                                           "H2D, the 22-kernel graph, report D2H, host wall clock"}
    with lanekit.GpuPipeline(W, H, cfg, max_batch=B, device=device, hooks=True) as p:
        L, h = lanekit.library(), p._h
        reps = (abi.LkFrameReport * B)()
        L.lk_run_batch(h, grey.ctypes.data, disp.ctypes.data, B, abi.LK_MEM_HOST, reps)
        L.lk_enqueue(h, B)
        L.lk_synchronize(h)
        st = torch.cuda.ExternalStream(L.lk_stream(h), device=device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(hooks_steps):
            L.lk_enqueue(h, B)
        e1.record(st)
        e1.synchronize()
        out["hooks_mode"] = {"value": B * hooks_steps / (e0.elapsed_time(e1) * 1e-3),
                             "unit": UNIT, "steps": hooks_steps,
                             "note": "LK_FLAG_HOOKS: exact LUT bilateral on every pixel, MASK / "
                                     "GX / GY / MAG / THETA / VPX_ACC / M0 / polylines "
                                     "materialised; device-resident"}
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def _read(self):
        for ln in self.proc.stdout:
            if ln.strip():
                self.lines.append(ln)

    def __enter__(self):
        import threading

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            t0 = time.time()  # the first sample marks nvidia-smi as running
            while not self.lines and time.time() - t0 < 5:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.start = len(self.lines)  # samples taken inside the timed region only
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.06)  # one more sample interval covers the region's tail
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        self.lines = self.lines[self.start:]

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_baseline(grey, disp, cfg, frames: int, impl_kind: str | None = None,
                 stereo: bool = False):
    """Reference CPU pipeline on this host's cores, frame-parallel (one frame per
    worker thread, each frame single-threaded as cfg.threads=1 runs it)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from checkers import Checker, ref_available

    kind = impl_kind or ("reference" if ref_available() else "port")
    chk = Checker("ref" if kind == "reference" else "oracle")
    cores = os.cpu_count() or 1
    n = min(frames, grey.shape[0])
    t0 = time.perf_counter()
    if stereo and kind == "reference":  # run_pipeline on the pairs (stages 1-12)
        from paper_1807_02752_b200 import abi

        reps = (abi.LkFrameReport * n)()
        chk.lib.lkref_run_stereo_batch.argtypes = [
            C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(abi.LkConfig), C.c_int,
            C.POINTER(abi.LkFrameReport)]
        chk.lib.lkref_run_stereo_batch(np.ascontiguousarray(grey[:n]).ctypes.data,
                                       np.ascontiguousarray(disp[:n]).ctypes.data, n,
                                       grey.shape[2], grey.shape[1], C.byref(cfg), cores, reps)
    else:
        reps = chk.run_batch(np.ascontiguousarray(grey[:n]), np.ascontiguousarray(disp[:n]),
                             cfg, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{n} frames of the same workload, frame-parallel on {cores} host threads "
                      f"(each frame single-threaded), {dt:.1f} s wall",
            "failed_frames": sum(1 for r in reps if r.status)}, reps


def run_reference(args):
    """--impl reference: the reference's own CPU implementation (oracle/_ref =
    the unmodified lanekit headers compiled here), all host threads."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    scene_fn, cfg, W, H, B, desc = workload(args.config, args.batch)
    cores = os.cpu_count() or 1
    per_step = cores  # one frame per host thread per step: a bounded sample
    sys.path.insert(0, str(ROOT / "tests"))
    from checkers import Checker, ref_available

    kind = "reference" if ref_available() else "port"
    chk = Checker("ref" if kind == "reference" else "oracle")
    # the same frames as the GPU arm's first per_step (seeds 1..), rendered by the
    # reference's own gen_scene (synth.hpp:103) so this process never loads the
    # product library; the port falls back to the repo's restatement of it
    grey, disp = (ref_frames(chk, scene_fn, per_step, 1) if kind == "reference"
                  else make_frames(scene_fn, per_step, per_step, 1))
    for _ in range(max(0, min(args.warmup, 1))):
        chk.run_batch(grey, disp, cfg, threads=cores)
    steps = max(1, min(args.steps, 8))
    t0 = time.perf_counter()
    for _ in range(steps):
        chk.run_batch(grey, disp, cfg, threads=cores)
    dt = time.perf_counter() - t0
    fps = steps * per_step / dt
    # the reference called one frame at a time (pipeline.hpp:118): latency with
    # its own intra-frame threading off (threads = 1) and on (threads = nproc)
    lat = {}
    for th in (1, cores):
        c1 = abi_default_copy(cfg, threads=th)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            chk.run_batch(grey[:1], disp[:1], c1, threads=1)
            ts.append((time.perf_counter() - t0) * 1e3)
        lat[f"threads_{th}"] = sorted(ts)[1]
    line = {
        # n_gpus mirrors the launch (--gpus N); the reference arm runs on rank 0's host cores
        "impl": "reference", "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": max(world, args.gpus),
        "device": "host cpu (rank 0 only)",
        "steps": steps, "warmup": min(args.warmup, 1), "ms_per_step": dt / steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc.replace(f"batch of {B}", f"sample of {per_step}").replace(
                       "stages 5-12 in one CUDA graph",
                       "stages 5-12 by the reference's CPU code (lanekit headers)"),
                   "frames_per_step": per_step, "width": W, "height": H,
                   "parallelism": f"frame-parallel on {cores} host threads"},
        "cpu_baseline": {"value": fps, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{steps} steps x {per_step} frames (one per thread)"},
        "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "single_frame_latency_ms": {**lat, "note": "one frame, median of 3; cfg.threads = the "
                                                   "reference's intra-frame parallel_for (bilateral "
                                                   "rows, lane energies)"},
    }
    if kind != "reference":
        line["note"] = "oracle/_ref missing: timed the repo's restatement instead"
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    from paper_1807_02752_b200 import abi, lanekit

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
    local = local % max(1, torch.cuda.device_count())  # ranks may share a GPU (tests)
    torch.cuda.set_device(local)
    from paper_1807_02752_b200 import shard as _shard

    all_cpus = os.sched_getaffinity(0)
    _shard.bind_local_cpus(local)  # pinned host buffers below NUMA-local to the GPU
    scene_fn, cfg, W, H, B, desc = workload(args.config, args.batch)
    pool = args.pool or B
    stereo = args.stereo
    if stereo:
        desc = desc.replace("(grey + dense disparity", "(stereo pairs").replace(
            "stages 5-12", "stages 1-12")
    grey, disp = make_frames(scene_fn, pool, B, 1 + rank * pool, stereo)
    px = W * H

    pipe = lanekit.GpuPipeline(W, H, cfg, max_batch=B, device=local, stereo=stereo)
    L = lanekit.library()
    run_fn = L.lk_run_stereo_batch if stereo else L.lk_run_batch
    enq_fn = L.lk_enqueue_stereo if stereo else L.lk_enqueue
    h = pipe._h
    stream = torch.cuda.ExternalStream(L.lk_stream(h), device=local)
    dg, dd = C.c_void_p(), C.c_void_p()
    L.lk_device_inputs(h, C.byref(dg), C.byref(dd))
    # inputs resident in HBM before the timed region (pinned staging -> device)
    hg = C.c_void_p()
    hd = C.c_void_p()
    L.lk_host_alloc(C.byref(hg), B * px)
    L.lk_host_alloc(C.byref(hd), B * px)
    C.memmove(hg, grey.ctypes.data, B * px)
    C.memmove(hd, disp.ctypes.data, B * px)
    reps = (abi.LkFrameReport * B)()
    st = run_fn(h, hg, hd, B, abi.LK_MEM_HOST, reps)
    if st not in (abi.LK_OK, abi.LK_ERR_FRAME):
        raise RuntimeError(L.lk_last_error().decode())
    failed = sum(1 for r in reps if r.status)
    gpu_reps = [abi.LkFrameReport.from_buffer_copy(r) for r in reps]

    launches = pipe.launches_per_batch
    for _ in range(args.warmup):
        enq_fn(h, B)
    L.lk_synchronize(h)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()

    # ---- device-resident throughput: K graph replays, CUDA events on the lib stream
    ms13 = (C.c_float * 13)()
    stage_acc = np.zeros(13)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            enq_fn(h, B)
            L.lk_stage_times(h, ms13)  # waits for this step; per-kernel events of this replay
            stage_acc += np.frombuffer(ms13, np.float32)
        e1.record(stream)
        torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1)
    tf_dev = L.lk_timed_frames(h) or B  # frames of one range of the timed graph
    # ---- end to end through the public API: pinned host buffers in, reports out
    for _ in range(2):
        run_fn(h, hg, hd, B, abi.LK_MEM_HOST, reps)
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    # as many host-fed steps as device steps: the first step's copy cannot overlap
    # earlier kernels (the stream starts cold inside the timed region), so with
    # few steps that one-time fill dominates (4.3 ms of copy before any compute)
    e2_steps = max(3, args.steps)
    # host-fed stream through the public API: every step copies its inputs from
    # pinned host memory and reads its reports back; lk_submit_batch /
    # lk_submit_stereo_batch overlap a step's copy with the previous step's kernels
    rbufs = []
    for _ in range(2):
        rp = C.c_void_p()
        L.lk_host_alloc(C.byref(rp), B * C.sizeof(abi.LkFrameReport))
        rbufs.append(C.cast(rp, C.POINTER(abi.LkFrameReport)))
    submit = L.lk_submit_stereo_batch if stereo else L.lk_submit_batch
    for k in range(2):
        submit(h, hg, hd, B, rbufs[k % 2])
    for _ in range(2):
        L.lk_wait_batch(h)
    torch.cuda.synchronize()
    e2e_failed = []  # failed frames of every streamed batch, counted after its wait

    def drain(k):
        if L.lk_wait_batch(h) not in (abi.LK_OK, abi.LK_ERR_FRAME):
            raise RuntimeError(L.lk_last_error().decode())
        e2e_failed.append(sum(1 for i in range(B) if rbufs[k % 2][i].status))

    h2d0, h2d1 = C.c_ulonglong(0), C.c_ulonglong(0)
    L.lk_h2d_bytes(h, C.byref(h2d0))
    e2.record(stream)
    for k in range(e2_steps):
        submit(h, hg, hd, B, rbufs[k % 2])
        if k >= 1:
            drain(k - 1)
    drain(e2_steps - 1)
    e3.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e2.elapsed_time(e3)
    L.lk_h2d_bytes(h, C.byref(h2d1))  # bytes the copies moved (road-row copy: grey rows from the horizon)
    h2d_per_step = (h2d1.value - h2d0.value) / e2_steps
    # the streamed batches' reports must equal the lk_run_batch ones, byte for byte
    last = rbufs[(e2_steps - 1) % 2]
    rsz = C.sizeof(abi.LkFrameReport)
    e2e_report_mismatch = sum(1 for i in range(B)
                              if C.string_at(C.addressof(last[i]), rsz) != C.string_at(C.addressof(reps[i]), rsz))
    failed = max([failed] + e2e_failed)
    for rb in rbufs:
        L.lk_host_free(C.cast(rb, C.c_void_p))

    from paper_1807_02752_b200 import shard

    dev_ms, e2e_ms = shard.max_over_ranks([dev_ms, e2e_ms])  # slowest GPU sets the time
    (failed,) = shard.sum_over_ranks([failed])

    fps = world * B * args.steps / (dev_ms * 1e-3)
    e2e_fps = world * B * e2_steps / (e2e_ms * 1e-3)
    stage_ms = stage_acc / args.steps
    first = 1 if stereo else 5
    # Roofline timing of the dominant stage: in the timed region several frame
    # ranges run concurrently, so one range's stage events also span the other
    # ranges' kernels. The kernel's own duration is therefore measured on a
    # single-range replay of the same resident batch (same kernels, CUDA events
    # on the library stream), right after the timed region.
    solo_ms = np.zeros(13)
    solo_steps = max(3, min(10, args.steps))
    prev_br = os.environ.get("LK_BRANCHES")
    os.environ["LK_BRANCHES"] = "1"
    try:
        solo = lanekit.GpuPipeline(W, H, cfg, max_batch=B, device=local, stereo=stereo)
    finally:
        if prev_br is None:
            os.environ.pop("LK_BRANCHES", None)
        else:
            os.environ["LK_BRANCHES"] = prev_br
    sh = solo._h
    (L.lk_run_stereo_batch if stereo else L.lk_run_batch)(sh, hg, hd, B, abi.LK_MEM_HOST, reps)
    for _ in range(2):
        (L.lk_enqueue_stereo if stereo else L.lk_enqueue)(sh, B)
    for _ in range(solo_steps):
        (L.lk_enqueue_stereo if stereo else L.lk_enqueue)(sh, B)
        L.lk_stage_times(sh, ms13)
        solo_ms += np.frombuffer(ms13, np.float32)
    solo_ms /= solo_steps
    solo.close()
    dom = int(np.argmax(solo_ms[first:13])) + first
    dom_ms = float(solo_ms[dom])
    tf = B  # frames one solo launch processes
    hbm_peak, peak_src = measured_peaks()
    bytes_per_frame = px * 2  # u8 grey + u8 disparity, or u8 left + right
    achieved = bytes_per_frame * tf / (dom_ms * 1e-3) / 1e9
    win = 2 * ((cfg.bf_window - 1) // 2) + 1
    taps = win * win * px * tf  # nominal range-weight evaluations of one launch
    pipe_fps_hbm = fps / world / (hbm_peak * 1e9 / bytes_per_frame)
    # stage 5 is one kernel, k_vdisparity (K1): the path's HBM-bound kernel.
    # Algorithmic bytes: the u8 disparity read + the transposed i32 histogram written.
    k1_ms = float(solo_ms[5])
    k1_bytes = px + 4 * H * (cfg.d_max + 1)
    k1_gbs = k1_bytes * tf / (k1_ms * 1e-3) / 1e9 if k1_ms > 0 else None

    line = {
        "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "frames_per_step_per_gpu": B, "width": W, "height": H,
                   "distinct_frames_per_gpu": min(pool, B),
                   "l2": f"inputs larger than L2 ({2 * B * px / 1e6:.0f} MB per batch, "
                         f"intermediates several GB)",
                   "parallelism": f"frame-sharded x{world}, no inter-GPU traffic"},
        "clocks": clk.summary(),
        "gpu_launches": launches * args.steps,
        "failed_frames": failed,
        "stage_ms": {str(k): round(float(stage_ms[k]), 4) for k in range(first, 13)},
        "e2e": {"value": e2e_fps, "unit": UNIT, "h2d_bytes_per_step": round(h2d_per_step),
                "report_mismatches_vs_run_batch": e2e_report_mismatch,
                "d2h_bytes_per_step": B * C.sizeof(abi.LkFrameReport),
                "api": ("lk_submit_stereo_batch / lk_wait_batch: pinned host left+right in, "
                        "reports out; step k+1's copy overlaps step k's kernels" if stereo else
                        "lk_submit_batch / lk_wait_batch: pinned host disparity in, then (after "
                        "stages 5-7 of the step on a side stream) the grey rows from the smallest "
                        "horizon - 1 - rho down, reports out; step k+1's copies overlap step k's "
                        "kernels")},
        "roofline": {
            "bound": "hbm", "kernel": f"stage {dom} ({abi.STAGE_NAMES[dom - 1]})",
            "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
            "traffic": None, "peak_source": peak_src,
            "algorithmic_bytes": f"{bytes_per_frame} B/frame (u8 "
                                 f"{'left + right' if stereo else 'grey + disparity'}) x {tf}",
            "frames_per_launch": tf,
            "kernel_ms": dom_ms,
            "timing": f"stage {dom} of a single-range replay of the same resident batch "
                      f"({solo_steps} steps, CUDA events on the library stream); the timed "
                      f"region runs {B // tf_dev} overlapping ranges of {tf_dev} frames",
            "pipeline_frac_of_hbm_roofline": pipe_fps_hbm,
            "compute": {
                "kernel": ("k_prescreen (certified box-moment pre-screen) + k_bilateral_need "
                           "(FP32 bilateral of the survivors' 3x3 neighbourhoods), DESIGN.md §3")
                          if dom == 9 else f"stage {dom} kernels (see stage_ms)",
                "nominal_taps_per_s": taps / (dom_ms * 1e-3) if dom == 9 else None,
                "note": "compute-bound stage (integer dp4a box sums, FP32 bound arithmetic, "
                        "shared-memory range-table gathers); the nominal taps count every pixel's "
                        "121-tap window although only the pre-screen survivors' neighbourhoods "
                        "are filtered (profiles/r02_*_ncu.txt)"},
        },
        "roofline_k1": {
            "bound": "hbm", "kernel": "k_vdisparity (stage 5, TMA bulk-staged rows)",
            "achieved": k1_gbs, "peak": hbm_peak, "unit": "GB/s",
            "frac": k1_gbs / hbm_peak if k1_gbs else None, "kernel_ms": k1_ms,
            "algorithmic_bytes": f"{k1_bytes} B/frame (u8 disparity in, i32 [D1][H] histogram "
                                 f"out) x {tf}",
            "timing": "stage 5 of the same single-range replay (CUDA events)"},
        "notes": f"paper: {PAPER_FPS} fps on GTX 970M + i7 (different hardware, context only)",
    }
    traffic = ROOT / "profiles" / "traffic.json"
    if traffic.exists():
        try:
            tj = json.loads(traffic.read_text()).get(args.config, {})
            t = tj.get(str(dom))
            if t:  # per launch, scaled to the frames this run's launch covers
                line["roofline"]["traffic"] = t * tf / tj["frames"]
        except Exception:
            pass
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if not stereo and args.config == "kitti":
            line["drop_in"] = drop_in_measurements(grey, disp, cfg, local)
        os.sched_setaffinity(0, all_cpus)  # the CPU baseline gets every host core
        cb, ref_reps = cpu_baseline(grey, disp, cfg, frames=2 * (os.cpu_count() or 8),
                                    stereo=stereo)
        line["cpu_baseline"] = cb
        # the frames the baseline just ran, compared report field by report field
        # with this run's GPU reports (tests/parity.py rules: integers exact,
        # FP within 1e-5)
        from parity import compare_reports

        bad = [(i, b) for i, r in enumerate(ref_reps)
               for b in compare_reports(gpu_reps[i], r)]
        line["parity"] = {"frames": len(ref_reps), "against": cb["kind"],
                          "mismatches": len({i for i, _ in bad}),
                          "first": bad[0][1] if bad else None,
                          # the GPU's lane-decision certificate over the whole batch
                          "certified_frames": sum(1 for r in gpu_reps if r.uncertain == 0),
                          "batch_frames": len(gpu_reps)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    pipe.close()
    L.lk_host_free(hg)
    L.lk_host_free(hd)
    if world > 1:
        torch.distributed.destroy_process_group()


def abi_default_copy(cfg, **overrides):
    """A copy of an LkConfig with fields overridden."""
    from paper_1807_02752_b200 import abi

    c = abi.LkConfig.from_buffer_copy(cfg)
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


class GpuStreamEngine:
    """Config-5 engine on one GPU: a resident pool of B distinct frames, batches
    queued with lk_submit_resident (kernels + asynchronous report read-back),
    two pinned report buffers so batch k's records are consumed while batch
    k+1 runs."""

    def __init__(self, B: int, device: int, seed0: int):
        import torch

        from paper_1807_02752_b200 import abi, lanekit, scenes

        self.torch, self.abi = torch, abi
        self.B = B
        grey, disp = make_frames(scenes.batch_scene, B, B, seed0)
        H, W = grey.shape[1:]
        self.pipe = lanekit.GpuPipeline(W, H, abi.default_config(), max_batch=B, device=device)
        self.L = lanekit.library()
        h = self.h = self.pipe._h
        reps = (abi.LkFrameReport * B)()
        st = self.L.lk_run_batch(h, grey.ctypes.data, disp.ctypes.data, B, abi.LK_MEM_HOST, reps)
        if st not in (abi.LK_OK, abi.LK_ERR_FRAME):  # the pool is now resident in HBM
            raise RuntimeError(self.L.lk_last_error().decode())
        self.rbufs = []
        for _ in range(2):
            rp = C.c_void_p()
            self.L.lk_host_alloc(C.byref(rp), B * C.sizeof(abi.LkFrameReport))
            self.rbufs.append(C.cast(rp, C.POINTER(abi.LkFrameReport * B)).contents)
        self.stream = torch.cuda.ExternalStream(self.L.lk_stream(h), device=device)
        self.pending = []

    def submit(self, k: int, n: int):
        if self.L.lk_submit_resident(self.h, n, self.rbufs[k % 2]) != self.abi.LK_OK:
            raise RuntimeError(self.L.lk_last_error().decode())
        self.pending.append((k, n))

    def wait(self, frame0: int):
        from paper_1807_02752_b200 import shard

        k, n = self.pending.pop(0)
        if self.L.lk_wait_batch(self.h) not in (self.abi.LK_OK, self.abi.LK_ERR_FRAME):
            raise RuntimeError(self.L.lk_last_error().decode())
        return shard.compact_records(self.rbufs[k % 2], frame0, n)

    def event(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        return e

    def elapsed_ms(self, e0, e1) -> float:
        e1.synchronize()
        return e0.elapsed_time(e1)

    def close(self):
        for rb in self.rbufs:
            self.L.lk_host_free(C.cast(C.pointer(rb), C.c_void_p))
        self.pipe.close()


def run_stream(args, engine_factory=None, emit=print):
    """BASELINE config 5: N frames sharded over the ranks (contiguous frame
    ranges, shard.shard_range); each rank streams its shard through its own
    engine in batches of B (a resident pool of B distinct frames cycled) and
    the compact lane records are host-gathered on rank 0 (gloo). Timed per rank
    from a barrier to the end of the gather on the engine's device clock; the
    slowest rank sets the time. Returns rank 0's JSON line (None elsewhere)."""
    from paper_1807_02752_b200 import shard

    rank, world, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist

        if not dist.is_initialized():
            dist.init_process_group("gloo")
    N, B = args.stream, args.batch or 256
    lo, hi = shard.shard_range(N, rank, world)
    if engine_factory is None:
        import torch

        device = local % max(1, torch.cuda.device_count())  # ranks may share a GPU
        torch.cuda.set_device(device)
        cpus = shard.bind_local_cpus(device)  # NUMA-local pinned buffers
        engine = GpuStreamEngine(B, device, 1 + lo)
    else:
        cpus, engine = None, engine_factory(B, 1 + lo)
    batches = [(f0, min(B, hi - f0)) for f0 in range(lo, hi, B)]
    for k in range(min(3, len(batches))):  # warm-up (graphs of the batch sizes captured)
        engine.submit(k, batches[k][1])
        engine.wait(0)
    if dist:
        dist.barrier()
    e0 = engine.event()
    recs = []
    for k, (f0, n) in enumerate(batches):
        engine.submit(k, n)
        if k >= 1:
            recs.append(engine.wait(batches[k - 1][0]))
    if batches:
        recs.append(engine.wait(batches[-1][0]))
    local_recs = np.concatenate(recs) if recs else np.zeros(0, shard.RECORD_DTYPE)
    gathered = shard.gather_records(local_recs)
    e1 = engine.event()
    ms = engine.elapsed_ms(e0, e1)
    (ms,) = shard.max_over_ranks([ms])
    failed = int((local_recs["status"] != 0).sum())
    (failed,) = shard.sum_over_ranks([failed])
    engine.close()
    line = None
    if rank == 0:
        ok = gathered is not None and len(gathered) == N and bool(
            np.array_equal(gathered["frame"], np.arange(N, dtype=np.uint32)))
        line = {
            "metric": METRIC, "value": N / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": len(batches), "warmup": min(3, len(batches)),
            "ms_per_step": ms / max(1, len(batches)), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config 5: stream of {N} synthetic KITTI-size 1242x375 "
                                   f"frames sharded over {world} rank(s), batches of {B} from a "
                                   f"resident pool of {B} distinct frames per rank; compact lane "
                                   f"records gathered on rank 0 inside the timed region",
                       "frames": N, "batch": B, "parallelism": f"frame-sharded x{world}",
                       "numa_cpus_rank0": f"{cpus[0]}-{cpus[-1]}" if cpus else None},
            "timing": "per rank: device events on the library stream from a barrier to after "
                      "the gather; max over ranks",
            "records": {"gathered": None if gathered is None else int(len(gathered)),
                        "in_frame_order": ok, "bytes_each": shard.RECORD_DTYPE.itemsize},
            "failed_frames": failed,
        }
        emit(json.dumps(line))
    if dist:
        dist.barrier()
    return line


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.stream:
        run_stream(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
