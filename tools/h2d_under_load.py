"""H2D copy bandwidth alone and while the pipeline's kernels run (device-
resident replays on the library stream), to attribute the e2e gap.
usage: python tools/h2d_under_load.py"""
import ctypes as C
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1807_02752_b200 import abi, lanekit  # noqa: E402


def copy_gbs(h, d, reps=10):
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record()
    e1.synchronize()
    return h.numel() * reps / (e0.elapsed_time(e1) * 1e6)


def main():
    fn, cfg, W, H, B, _ = bench.workload("kitti", 0)
    grey, disp = bench.make_frames(fn, B, B, 1)
    pipe = lanekit.GpuPipeline(W, H, cfg, max_batch=B)
    L = lanekit.library()
    reps = (abi.LkFrameReport * B)()
    L.lk_run_batch(pipe._h, grey.ctypes.data, disp.ctypes.data, B, abi.LK_MEM_HOST, reps)
    n = 2 * B * W * H
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    copy_gbs(h, d, 3)
    alone = copy_gbs(h, d)
    for _ in range(30):  # ~150 ms of kernels queued on the library's own stream
        L.lk_enqueue(pipe._h, B)
    time.sleep(0.005)
    loaded = copy_gbs(h, d)
    L.lk_synchronize(pipe._h)
    print(f"H2D {n / 1e6:.0f} MB: alone {alone:.1f} GB/s, under pipeline load {loaded:.1f} GB/s")


if __name__ == "__main__":
    main()
