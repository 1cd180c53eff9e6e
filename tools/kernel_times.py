"""Device-resident replays only (no e2e, no CPU baseline): a clean target for
an ncu launch list. usage: python tools/kernel_times.py [kitti|hires] [steps] [stereo]"""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1807_02752_b200 import abi, lanekit  # noqa: E402


def main():
    # one range per launch: every kernel launch covers the whole batch
    os.environ.setdefault("LK_BRANCHES", "1")
    os.environ.setdefault("LK_H2D_CHUNKS", "1")
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "kitti"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    stereo = len(sys.argv) > 3 and sys.argv[3] == "stereo"
    fn, cfg, W, H, B, _ = bench.workload(cfg_name, 0)
    grey, disp = bench.make_frames(fn, B, B, 1, stereo)
    pipe = lanekit.GpuPipeline(W, H, cfg, max_batch=B, stereo=stereo)
    L = lanekit.library()
    h = pipe._h
    dg, dd = C.c_void_p(), C.c_void_p()
    L.lk_device_inputs(h, C.byref(dg), C.byref(dd))
    reps = (abi.LkFrameReport * B)()
    run = L.lk_run_stereo_batch if stereo else L.lk_run_batch
    run(h, grey.ctypes.data, disp.ctypes.data, B, abi.LK_MEM_HOST, reps)
    for _ in range(steps):
        (L.lk_enqueue_stereo if stereo else L.lk_enqueue)(h, B)
    L.lk_synchronize(h)
    print("ok", B, "frames x", steps)


if __name__ == "__main__":
    main()
