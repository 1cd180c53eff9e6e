"""Host feed probe for the e2e (host-fed) path: how fast can pinned host memory
reach one GPU, and how much host DRAM bandwidth is there to feed eight?

  python tools/h2d_probe.py [--out profiles/r02_h2d_probe.json]

Measures (CUDA events / wall clock, best of 5):
  - H2D from pinned memory, 1 stream, 238 MB (one KITTI batch of grey + disparity);
  - the same split over 2 and 4 concurrent streams (separate pinned buffers);
  - host memcpy bandwidth with 1..all threads (numpy copies release the GIL):
    the ceiling on frames/s that host DRAM can source for N GPUs at once.
The 8-GPU e2e ceiling printed is min(8 x per-GPU link, host copy bandwidth)
/ 931,500 B per frame; the per-GPU link figure is this box's (one GPU).
"""
import argparse
import json
import os
import threading
import time

import numpy as np
import torch

BYTES_PER_FRAME = 1242 * 375 * 2


def h2d(n_bytes, streams, reps=5):
    hs = [torch.empty(n_bytes // streams, dtype=torch.uint8, pin_memory=True) for _ in range(streams)]
    ds = [torch.empty(n_bytes // streams, dtype=torch.uint8, device="cuda") for _ in range(streams)]
    ss = [torch.cuda.Stream() for _ in range(streams)]
    best = 0.0
    for _ in range(reps + 2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for h, d, s in zip(hs, ds, ss):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d.copy_(h, non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, n_bytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def host_copy(n_bytes, threads, reps=3):
    src = np.ones(n_bytes, np.uint8)
    dst = np.empty_like(src)
    chunks = np.array_split(np.arange(n_bytes), threads)
    bounds = [(c[0], c[-1] + 1) for c in chunks if len(c)]
    best = 0.0
    for _ in range(reps):
        ts = [threading.Thread(target=lambda a=a, b=b: np.copyto(dst[a:b], src[a:b])) for a, b in bounds]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        dt = time.perf_counter() - t0
        best = max(best, 2 * n_bytes / dt / 1e9)  # read + write
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    n = 256 * BYTES_PER_FRAME
    res = {"batch_bytes": n, "h2d_gbs": {str(k): h2d(n, k) for k in (1, 2, 4)}}
    cores = os.cpu_count() or 1
    res["host_copy_gbs"] = {str(t): host_copy(n, t) for t in sorted({1, 4, cores // 2 or 1, cores})}
    link = max(res["h2d_gbs"].values())
    host = max(res["host_copy_gbs"].values())
    res["gpu"] = torch.cuda.get_device_name(0)
    res["host_cores"] = cores
    res["e2e_ceiling_frames_per_s"] = {
        "1_gpu_link": link * 1e9 / BYTES_PER_FRAME,
        "8_gpu_links": 8 * link * 1e9 / BYTES_PER_FRAME,
        "host_dram_copy": host * 1e9 / BYTES_PER_FRAME,
        "note": "8 GPUs are fed at min(8 x link, host DRAM) only if each GPU has its own "
                "PCIe root and the pinned buffers are NUMA-local (shard.bind_local_cpus); the "
                "link figure is measured on this single-GPU box",
    }
    print(json.dumps(res, indent=1))
    if a.out:
        open(a.out, "w").write(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
