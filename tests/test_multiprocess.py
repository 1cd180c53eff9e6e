"""The N>1 path on CPU: two gloo ranks shard the frames, each processes its
contiguous range (with the CPU oracle standing in for the GPU, which this
container does not have), timings are max-reduced and the lane records are
gathered on rank 0 — and must equal a single-process run frame for frame."""
import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_frames, out_path):
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import json

    import torch.distributed as dist

    from checkers import Checker
    from paper_1807_02752_b200 import lanekit, scenes, shard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard.shard_range(n_frames, rank, world)
    params = [scenes.acceptance_scene(i) for i in range(lo, hi)]
    grey, disp = lanekit.synth_batch(params, threads=2)
    reps = Checker("oracle").run_batch(grey, disp, scenes.acceptance_config(), threads=2)
    recs = shard.gather_records([shard.lane_record(r) for r in reps])
    t = shard.max_over_ranks([float(rank + 1), 10.0 * (world - rank)])
    f = shard.sum_over_ranks([sum(r.status != 0 for r in reps), hi - lo])
    if rank == 0:
        Path(out_path).write_text(json.dumps({"records": recs, "t": t, "f": f}))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_partition():
    from paper_1807_02752_b200 import shard

    for n in (1, 7, 256, 65536):
        for world in (1, 2, 4, 8):
            ranges = [shard.shard_range(n, g, world) for g in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def test_two_rank_gloo_shards_match_single_process(tmp_path):
    import json

    from checkers import Checker
    from paper_1807_02752_b200 import lanekit, scenes, shard

    n = 6
    out = tmp_path / "rank0.json"
    mp.spawn(_worker, args=(2, _free_port(), n, str(out)), nprocs=2, join=True)
    got = json.loads(out.read_text())
    params = [scenes.acceptance_scene(i) for i in range(n)]
    grey, disp = lanekit.synth_batch(params, threads=2)
    reps = Checker("oracle").run_batch(grey, disp, scenes.acceptance_config(), threads=2)
    want = [shard.lane_record(r) for r in reps]
    assert json.loads(json.dumps(want)) == got["records"]
    assert got["t"] == [2.0, 20.0]      # max over ranks
    assert got["f"] == [0, n]           # failures summed, frames summed


class _CpuStreamEngine:
    """bench.run_stream's engine contract on CPU: the oracle (test infrastructure)
    stands in for the GPU; a pool of B acceptance-size frames cycled."""

    def __init__(self, B, seed0):
        import time

        from checkers import Checker
        from paper_1807_02752_b200 import lanekit, scenes

        self.time = time
        self.grey, self.disp = lanekit.synth_batch(
            [scenes.acceptance_scene(seed0 + i) for i in range(B)], threads=2)
        self.chk, self.cfg, self.pending = Checker("oracle"), scenes.acceptance_config(), []

    def submit(self, k, n):
        self.pending.append(n)

    def wait(self, frame0):
        import ctypes as C

        from paper_1807_02752_b200 import abi, shard

        n = self.pending.pop(0)
        reps = self.chk.run_batch(self.grey[:n], self.disp[:n], self.cfg, threads=2)
        arr = (abi.LkFrameReport * n)(*reps)
        return shard.compact_records(arr, frame0)

    def event(self):
        return self.time.perf_counter()

    def elapsed_ms(self, e0, e1):
        return (e1 - e0) * 1e3

    def close(self):
        pass


def _stream_worker(rank, world, port, out_path):
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import argparse
    import json

    import bench

    args = argparse.Namespace(stream=10, batch=4)
    line = bench.run_stream(args, engine_factory=_CpuStreamEngine, emit=lambda s: None)
    if rank == 0:
        Path(out_path).write_text(json.dumps(line))


def test_bench_stream_two_ranks_gather(tmp_path):
    """bench.py --stream under two gloo ranks: shards [0, 5) and [5, 10), batches of
    4 (+1), the compact lane records gathered on rank 0 in frame order, the slowest
    rank's time, one JSON line on rank 0 only."""
    import json

    out = tmp_path / "line.json"
    mp.spawn(_stream_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    line = json.loads(out.read_text())
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["records"] == {"gathered": 10, "in_frame_order": True,
                               "bytes_each": line["records"]["bytes_each"]}
    assert line["failed_frames"] == 0 and line["value"] > 0
    assert line["config"]["frames"] == 10 and line["steps"] == 2


def test_bench_reference_arm_two_ranks():
    """bench.py --impl reference launched as the driver launches it for N = 2
    (torchrun, 127.0.0.1): rank 0 alone times the compiled reference on the host
    cores and prints one JSON line; rank 1 exits 0 without work."""
    import json
    import subprocess

    if not (ROOT / "oracle" / "_ref" / "liblk_ref.so").exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
