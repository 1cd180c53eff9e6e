"""Frame sharding across GPUs: contiguous frame ranges per
rank, no inter-GPU traffic on the data path; the only exchanges are the
max-over-ranks device time and a host gather of the compact per-frame lane
records. torch.distributed is plumbing here (gloo works on CPU)."""
from __future__ import annotations

from typing import Sequence


def shard_range(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Frames [g*N/G, (g+1)*N/G) for rank g."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    return rank * n_frames // world, (rank + 1) * n_frames // world


def lane_record(rep) -> dict:
    """Compact host-side record of one frame (~64 B + 12 B per lane)."""
    d = rep.as_dict()
    return {"status": d["status"], "failed_stage": d["failed_stage"], "beta": d["beta"],
            "gamma": d["gamma"], "horizon": d["horizon"], "lane_count": d["lane_count"],
            "lanes": list(zip(d["lane_bottom_col"], d["lane_energy"]))}


def max_over_ranks(values: Sequence[float]) -> list[float]:
    """Element-wise max over ranks (device timings: the slowest GPU sets the time)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def sum_over_ranks(values: Sequence[int]) -> list[int]:
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.int64)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t)
    return [int(x) for x in t.tolist()]


def gather_records(records: list) -> list | None:
    """Host gather of every rank's records, in rank (= frame) order, on rank 0."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return records
    out = [None] * dist.get_world_size() if dist.get_rank() == 0 else None
    dist.gather_object(records, out, dst=0)
    if dist.get_rank() != 0:
        return None
    return [r for part in out for r in part]
