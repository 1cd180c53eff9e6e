"""Frame sharding across GPUs: contiguous frame ranges per
rank, no inter-GPU traffic on the data path; the only exchanges are the
max-over-ranks device time and a host gather of the compact per-frame lane
records. torch.distributed is plumbing here (gloo works on CPU)."""
from __future__ import annotations

from typing import Sequence

import numpy as np

from . import abi

# compact per-frame record of the host gather (~64 B + 12 B per lane)
RECORD_DTYPE = np.dtype([
    ("frame", "<u4"), ("status", "<i4"), ("failed_stage", "<i4"), ("horizon", "<i4"),
    ("beta", "<f8", 3), ("gamma", "<f8", 5), ("lane_count", "<i4"),
    ("lane_bottom_col", "<i4", abi.LK_MAX_INLINE_LANES),
    ("lane_energy", "<f4", abi.LK_MAX_INLINE_LANES), ("uncertain", "<i4"),
])


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
            "lanes": list(zip(d["lane_bottom_col"], d["lane_energy"])),
            "uncertain": d["uncertain"]}


def compact_records(reports, frame0: int, n: int | None = None) -> np.ndarray:
    """Compact records of a ctypes array of LkFrameReport (frames frame0, ...):
    one vectorised copy through the reports' structured numpy view."""
    rep = np.ctypeslib.as_array(reports)
    if n is not None:
        rep = rep[:n]
    out = np.zeros(len(rep), RECORD_DTYPE)
    out["frame"] = frame0 + np.arange(len(rep), dtype=np.uint32)
    for k in ("status", "failed_stage", "horizon", "beta", "gamma", "lane_count",
              "lane_bottom_col", "lane_energy", "uncertain"):
        out[k] = rep[k]
    return out


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


def gather_records(records):
    """Host gather of every rank's records, in rank (= frame) order, on rank 0:
    a list of dicts (lane_record) or a RECORD_DTYPE array (compact_records)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return records
    out = [None] * dist.get_world_size() if dist.get_rank() == 0 else None
    dist.gather_object(records, out, dst=0)
    if dist.get_rank() != 0:
        return None
    if isinstance(records, np.ndarray):
        return np.concatenate(out)
    return [r for part in out for r in part]


def local_cpus(device: int) -> list[int] | None:
    """Host CPUs on the NUMA node of CUDA device `device` (sysfs local_cpulist of
    its PCI function), or None when unknown."""
    try:
        import torch

        props = torch.cuda.get_device_properties(device)
        bus = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
        txt = open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
    except Exception:
        return None
    cpus = []
    for part in txt.split(","):
        a, _, b = part.partition("-")
        cpus += list(range(int(a), int(b or a) + 1))
    return cpus or None


def bind_local_cpus(device: int) -> list[int] | None:
    """Pins this process to the CPUs of its GPU's NUMA node, so pinned host
    buffers allocated afterwards (first touch by this process) are NUMA-local
    to the GPU's PCIe root."""
    import os

    cpus = local_cpus(device)
    if cpus:
        try:
            os.sched_setaffinity(0, cpus)
        except OSError:
            return None
    return cpus
