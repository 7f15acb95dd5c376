"""Multi-GPU report gather.

Instances shard contiguously across ranks (rank r owns instances
[r*I/G, (r+1)*I/G) and passes instance_offset accordingly), so there is no
exchange during execution.  The only collective is this gather: an
all_gather of each rank's {report count, rc_stats}, then of the report
buffers padded to the largest count.  Concatenating in rank order is already
globally canonical because instance ranges ascend with the rank.

torch.distributed is the plumbing (NCCL over NVLink on GPUs, gloo in the CPU
tests); reports move as raw 32-byte records viewed as int32.
"""
from __future__ import annotations

import numpy as np

from .rc import REPORT_DTYPE

STAT_FIELDS = ["checked_accesses", "loads", "stores", "instructions", "intervals_max"]


def shard(n_instances: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous instance range of `rank` (remainder spread over the first ranks)."""
    base, rem = divmod(n_instances, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def gather_reports(reports: np.ndarray, stats: dict, group=None, device=None):
    """All-gather reports + stats of every rank.  Returns (reports, stats) of
    the whole job on every rank: reports concatenated in rank order, stats
    summed (intervals_max: max)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")
    head = np.zeros(2 + len(STAT_FIELDS) + 8, dtype=np.int64)
    head[0] = len(reports)
    head[1:1 + len(STAT_FIELDS)] = [int(stats[k]) for k in STAT_FIELDS]
    head[1 + len(STAT_FIELDS):1 + len(STAT_FIELDS) + 8] = stats["lanes_final"]
    h = torch.from_numpy(head).to(dev)
    hs = torch.empty((world * h.numel(),), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(hs, h, group=group)
    hs = hs.cpu().numpy().reshape(world, -1)
    counts = hs[:, 0]
    mx = int(counts.max())
    out_stats = {k: int(hs[:, 1 + i].sum()) for i, k in enumerate(STAT_FIELDS)}
    out_stats["intervals_max"] = int(hs[:, 1 + STAT_FIELDS.index("intervals_max")].max())
    out_stats["lanes_final"] = [int(x) for x in hs[:, 1 + len(STAT_FIELDS):1 + len(STAT_FIELDS) + 8].sum(0)]
    if mx == 0:
        return np.zeros(0, dtype=REPORT_DTYPE), out_stats
    buf = np.zeros(mx, dtype=REPORT_DTYPE)
    buf[:len(reports)] = reports
    t = torch.from_numpy(buf.view(np.int32).reshape(mx, 8).copy()).to(dev)
    ts = torch.empty((world * mx, 8), dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(ts, t, group=group)
    ts = ts.cpu().numpy().reshape(world, mx, 8)
    parts = [ts[r, :counts[r]].copy().view(REPORT_DTYPE).reshape(-1) for r in range(world)]
    return np.concatenate(parts), out_stats
