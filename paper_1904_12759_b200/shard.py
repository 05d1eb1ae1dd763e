"""Row sharding over GPUs.

Entries are independent, so each rank estimates a contiguous, equal-count
block of the requested rows on its own full matrix replica; the only
exchange is the final gather of the (value, std_error, jumps) slices.
Because a walker's Philox stream is keyed by (seed, row, walker) and the
per-entry reduction order is fixed, the gathered vector is bitwise identical
for any number of ranks.

The gather uses ``torch.distributed`` (NCCL on GPUs, gloo in the CPU tests):
slices are padded to equal length and all-gathered in one collective.
"""
from __future__ import annotations

import numpy as np


def plan_shards(nrows: int, world: int):
    """Contiguous equal-count blocks: [(lo, hi)] for ranks 0..world-1."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    base, rem = divmod(nrows, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


def shard_rows(rows: np.ndarray, rank: int, world: int) -> np.ndarray:
    lo, hi = plan_shards(len(rows), world)[rank]
    return rows[lo:hi]


def gather_slices(value, se, jumps, nrows: int, group=None):
    """All-gather per-rank slices (torch tensors, float64 / float64 / int64,
    on the backend's device) into full-length tensors, in rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    plan = plan_shards(nrows, world)
    width = max(hi - lo for lo, hi in plan)
    dev = value.device
    packed = torch.zeros(3, width, dtype=torch.float64, device=dev)
    k = value.numel()
    packed[0, :k] = value
    packed[1, :k] = se
    packed[2, :k] = jumps.view(torch.float64) if jumps.dtype == torch.int64 else \
        jumps.to(torch.int64).view(torch.float64)
    flat = torch.empty(world * 3 * width, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(flat, packed.reshape(-1), group=group)
    out = flat.view(world, 3, width)
    vals, ses, js = [], [], []
    for r, (lo, hi) in enumerate(plan):
        m = hi - lo
        vals.append(out[r, 0, :m])
        ses.append(out[r, 1, :m])
        js.append(out[r, 2, :m].contiguous().view(torch.int64))
    return torch.cat(vals), torch.cat(ses), torch.cat(js)
