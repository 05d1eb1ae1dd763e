"""Row sharding over GPUs.

Entries are independent, so each rank estimates a contiguous, equal-count
block of the requested rows on its own full matrix replica; the only
exchange is the final gather of the (value, std_error, jumps) slices.
Because a walker's Philox stream is keyed by (seed, row, walker) and the
per-entry reduction order is fixed, the gathered vector is bitwise identical
for any number of ranks.

The gather uses ``torch.distributed`` (NCCL on GPUs, gloo in the CPU tests):
slices are padded to equal length and all-gathered in one collective.

The Theorem-2 estimators (vector_estimate / tc_estimate) shard by START
row: every rank draws the same multinomial start counts and global jumper
numbering (a pure function of the seed), then runs only the walkers that
start in its row block.  The shards run exactly the unsharded call's
walkers; their per-end contributions (full n-vectors: walkers end anywhere)
and tallies are all-gathered and added in rank order, so the result is
deterministic for a given rank count and equal to the single-GPU result up
to floating-point summation order (tested to 1e-12).
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


def combine_vector_shards(parts, samples: int, v_sum: float):
    """Rank-ordered combination of vector_estimate_rows results
    [(values, s1, s2, jumps)] into a VectorEstimate (finalize on the totals)."""
    from .estimator import VectorEstimate, finalize

    vals = np.array(parts[0][0], dtype=np.float64, copy=True)
    s1, s2, jm = parts[0][1], parts[0][2], parts[0][3]
    for v, a, b, j in parts[1:]:
        vals += v
        s1 += a
        s2 += b
        jm += j
    est = finalize(s1, s2, samples, jm)
    return VectorEstimate(vals, est.std_error, samples, int(jm), v_sum)


def combine_tc_shards(parts, samples: int):
    """Rank-ordered combination of tc_estimate_rows results [(s1, s2, jumps)]."""
    from .estimator import finalize

    s1, s2, jm = parts[0]
    for a, b, j in parts[1:]:
        s1 += a
        s2 += b
        jm += j
    return finalize(s1, s2, samples, jm)


def _gather_packed(local: np.ndarray, group=None):
    """All-gather one float64 vector of equal length per rank -> [world, len]."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else \
        torch.device("cpu")
    t = torch.from_numpy(local).to(dev)
    out = torch.empty(world * t.numel(), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(out, t, group=group)
    return out.view(world, -1).cpu().numpy()


def _pack(values, s1, s2, jumps):
    tail = np.array([s1, s2, 0.0])
    tail[2:] = np.array([jumps], dtype=np.uint64).view(np.float64)
    return np.concatenate([values, tail])


def _unpack(row, n):
    return row[:n], float(row[n]), float(row[n + 1]), int(row[n + 2:n + 3].view(np.uint64)[0])


def vector_estimate_sharded(m, v, p, group=None, shard_fn=None):
    """vector_estimate over the ranks of ``group``: rank r runs the walkers
    starting in its contiguous row block, shards are gathered and combined in
    rank order.  ``shard_fn(lo, hi)`` overrides the per-rank computation (the
    CPU tests pass a stand-in)."""
    import torch.distributed as dist

    from .estimator import vector_estimate_rows

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = len(v)
    lo, hi = plan_shards(n, world)[rank]
    if shard_fn is None:
        vals, s1, s2, jm = vector_estimate_rows(m, v, p, lo, hi)
    else:
        vals, s1, s2, jm = shard_fn(lo, hi)
    rows = _gather_packed(_pack(np.asarray(vals, np.float64), s1, s2, jm), group)
    parts = [_unpack(rows[r], n) for r in range(world)]
    return combine_vector_shards(parts, p.samples, float(np.sum(np.asarray(v, np.float64))))


def tc_estimate_sharded(m, p, n: int, group=None, shard_fn=None):
    """tc_estimate over the ranks of ``group`` (start-row shards, rank order)."""
    import torch.distributed as dist

    from .estimator import tc_estimate_rows

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = plan_shards(n, world)[rank]
    s1, s2, jm = (tc_estimate_rows(m, p, lo, hi) if shard_fn is None else shard_fn(lo, hi))
    rows = _gather_packed(_pack(np.zeros(0), s1, s2, jm), group)
    return combine_tc_shards([_unpack(rows[r], 0)[1:] for r in range(world)], p.samples)
