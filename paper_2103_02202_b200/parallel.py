"""Multi-GPU plumbing: shot sharding and the end-of-run reductions.

Shots are independent, so the path shards with no exchange during
propagation: rank r owns a contiguous, tile-aligned range of
global shot indices, and the counter-based RNG is keyed by the global tile, so
the union of all ranks' outputs is bit-identical to a single-GPU run.  The only
collectives are at the end: a u64 sum of per-column counts (config 3) and an
optional rank-ordered gather of b8 shards.  One process per GPU, NCCL for CUDA
tensors (gloo works for CPU tensors, which is how the CPU tests drive it).
"""

from __future__ import annotations

import numpy as np


def shard(total_shots: int, world: int, rank: int, tile_shots: int,
          weak: bool = False) -> tuple[int, int]:
    """(global shot offset, shot count) of `rank`.

    weak=True: every rank samples `total_shots` of its own (offset rank*total).
    weak=False: `total_shots` are split into tile-aligned contiguous ranges.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if weak:
        per = -(-total_shots // tile_shots) * tile_shots
        return rank * per, total_shots
    tiles = -(-total_shots // tile_shots)
    base, extra = divmod(tiles, world)
    t0 = rank * base + min(rank, extra)
    nt = base + (1 if rank < extra else 0)
    off = t0 * tile_shots
    cnt = max(0, min(total_shots - off, nt * tile_shots))
    return off, cnt


def all_reduce_counts(counts: np.ndarray, group=None, device=None) -> np.ndarray:
    """Sum uint64 per-column counts over ranks (NCCL on CUDA, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.int64).copy())
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy().astype(np.uint64)


def gather_shards(local: np.ndarray, group=None, device=None) -> np.ndarray | None:
    """Rank-ordered concatenation of per-rank b8 shards along the shot axis
    (returned on rank 0, None elsewhere).  Shards may differ in length."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    arr = np.ascontiguousarray(local, dtype=np.uint8)
    n = torch.tensor([arr.shape[0]], dtype=torch.int64, device=device)
    sizes = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    width = arr.shape[1] if arr.ndim == 2 else 0
    mx = max(sizes)
    buf = np.zeros((mx, width), dtype=np.uint8)
    buf[:arr.shape[0]] = arr
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    outs = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    if rank != 0:
        return None
    return np.concatenate([o.cpu().numpy()[:s] for o, s in zip(outs, sizes)], axis=0)


def rank_offset(shots_per_rank: int, world: int, rank: int, tile_shots: int) -> int:
    """Global shot offset of `rank` under weak scaling (bench.py: every rank
    samples `shots_per_rank` shots of its own, tile-aligned, disjoint)."""
    return shard(shots_per_rank, world, rank, tile_shots, weak=True)[0]


def reduce_max(value: float, device=None) -> float:
    """Max of a per-rank scalar (device-timed seconds) over all ranks; the
    value itself when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def counts_steps(sample_counts, counts, shots_per_rank: int, tile_shots: int, world: int, rank: int,
                 steps: int, seed0: int):
    """The config-3 step loop of bench.py: `steps` weak-scaled sampling steps of
    per-column event counts on this rank (`sample_counts(shots, seed, offset,
    out)` overwrites `counts`, a torch int64 tensor), then one in-place sum
    over ranks (NCCL for CUDA tensors, gloo for CPU ones).  Returns `counts`:
    the last step's counts summed over all ranks."""
    import torch.distributed as dist

    off = rank_offset(shots_per_rank, world, rank, tile_shots)
    for i in range(steps):
        sample_counts(shots_per_rank, seed0 + i, off, counts)
    if world > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    return counts
