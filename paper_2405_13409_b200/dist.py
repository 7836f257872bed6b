"""Multi-GPU plumbing of the hot path: the path shards by query, there is no exchange step
inside a solve, so the only collectives are the final gathers.

- ``shard_tiles``: fixed tiles of queries assigned round-robin to ranks (tile t -> rank t mod g), so hot
  spots (caustic focus regions) spread over ranks without work stealing (strong scaling of one frame).
- ``gather_per_query``: every rank's per-query sums of its shard -> the full per-query array on every rank
  (``all_gather`` of equal-size padded slices, then a local scatter back to query order).
- ``allreduce_counters``: sum of the SolveReport counters.

Works with any torch.distributed backend (``nccl`` on the GPU box, ``gloo`` in the CPU tests).  No solve
arithmetic lives here.
"""
from __future__ import annotations

import numpy as np


def shard_tiles(nq: int, world: int, rank: int, tile: int = 4096) -> np.ndarray:
    """Query indices owned by `rank`: tiles of `tile` consecutive queries, tile t -> rank t % world."""
    ntiles = (nq + tile - 1) // tile
    mine = [np.arange(t * tile, min(nq, (t + 1) * tile)) for t in range(rank, ntiles, world)]
    return np.concatenate(mine) if mine else np.zeros(0, np.int64)


def gather_per_query(local_vals, local_idx, nq: int, group=None):
    """local_vals: tensor (n_local,) float64 (this rank's per-query sums, order of local_idx).
    Returns a tensor (nq,) float64 with every rank's values at their global query index."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = local_vals.device
    n = torch.tensor([local_vals.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    m = int(max(int(s.item()) for s in sizes))
    pv = torch.zeros(m, dtype=local_vals.dtype, device=dev)
    pi = torch.full((m,), -1, dtype=torch.int64, device=dev)
    pv[:local_vals.numel()] = local_vals
    pi[:local_vals.numel()] = torch.as_tensor(np.asarray(local_idx), dtype=torch.int64, device=dev)
    gv = [torch.empty_like(pv) for _ in range(world)]
    gi = [torch.empty_like(pi) for _ in range(world)]
    dist.all_gather(gv, pv, group=group)
    dist.all_gather(gi, pi, group=group)
    out = torch.zeros(nq, dtype=local_vals.dtype, device=dev)
    for v, i in zip(gv, gi):
        keep = i >= 0
        out[i[keep]] = v[keep]
    return out


def allreduce_counters(counters: dict, device, group=None) -> dict:
    import torch
    import torch.distributed as dist
    keys = sorted(counters)
    t = torch.tensor([float(counters[k]) for k in keys], dtype=torch.float64, device=device)
    dist.all_reduce(t, group=group)
    return {k: int(v) for k, v in zip(keys, t.tolist())}
