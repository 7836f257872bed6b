"""Multi-GPU plumbing of the hot path: the path shards by query, there is no exchange step
inside a solve, so the only collectives are the final reductions and gathers.

- ``shard_grid_tiles``: a row-major W x H query grid cut into 64 x 64 tiles, tile t -> rank t mod g
  (strong scaling of one frame; caustic hot spots spread over ranks without work stealing).
- ``shard_tiles``: the same for an unstructured query list (runs of ``tile`` consecutive queries).
- ``gather_per_query``: every rank's per-query sums of its shard -> the full per-query array on every rank
  (``all_gather`` of equal-size padded slices, then a local scatter back to query order).
- ``gather_rows``: ragged per-rank row arrays (e.g. solution lists) -> rank order on every rank, moved in
  ``chunk``-row padded ``all_gather`` rounds so no rank ever allocates more than world x chunk rows of buffer.
- ``allreduce_counters``: exact int64 sum of the SolveReport counters; ``allreduce_max_mean``: max and mean of
  a per-rank time.

Works with any torch.distributed backend (``nccl`` on the GPU box, ``gloo`` in the CPU tests).  No solve
arithmetic lives here.
"""
from __future__ import annotations

import numpy as np


def grid_tile_side(width: int, height: int, world: int, tile: int = 64, min_tile: int = 8) -> int:
    """64, halved while the frame would give fewer than 4 tiles per rank (a 128 x 128 frame has only 4 tiles of 64:
    over 8 ranks half of them would idle), down to `min_tile`."""
    while tile > min_tile and ((width + tile - 1) // tile) * ((height + tile - 1) // tile) < 4 * world:
        tile //= 2
    return tile


def shard_grid_tiles(width: int, height: int, world: int, rank: int, tile: int = 64) -> np.ndarray:
    """Query indices (row-major, q = y * width + x) owned by `rank`: tile (ty, tx) has index t = ty * ntx + tx
    and goes to rank t % world; within a tile, row-major.  Ragged edge tiles are kept whole."""
    ntx = (width + tile - 1) // tile
    nty = (height + tile - 1) // tile
    out = []
    for t in range(rank, ntx * nty, world):
        ty, tx = divmod(t, ntx)
        ys = np.arange(ty * tile, min(height, (ty + 1) * tile))
        xs = np.arange(tx * tile, min(width, (tx + 1) * tile))
        out.append((ys[:, None] * width + xs[None, :]).ravel())
    return np.concatenate(out).astype(np.int64) if out else np.zeros(0, np.int64)


def shard_tiles(nq: int, world: int, rank: int, tile: int = 4096) -> np.ndarray:
    """Unstructured query list: tiles of `tile` consecutive queries, tile t -> rank t % world."""
    ntiles = (nq + tile - 1) // tile
    mine = [np.arange(t * tile, min(nq, (t + 1) * tile)) for t in range(rank, ntiles, world)]
    return np.concatenate(mine).astype(np.int64) if mine else np.zeros(0, np.int64)


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


def gather_rows(local_rows, chunk: int = 1 << 20, group=None):
    """local_rows: tensor (n_local, ...) on this rank.  Returns the concatenation of every rank's rows in rank
    order (identical on every rank).  Rows move in rounds of at most `chunk` rows per rank (padded all_gather),
    so the staging buffers stay bounded however ragged the ranks' counts are."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = local_rows.device
    n = torch.tensor([local_rows.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    counts = [int(s.item()) for s in sizes]
    rest = tuple(local_rows.shape[1:])
    parts = [[] for _ in range(world)]
    rounds = (max(counts) + chunk - 1) // chunk if max(counts) else 0
    for r in range(rounds):
        lo = r * chunk
        buf = torch.zeros((chunk,) + rest, dtype=local_rows.dtype, device=dev)
        mine = local_rows[lo:lo + chunk]
        buf[:mine.shape[0]] = mine
        got = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(got, buf, group=group)
        for w in range(world):
            take = max(0, min(chunk, counts[w] - lo))
            if take:
                parts[w].append(got[w][:take])
    flat = [p for w in range(world) for p in parts[w]]
    return torch.cat(flat) if flat else torch.zeros((0,) + rest, dtype=local_rows.dtype, device=dev)


def allreduce_counters(counters: dict, device, group=None) -> dict:
    """Exact sum over ranks of integer counters (int64 on the wire: no float rounding above 2^53)."""
    import torch
    import torch.distributed as dist
    keys = sorted(counters)
    t = torch.tensor([int(counters[k]) for k in keys], dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    return {k: int(v) for k, v in zip(keys, t.tolist())}


def allreduce_max_mean(value: float, device, group=None):
    """(max, mean) over ranks of a per-rank float (e.g. a rank's device time)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor([value, value], dtype=torch.float64, device=device)
    mx = t[:1].clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    sm = t[1:].clone()
    dist.all_reduce(sm, group=group)
    return float(mx.item()), float(sm.item()) / world
