"""World-size-2 gloo test of the multi-GPU plumbing (query-tile sharding + gathers), on CPU.

Each rank solves its shard with the oracle (the solve is irrelevant to the plumbing; the GPU ranks call
spoly_solve instead) and the gathered per-query array must equal the single-process result exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2405_13409_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_tiles_partition():
    for nq, world, tile in [(1000, 2, 64), (65536, 8, 4096), (5, 4, 2), (0, 2, 8)]:
        parts = [D.shard_tiles(nq, world, r, tile) for r in range(world)]
        allq = np.sort(np.concatenate(parts)) if nq else np.zeros(0)
        assert np.array_equal(allq, np.arange(nq))
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= tile


def test_shard_grid_tiles_partition():
    """64 x 64 tiles of a row-major grid, round-robin: a partition of the queries, every tile square and whole."""
    for w, h, world in [(256, 256, 8), (1024, 1024, 8), (100, 70, 3), (64, 64, 2), (1, 1, 4)]:
        parts = [D.shard_grid_tiles(w, h, world, r) for r in range(world)]
        allq = np.sort(np.concatenate(parts))
        assert np.array_equal(allq, np.arange(w * h))
        ntiles = ((w + 63) // 64) * ((h + 63) // 64)
        for r, p in enumerate(parts):
            assert len(p) <= ((ntiles - r + world - 1) // world) * 64 * 64
            if len(p):
                y, x = np.divmod(p[:64 * 64], w)
                assert y.max() - y.min() < 64 and x.max() - x.min() < 64  # first tile is a 64 x 64 block


def test_grid_tile_side_keeps_ranks_busy():
    """small frames get smaller tiles (at least 4 per rank, down to 8 x 8); large frames keep 64 x 64"""
    assert D.grid_tile_side(1024, 1024, 8) == 64
    assert D.grid_tile_side(256, 256, 8) == 32      # 16 tiles of 64 < 32 -> 64 tiles of 32
    assert D.grid_tile_side(128, 128, 8) == 16      # C4: 256 tiles of 16 x 16
    assert D.grid_tile_side(32, 32, 8) == 8
    for w, world in [(128, 8), (256, 4), (100, 3)]:
        t = D.grid_tile_side(w, w, world)
        parts = [D.shard_grid_tiles(w, w, world, r, t) for r in range(world)]
        assert np.array_equal(np.sort(np.concatenate(parts)), np.arange(w * w))
        assert min(len(p) for p in parts) > 0


def _worker(rank, world, port, ret):
    import torch
    import torch.distributed as dist
    import oracle
    from paper_2405_13409_b200 import workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = W.patch_c1()
    ep = np.repeat(w.endpoints, 24, axis=0)
    ep[:, 1, 0] += np.linspace(-0.3, 0.3, 24)
    nq = ep.shape[0]
    idx = D.shard_tiles(nq, world, rank, tile=5)
    r = oracle.solve(w.mesh, "R", ep[idx], cfg=oracle.default_config(), nthreads=1)
    full = D.gather_per_query(torch.as_tensor(r.per_query), idx, nq)
    cnt = D.allreduce_counters({"admissible": r.report["admissible"], "pairs": r.report["pairs_in"],
                                "big": (1 << 60) + rank}, "cpu")
    # solution rows (query, u, v) gathered in chunks of 3 rows: ragged counts, many rounds
    rows = torch.as_tensor(np.c_[idx[r.query], r.bary])
    allrows = D.gather_rows(rows, chunk=3)
    mx, mean = D.allreduce_max_mean(float(rank + 1), "cpu")
    if rank == 0:
        ret["full"] = full.numpy().tolist()
        ret["cnt"] = cnt
        ret["rows"] = allrows.numpy().tolist()
        ret["maxmean"] = (mx, mean)
    dist.barrier()
    dist.destroy_process_group()


def test_gather_matches_single_process():
    import oracle
    from paper_2405_13409_b200 import workloads as W
    oracle.build()
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, port, ret), nprocs=2, join=True)
    w = W.patch_c1()
    ep = np.repeat(w.endpoints, 24, axis=0)
    ep[:, 1, 0] += np.linspace(-0.3, 0.3, 24)
    ref = oracle.solve(w.mesh, "R", ep, nthreads=1)
    assert np.array_equal(np.array(ret["full"]), ref.per_query)
    assert ret["cnt"]["admissible"] == ref.report["admissible"]
    assert ret["cnt"]["pairs"] == ref.report["pairs_in"]
    assert ret["cnt"]["big"] == 2 * (1 << 60) + 1  # exact int64 reduction (a float64 sum would round)
    rows = np.array(ret["rows"])
    got = sorted(map(tuple, rows))
    want = sorted(map(tuple, np.c_[ref.query, ref.bary]))
    assert got == want
    assert ret["maxmean"] == (2.0, 1.5)
