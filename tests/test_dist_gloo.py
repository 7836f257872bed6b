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
    cnt = D.allreduce_counters({"admissible": r.report["admissible"], "pairs": r.report["pairs_in"]}, "cpu")
    if rank == 0:
        ret["full"] = full.numpy().tolist()
        ret["cnt"] = cnt
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
