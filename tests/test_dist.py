"""World-size-2 gloo test of the multi-GPU plumbing (paper_2506_08276_b200/dist.py):
query shards are disjoint and cover each step, the gathered results equal the
single-process results, and timings reduce to the max over ranks."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_search(idx: np.ndarray, k: int = 3):
    """Deterministic stand-in for a per-query search result."""
    ids = (idx[:, None] * 7 + np.arange(k)[None, :]) % 1000
    d = -(idx[:, None].astype(np.float32) / 100.0) + np.arange(k)[None, :]
    return torch.from_numpy(ids.astype(np.int64)), torch.from_numpy(d.astype(np.float32))


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_08276_b200.dist import gather_results, max_over_ranks, shard_queries, \
        sum_over_ranks
    res = []
    for step in range(3):
        idx = shard_queries(step, rank, world, batch=5, n_queries=12)
        ids, d = _fake_search(idx)
        g_ids, g_d = gather_results(ids, d)
        res.append((g_ids.numpy(), g_d.numpy()))
    t = max_over_ranks(10.0 + rank)
    s = sum_over_ranks([rank, 1])
    if rank == 0:
        out_q.put((res, t, s))
    dist.barrier()
    dist.destroy_process_group()


def test_shards_cover_and_are_disjoint():
    from paper_2506_08276_b200.dist import shard_queries
    for world in (1, 2, 4, 8):
        for step in range(4):
            got = np.concatenate([shard_queries(step, r, world, 64, 4096) for r in range(world)])
            assert len(set(got.tolist())) == got.size == 64 * world


def test_world_size_2_gather_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res, t, s = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_2506_08276_b200.dist import shard_queries
    for step, (g_ids, g_d) in enumerate(res):
        idx = np.concatenate([shard_queries(step, r, 2, 5, 12) for r in range(2)])
        ids, d = _fake_search(idx)
        assert np.array_equal(g_ids, ids.numpy())
        assert np.array_equal(g_d, d.numpy())
    assert t == 11.0
    assert s == [1.0, 2.0]


def test_shard_bounds_cover_uneven_batches():
    from paper_2506_08276_b200.dist import shard_bounds
    for B in (0, 1, 7, 101, 4096):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(B, r, world) for r in range(world)]
            rows = [i for lo, hi in spans for i in range(lo, hi)]
            assert rows == list(range(B))
